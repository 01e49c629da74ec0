"""SASS instruction census and ptxas resource report of libtilefact.so (measurement
hygiene: what the tile kernels compile to on sm_100a).

    python tools/sass_census.py > profiles/r02_sass_census.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_0709_1272_b200", "libtilefact.so")
OPS = ["DMMA", "DFMA", "DADD", "DMUL", "LDGSTS", "UBLKCP", "UTMALDG", "REDG", "ATOMG", "LDS", "STS", "LDG", "STG",
       "LDL", "STL", "BAR", "SYNCS", "SHFL", "REDUX", "MATCH", "NOP", "CALL"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
        return dict(zip(names, out))
    except OSError:
        return {n: n for n in names}


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    # split into functions: kernels ("Function : ...") and their internal device functions
    # (labels "$<kernel>$<function>:" inside the kernel's text)
    funcs = collections.OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*\$\S+?\$(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs.setdefault(cur, collections.Counter())
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m and cur:
            funcs[cur]["n"] += 1
            op = m.group(2)
            for o in OPS:
                if op == o or op.startswith(o):
                    funcs[cur][o] += 1
                    break
    dm = demangle(list(funcs))
    print("# SASS census of libtilefact.so (sm_100a)\n")
    print(f"`cuobjdump -sass {os.path.relpath(LIB, ROOT)}`; per function (kernels and the noinline tile-kernel "
          "variants they call).  FP64 tensor work is `DMMA.8x8x4` (mma.sync m8n8k4 f64; tcgen05 has no f64 kind on "
          "sm_100a), operand staging is `LDGSTS` (cp.async) and `LDS`; `REDG` is the GEMM/SYRK epilogue's L2 "
          "reduction.  No `UTMALDG` / `UBLKCP`: no TMA in the default build.\n")
    cols = ["n"] + OPS
    print("| function | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    tot = collections.Counter()
    for f, c in funcs.items():
        if c["n"] < 50:
            continue
        name = dm.get(f, f)
        name = re.sub(r"\(.*", "", name)[:70]
        print(f"| `{name}` | " + " | ".join(str(c[k]) for k in cols) + " |")
        tot.update(c)
    print("| **total** | " + " | ".join(str(tot[k]) for k in cols) + " |\n")
    log = os.path.join(ROOT, "paper_0709_1272_b200", "build_ptxas.log")
    if os.path.exists(log):
        print("## ptxas resource usage (registers, stack, spills) per function\n")
        print("| function | regs | stack B | spill st B | spill ld B |")
        print("|---|---|---|---|---|")
        txt = open(log).read()
        props = re.findall(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, "
                           r"(\d+) bytes spill loads(?:\n[^\n]*Used (\d+) registers)?", txt)
        names = demangle([p[0] for p in props])
        for fn, st, ss, sl, regs in props:
            print(f"| `{re.sub(r'[(].*', '', names.get(fn, fn))[:70]}` | {regs or '-'} | {st} | {ss} | {sl} |")


if __name__ == "__main__":
    main()
