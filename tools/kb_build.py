"""Build single-kind kbench binaries in parallel: build/kb_<kind> (nvcc -DKB_KIND=<id>).

    python tools/kb_build.py gemm getrf tstrf [-D...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["potrf", "trsm", "syrk", "gemm", "geqrt", "larfb", "tsqrt", "ssrfb", "getrf", "gessm", "tstrf", "ssssm"]


def build(kind, defs):
    out = os.path.join(ROOT, "build", f"kb_{kind}")
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
           f"-DKB_KIND={NAMES.index(kind)}", *defs, "-o", out, os.path.join(ROOT, "tools", "kbench.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    lines = [ln for ln in r.stderr.splitlines() if "kb_kernel" in ln or "spill" in ln or "Used" in ln]
    return kind, r.returncode, "\n".join(lines[-6:])


if __name__ == "__main__":
    kinds = [a for a in sys.argv[1:] if not a.startswith("-")]
    defs = [a for a in sys.argv[1:] if a.startswith("-")]
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(kinds)) as ex:
        for kind, rc, log in ex.map(lambda k: build(k, defs), kinds):
            print(f"== {kind} rc={rc}\n{log}")
