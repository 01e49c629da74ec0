"""Build libtilefact.so in-tree with nvcc for sm_100a (B200).

    python -m paper_0709_1272_b200.build [--force]

The library statically links the CUDA runtime so the host-only entry points (task-graph
export, argument validation) load on machines without a GPU.  It has no NCCL
dependency: the multi-GPU data path is device-initiated stores into peers' CUDA-IPC
mapped memory (tf_device.cu), and the handles are exchanged by the caller.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtilefact.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-v",
    "--fmad=true",
    "-cudart", "static",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + [
        os.path.join(ROOT, "include", "tilefact.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def _obj_deps(src):
    """Headers a translation unit depends on (conservative: every header for CUDA files)."""
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")))
    inc = os.path.join(ROOT, "include", "tilefact.h")
    if src.endswith(".cpp"):
        hdrs = [h for h in hdrs if h.endswith(".h")]
    return [src, inc, *hdrs]


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libtilefact.so (or `out`, with extra -D `defines`, for A/B experiments).

    Each source compiles to its own object (so host-only edits do not recompile the
    kernels); objects are rebuilt when the source or a header it depends on changes."""
    lib = out or LIB
    if not force and out is None and not defines and not needs_build():
        return LIB
    tag = "default" if not defines else "_".join(d.replace("=", "-") for d in defines)
    odir = os.path.join(ROOT, "build", "obj", tag)
    os.makedirs(odir, exist_ok=True)
    objs, logs, todo = [], {}, []
    for src in sources():
        obj = os.path.join(odir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj)
                                                     for d in _obj_deps(src)):
            log = obj + ".log"
            if os.path.exists(log):
                logs[src] = open(log).read()
            continue
        todo.append((src, obj))

    def compile_one(job):
        src, obj = job
        tmp = obj + f".tmp{os.getpid()}"
        cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", "-o", tmp, src,
               "-I", os.path.join(ROOT, "include")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc compile of {os.path.basename(src)} failed")
        with open(obj + ".log", "w") as f:
            f.write(r.stderr)
        os.replace(tmp, obj)
        return src, r.stderr

    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, len(todo))) as ex:
        for src, log in ex.map(compile_one, todo):
            logs[src] = log
    logs = [logs[s] for s in sources() if s in logs]
    tmp = lib + f".tmp{os.getpid()}"
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link of libtilefact.so failed")
    if verbose:
        sys.stderr.write("".join(logs))
    if out is None:
        with open(os.path.join(HERE, "build_ptxas.log"), "w") as f:
            f.write("".join(logs))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    defs = []
    for a in args:
        if a.startswith("--out="):
            out = a.split("=", 1)[1]
        elif a.startswith("-D"):
            defs.append(a[2:])
    print(build(force="--force" in args, verbose="-v" in args, out=out, defines=defs))
