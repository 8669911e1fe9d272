"""Build libatom.so in-tree: every csrc/*.cu / *.cpp compiled by nvcc for sm_100a.

    python -m paper_2403_10504_b200.build [-j N] [--force]

Objects go to paper_2403_10504_b200/build/, the shared library to
paper_2403_10504_b200/libatom.so (git-ignored, travels to the GPU box with gpurun).
Static cudart; NCCL from the torch-bundled wheel (the same libnccl.so.2 torch loads).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libatom.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for p in spec.submodule_search_locations:
            cands.append(os.path.join(p, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _flags():
    inc, _ = _nccl_dirs()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                   "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]


def _needs(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    return max(os.path.getmtime(src), hdr_mtime) > os.path.getmtime(obj)


def build(force=False, jobs=None, verbose=True):
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_mtime = max([os.path.getmtime(h) for h in hdrs] + [os.path.getmtime(__file__)])
    flags = _flags()
    todo = []
    objs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _needs(s, o, hdr_mtime):
            todo.append((s, o))

    def comp(so):
        s, o = so
        cmd = [NVCC] + flags + ["-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return s, r

    errors = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
            for s, r in ex.map(comp, todo):
                if verbose:
                    print(f"[build] {os.path.basename(s)}", file=sys.stderr)
                if r.returncode != 0:
                    errors.append((s, r.stderr))
                elif verbose and ("warning" in r.stderr):
                    print(r.stderr, file=sys.stderr)
    if errors:
        for s, e in errors:
            print(f"--- {s}\n{e}", file=sys.stderr)
        raise RuntimeError(f"libatom build failed ({len(errors)} files)")
    if todo or not os.path.exists(LIB) or max(os.path.getmtime(o) for o in objs) > os.path.getmtime(LIB):
        _, libdir = _nccl_dirs()
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            print(r.stderr, file=sys.stderr)
            raise RuntimeError("libatom link failed")
        if verbose:
            print(f"[build] linked {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
