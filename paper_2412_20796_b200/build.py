"""Build libchg.so (the C-ABI library) in-tree for sm_100a with nvcc.

Objects go to paper_2412_20796_b200/build/, the library to
paper_2412_20796_b200/libchg.so.  Rebuilds only what changed (mtime).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# CHG_BUILD_DEBUG=1: a separate timing/debug build (-DCHG_TC_DEBUG: CHG_TC_SKIP knobs, per-CTA
# trace) into libchg_dbg.so, loaded with CHG_LIB_PATH; the product library never has the knobs
DEBUG = os.environ.get("CHG_BUILD_DEBUG") == "1"
OBJ = os.path.join(PKG, "build_dbg" if DEBUG else "build")
LIB = os.path.join(PKG, "libchg_dbg.so" if DEBUG else "libchg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (same soname torch loads)
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _flags():
    return _flags_base() + (["-DCHG_TC_DEBUG"] if DEBUG else [])


def _flags_base():
    inc, _ = _nccl_dirs()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + inc,
                   "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr", "-Xptxas", "-v"] \
        if os.environ.get("CHG_PTXAS_V") else \
        ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + inc,
                "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "chg.h")]
    hdr_mtime = max(os.path.getmtime(h) for h in hdrs)
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s).replace(".cu", ".o"))
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_mtime):
            jobs.append([NVCC] + _flags() + ["-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)
        return cmd[-3]

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for done in ex.map(run, jobs):
            if verbose:
                print("compiled", os.path.basename(done), file=sys.stderr)
    if jobs or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _, libdir = _nccl_dirs()
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
