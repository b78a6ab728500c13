"""Build libtacsnn.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2603_13810_b200.build [--force] [--verbose]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2603_13810_b200/libtacsnn.so`` (C ABI only, no torch types), which the
ctypes binding (tacsnn.py) loads.  Objects are cached under build/ by mtime.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# Variant builds for A/B timing: TACSNN_LIB_NAME=libtacsnn_x.so TACSNN_DEFS="-DFOO=1"
# (load with TACSNN_LIB=<pkg>/libtacsnn_x.so); the default build is libtacsnn.so.
_NAME = os.environ.get("TACSNN_LIB_NAME", "libtacsnn.so")
_DEFS = os.environ.get("TACSNN_DEFS", "").split()
OBJ = os.path.join(ROOT, "build", "obj" if _NAME == "libtacsnn.so" else "obj_" + _NAME.replace(".so", ""))
LIB = os.path.join(PKG, _NAME)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps(src):
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "tacsnn.h")]
    return [src] + hdrs


def _compile(src, force, verbose, ptxas_v):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    trace = os.environ.get("TACSNN_TRACE") == "1"  # debug timeline build (see tc.cu trace_mark)
    if not force and os.path.exists(obj) and all(
            os.path.getmtime(obj) >= os.path.getmtime(d) for d in _deps(src)):
        return obj, ""
    cmd = [nvcc(), *ARCH, *FLAGS, *(["-DTACSNN_TRACE"] if trace else []), *_DEFS, "-c", src, "-o", obj]
    if ptxas_v:
        cmd += ["-Xptxas", "-v"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose, ptxas_v), srcs))
    objs = [o for o, _ in results]
    if ptxas_v:
        for _, log in results:
            if log:
                print(log)
    if force or not os.path.exists(LIB) or any(
            os.path.getmtime(LIB) < os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
               "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.ptxas_v))
