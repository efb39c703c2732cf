"""Build libblindmatch.so in-tree (sm_100a).  Usage: python -m paper_2408_06167_b200.build"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
# BM_VARIANT=name (A/B builds only, tools/ab.sh): objects in build/var_<name>, the library at
# paper_2408_06167_b200/variants/libblindmatch_<name>.so (loaded with BM_LIB_PATH); the product is the default
_VAR = os.environ.get("BM_VARIANT")
BUILD = os.path.join(ROOT, "build", f"var_{_VAR}") if _VAR else os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "variants", f"libblindmatch_{_VAR}.so") if _VAR else os.path.join(PKG, "libblindmatch.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = ["host.cpp", "device.cu"]
HEADERS = ["bm_common.cuh", "bm_host.h", "ntt_base.cuh", "ntt2.cuh", "ntt3.cuh", "ntt3f.cuh",
           "k_match.cuh", "k_tensor_mma.cuh", "k_next.cuh", "k_setup.cuh"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force=False, verbose=True):
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INC, "blindmatch.h")]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not (force or _newer(obj, [path] + hdrs)):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   *os.environ.get("BM_NVCC_FLAGS", "").split(), "-I", INC, "-c", path, "-o", obj]
        else:
            cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", "-Wno-unknown-pragmas",
                   "-I", os.path.join(CUDA, "include"), "-I", INC, "-c", path, "-o", obj]
        _run(cmd, verbose)
    if force or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lquadmath", "-lpthread"], verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
