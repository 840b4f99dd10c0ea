"""Build libddh.so (sm_100a) in-tree: paper_2305_03284_b200/lib/libddh.so.

Compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a`` only (no
other architecture, no PTX fallback).  Run ``python -m paper_2305_03284_b200.build``.
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libddh.so")
# bounds-checked debug build (DDH_DEBUG_BOUNDS: device traps on out-of-tile /
# wrong-colour shared-memory indices and out-of-range global indices), the
# sanitizer substitute run by tests/test_gpu_debug.py
LIB_DEBUG = os.path.join(HERE, "lib", "libddh_debug.so")
SOURCES = ["ddh_kernels.cu", "ddh_stream.cu", "ddh_chain.cu", "ddh_synth.cu", "ddh_api.cpp"]
HEADERS = ["ddh_kernels.h", "ddh_fft.cuh", "ddh_common.cuh", "ddh_f32x2.cuh", "ddh_fft_reg.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-warn-spills",
]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ddh.h")]
    return any(os.path.getmtime(d) > t for d in deps)


# The CUDA runtime is linked dynamically from the toolkit (same image on the GPU box): a static
# cudart would embed every runtime entry point's name in the shipped .so.
CUDA_LIB = "/usr/local/cuda/lib64"
EXTRA = os.environ.get("DDH_NVCC_EXTRA", "").split()


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    objs = []
    bdir = os.path.join(HERE, "lib", "obj_debug" if debug else "obj")
    os.makedirs(bdir, exist_ok=True)
    extra = ["-DDDH_DEBUG_BOUNDS=1"] if debug else []
    for src in SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *EXTRA, *extra, "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd.insert(1, "-x")
            cmd.insert(2, "cu")
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "shared",
           "-Xlinker", "-rpath," + CUDA_LIB, "-o", tmp, *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv))
