"""In-tree native build of the package (no JIT caches, nothing outside the repo).

Outputs (git-ignored, but shipped to the GPU box by gpurun):
  lib/libfragfield_cuda.so   C-ABI + sm_100a kernels + C++ host facade
  lib/_fragfield*.so         pybind11 module over the C++ facade

Usage: python paper_2402_17993_b200/_build.py [--force]   (by path: the package
import itself needs the built libraries)
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "build")
INC = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# The image exports CXX=/opt/gcc/bin/g++ (a wrapper); the system toolchain is the one nvcc uses.
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL: the torch-bundled 2.28.9 (headers + libnccl.so.2 in the venv)
import importlib.util as _ilu

_nv = _ilu.find_spec("nvidia")
NCCL_DIR = os.path.join(list(_nv.submodule_search_locations)[0], "nccl") if _nv else "/usr"
NCCL_INC = os.path.join(NCCL_DIR, "include")
NCCL_LIB = os.path.join(NCCL_DIR, "lib")
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INC,
                  "-I" + NCCL_INC, "-ccbin", CXX]
# experiments only: extra nvcc flags (e.g. FFQ_NVCC_EXTRA="-DSOME_EXPERIMENT")
NVFLAGS += os.environ.get("FFQ_NVCC_EXTRA", "").split()
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-I" + INC, "-I/usr/local/cuda/include"]

CUDA_SOURCES = [os.path.join(CSRC, "ffq_capi.cu")]
CUDA_DEPS = [os.path.join(CSRC, f) for f in ("ffq_compile.hpp", "ffq_kernels.cuh", "ffq_sparse.cuh",
                                               "ffq_shard.inl", "ffq_sector.cuh", "ffq_krylov.inl",
                                               "ffq_compact.inl", "ffq_multi.inl")] + [
    os.path.join(INC, "fragfield_cuda.h")]
HOST_SOURCES = [os.path.join(CSRC, "host", "fragfield_host.cpp")]
HOST_DEPS = [os.path.join(INC, "fragfield", f) for f in os.listdir(os.path.join(INC, "fragfield"))]
PY_SOURCE = os.path.join(CSRC, "host", "pymodule.cpp")

LIBCUDA = os.path.join(LIB, "libfragfield_cuda.so")
EXT_SUFFIX = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PYMOD = os.path.join(LIB, "_fragfield" + EXT_SUFFIX)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd):
    print("[build]", " ".join(os.path.basename(c) if c.startswith(ROOT) else c for c in cmd[:3]), "...",
          flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    for src in CUDA_SOURCES:
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        if force or _stale(o, [src] + CUDA_DEPS):
            _run([NVCC] + NVFLAGS + ["-c", src, "-o", o])
        objs.append(o)
    for src in HOST_SOURCES:
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        if force or _stale(o, [src] + HOST_DEPS + CUDA_DEPS):
            _run([CXX] + CXXFLAGS + ["-c", src, "-o", o])
        objs.append(o)
    if force or _stale(LIBCUDA, objs):
        _run([NVCC] + ARCH + ["-shared", "-ccbin", CXX, "-o", LIBCUDA] + objs +
             ["-L" + NCCL_LIB, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + NCCL_LIB])
    import pybind11

    if force or _stale(PYMOD, [PY_SOURCE, LIBCUDA] + HOST_DEPS):
        _run([CXX] + CXXFLAGS + ["-shared", "-I" + pybind11.get_include(),
                                 "-I" + sysconfig.get_paths()["include"], PY_SOURCE, "-o", PYMOD,
                                 "-L" + LIB, "-lfragfield_cuda", "-Wl,-rpath,$ORIGIN"])


if __name__ == "__main__":
    build(force="--force" in sys.argv)
