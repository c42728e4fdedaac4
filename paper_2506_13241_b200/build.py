"""In-tree build of the native pieces (no pip install, no JIT cache).

* ``libppgpu.so``      -- CUDA kernels + C-ABI (include/pauliprop_gpu.h), sm_100a
* ``_pauliprop*.so``   -- pybind11 module: host C++ API + Python drop-in
* ``oracle/_build/libpporacle.so`` -- the C restatement used as the checker
* ``oracle/_ref/libppref.so``      -- the reference compiled in place (only
  when /root/reference is present; the .so then travels with the repo)

Run ``python -m paper_2506_13241_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(CSRC, "host")
INCLUDE = os.path.join(ROOT, "include")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

GPU_LIB = os.path.join(PKG, "libppgpu.so")
EXT_SUFFIX = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PY_EXT = os.path.join(PKG, "_pauliprop" + EXT_SUFFIX)
ORACLE_LIB = os.path.join(ROOT, "oracle", "_build", "libpporacle.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd, **kw):
    print("[build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, **kw)


def _sources(d, exts):
    return [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith(exts)]


def build_gpu(force=False):
    srcs = _sources(CSRC, (".cu", ".cuh")) + [os.path.join(INCLUDE, "pauliprop_gpu.h")]
    if not force and not _newer(GPU_LIB, srcs):
        return
    _run([NVCC, "-std=c++17", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
          "-o", GPU_LIB, os.path.join(CSRC, "pp_engine.cu")])


def build_ext(force=False):
    import pybind11

    srcs = _sources(HOST, (".cpp", ".hpp")) + [os.path.join(INCLUDE, "pauliprop_gpu.h"), GPU_LIB]
    if not force and not _newer(PY_EXT, srcs):
        return
    py_inc = sysconfig.get_paths()["include"]
    _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-fvisibility=hidden",
          "-I", py_inc, "-I", pybind11.get_include(), "-I", INCLUDE,
          os.path.join(HOST, "pauliprop.cpp"), os.path.join(HOST, "bindings.cpp"),
          "-L", PKG, "-lppgpu", "-Wl,-rpath,$ORIGIN",
          "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart",
          "-o", PY_EXT])


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle", "pp_oracle.c")
    os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
    if force or _newer(ORACLE_LIB, [src]):
        # -ffp-contract=off: one IEEE rounding per operation, as in the reference build
        _run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", src, "-o", ORACLE_LIB, "-lm"])
    script = os.path.join(ROOT, "oracle", "build_ref.sh")
    if os.path.isdir("/root/reference/proj/src"):
        _run(["bash", script])


def build_all(force=False):
    build_gpu(force)
    build_ext(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
