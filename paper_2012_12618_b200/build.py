"""In-tree build of the native libraries (sm_100a only).

    python -m paper_2012_12618_b200.build

* lib/librvk_gpu.so   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3
                      csrc/rvk_kernels.cu csrc/rvk_capi.cu      (C-ABI, include/rvk_gpu.h)
* lib/rvk_gpu          g++ csrc/rvk_cli.cpp: the reference CLI's `estimate` command
                      (frame CSV in, estimate CSV out) on the device path.
* lib/librvk_dropin.so g++ csrc/rvk_dropin.cpp against the Eigen stand-in: the
                      reference's C++ API (rvk::run_ransac, rvk::estimate_all, ...)
                      re-exported over the C-ABI.
Rebuilds only what is out of date.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
REF_INCLUDE = "/root/reference/proj/include"


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout[-6000:] +
                           r.stderr[-6000:])
    return r


def build_gpu(force=False):
    srcs = [os.path.join(CSRC, f) for f in ("rvk_kernels.cu", "rvk_dbscan.cu", "rvk_capi.cu")]
    deps = srcs + [os.path.join(CSRC, f) for f in ("rvk_device.cuh", "rvk_kernels.cuh")] + \
        [os.path.join(INCLUDE, "rvk_gpu.h")]
    out = os.path.join(LIB, "librvk_gpu.so")
    if force or _stale(out, deps):
        # RVK_NVCC_FLAGS: extra -D switches for A/B builds of kernel variants
        extra = os.environ.get("RVK_NVCC_FLAGS", "").split()
        _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              *extra, "-I", INCLUDE, "-o", out, *srcs])
    return out


def build_probe(force=False):
    src = os.path.join(CSRC, "rvk_probe.cu")
    out = os.path.join(LIB, "librvk_probe.so")
    if force or _stale(out, [src]):
        _run([NVCC, *ARCH, "-lineinfo", "-O3", "-Xcompiler", "-fPIC", "-shared", "-o", out, src])
    return out


def build_dropin(force=False):
    """The C++ drop-in needs the reference's public headers (include/rvk/*.hpp)
    only at compile time; it is built where they are available."""
    src = os.path.join(CSRC, "rvk_dropin.cpp")
    out = os.path.join(LIB, "librvk_dropin.so")
    if not os.path.exists(src) or not os.path.isdir(REF_INCLUDE):
        return None
    if force or _stale(out, [src, os.path.join(INCLUDE, "rvk_gpu.h")]):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", REF_INCLUDE, "-I", INCLUDE,
              "-I", os.path.join(ROOT, "compat", "eigen_shim"), "-o", out, src,
              "-L", LIB, "-lrvk_gpu", "-Wl,-rpath,$ORIGIN"])
    return out


def build_cli(force=False):
    """lib/rvk_gpu: the reference CLI's `estimate` command on the device path."""
    src = os.path.join(CSRC, "rvk_cli.cpp")
    out = os.path.join(LIB, "rvk_gpu")
    if force or _stale(out, [src, os.path.join(INCLUDE, "rvk_gpu.h")]):
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-pthread", "-I", INCLUDE, "-o",
              out, src, "-L", LIB, "-lrvk_gpu", "-Wl,-rpath,$ORIGIN"])
    return out


def build(force=False):
    os.makedirs(LIB, exist_ok=True)
    return [build_gpu(force), build_probe(force), build_dropin(force),
            build_cli(force)]


if __name__ == "__main__":
    for p in build(force="--force" in sys.argv):
        if p:
            print(p)
