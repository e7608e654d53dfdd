"""ctypes binding of the in-tree native libraries.

* ``lib/librvk_gpu.so``   -- the sm_100a kernels + C-ABI (include/rvk_gpu.h).
* ``lib/librvk_probe.so`` -- the FP32-pipe peak probe (bench.py's roofline denominator).

There is no fallback: if the CUDA library is missing, ``gpu()`` raises. Build
with ``python -m paper_2012_12618_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PKG, "lib")
# RVK_GPU_SO: an alternative in-tree build of the same library (A/B of kernel variants)
GPU_SO = os.environ.get("RVK_GPU_SO") or os.path.join(LIB_DIR, "librvk_gpu.so")
PROBE_SO = os.path.join(LIB_DIR, "librvk_probe.so")

RVK_OK, RVK_EINVAL, RVK_ECLUSTER_TOO_SMALL, RVK_ECUDA, RVK_ENOMEM = range(5)


class RansacParamsC(C.Structure):
    """rvk_ransac_params (include/rvk_gpu.h)."""

    _fields_ = [("max_trials", C.c_int32), ("reserved", C.c_int32),
                ("threshold_scale", C.c_double), ("rng_seed", C.c_uint64)]


class ClusteringParamsC(C.Structure):
    """rvk_clustering_params (include/rvk_gpu.h)."""

    _fields_ = [("eps", C.c_double), ("min_pts", C.c_int32), ("features", C.c_int32)]


class EstimateC(C.Structure):
    """rvk_estimate (include/rvk_gpu.h)."""

    _fields_ = [("frame_id", C.c_int64), ("cluster_id", C.c_int32), ("inlier_count", C.c_int32),
                ("v_x", C.c_double), ("v_y", C.c_double), ("heading", C.c_double),
                ("has_heading", C.c_int32), ("condition_ok", C.c_int32)]


ESTIMATE_DTYPE = np.dtype([("frame_id", "<i8"), ("cluster_id", "<i4"), ("inlier_count", "<i4"),
                           ("v_x", "<f8"), ("v_y", "<f8"), ("heading", "<f8"),
                           ("has_heading", "<i4"), ("condition_ok", "<i4")])
assert ESTIMATE_DTYPE.itemsize == C.sizeof(EstimateC) == 48

_lock = threading.Lock()
_gpu = None

_P = C.c_void_p
_I32, _I64, _U64, _F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double

# name -> (restype, argtypes); every symbol declared in include/rvk_gpu.h.
GPU_SIGNATURES = {
    "rvk_abi_version": (_I32, []),
    "rvk_last_error": (C.c_char_p, []),
    "rvk_last_error_cluster": (_I32, []),
    "rvk_kernel_launches": (_I64, []),
    "rvk_reset_kernel_launches": (None, []),
    "rvk_run_ransac": (C.c_int, [_I32, _P, _P, _P, _P, _P, _I32, _P, _P, _P]),
    "rvk_estimate_all": (C.c_int, [_I64, _I32, _P, _P, _P, _P, _P, _I32, _P]),
    "rvk_ransac_estimate": (C.c_int, [_I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "rvk_ransac_estimate_packed": (C.c_int, [_I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                             _P]),
    "rvk_ransac_estimate_multi": (C.c_int, [_I32, _P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                                            _P, _P]),
    "rvk_ransac_estimate_device": (C.c_int, [_I64, _I32, _I64, _P, _P, _P, _P, _P, _P, _P, _P,
                                             _P, _P, _P]),
    "rvk_trial_counts": (C.c_int, [_I32, _P, _P, _P, _P, _P, _P]),
    "rvk_seed_pairs": (C.c_int, [_I32, _P, _P, _P, _P]),
    "rvk_cluster_thresholds": (C.c_int, [_I32, _P, _P, _P, _F64, _P, _P]),
    "rvk_stream_create": (C.c_int, [_P, _I32, _P]),
    "rvk_stream_submit": (C.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "rvk_stream_submit_packed": (C.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                           _P]),
    "rvk_stream_wait": (C.c_int, [_P, _I64]),
    "rvk_stream_destroy": (C.c_int, [_P]),
    "rvk_dbscan": (C.c_int, [_I64, _P, _P, _P, _P, _P]),
    "rvk_extract_clusters": (C.c_int, [_I64, _P, _I32, _P, _P, _P]),
    "rvk_estimate_frame": (C.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P,
                                     _P, _P, _P, _P]),
    "rvk_combine_masks": (C.c_int, [_I64, _P, _I32, _P, _P, _P, _P]),
    "rvk_profile_enable": (None, [_I32]),
    "rvk_profile_read": (C.c_int, [_P, _P, _I32]),
}

def _bind(lib, sigs):
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def gpu():
    """The CUDA library (loads it on first use; raises if it was not built)."""
    global _gpu
    with _lock:
        if _gpu is None:
            if not os.path.exists(GPU_SO):
                raise RuntimeError(
                    f"{GPU_SO} is missing: build it with `python -m paper_2012_12618_b200.build` "
                    "(there is no CPU fallback)")
            _gpu = _bind(C.CDLL(GPU_SO), GPU_SIGNATURES)
            if _gpu.rvk_abi_version() != 1:
                raise RuntimeError("librvk_gpu.so ABI mismatch")
        return _gpu


def probe():
    """FP32-peak probe library (measurement only)."""
    lib = C.CDLL(PROBE_SO)
    lib.rvk_probe_fp32.restype = C.c_int
    lib.rvk_probe_fp32.argtypes = [_I32, _I32, _I32, _P, _P]
    lib.rvk_probe_flops.restype = _I64
    lib.rvk_probe_flops.argtypes = [_I32, _I32]
    return lib


def ptr(a):
    """Raw data pointer of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor
