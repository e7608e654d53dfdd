"""TEST INFRASTRUCTURE ONLY -- ctypes bindings of the two CPU checkers.

* ``Oracle``    -> oracle/_build/librvk_oracle.so, the plain-C restatement
  (oracle/rvk_oracle.c), always built by ``__graft_entry__.build()``.
* ``Reference`` -> oracle/_ref/librvk_ref.so, the UNMODIFIED reference
  sources (/root/reference/proj/src) compiled by oracle/Makefile. Present
  wherever it was built (this container; the GPU box receives the prebuilt
  file with the repo snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "librvk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librvk_ref.so")

RVK_OK, RVK_EINVAL, RVK_ECLUSTER_TOO_SMALL = 0, 1, 2


class RansacParams(C.Structure):
    """rvk_ransac_params (include/rvk_gpu.h) == rvk::RansacParams (ransac.hpp:19-23)."""

    _fields_ = [("max_trials", C.c_int32), ("reserved", C.c_int32),
                ("threshold_scale", C.c_double), ("rng_seed", C.c_uint64)]


class Estimate(C.Structure):
    """rvk_estimate (include/rvk_gpu.h) == rvk::VelocityEstimate (types.hpp:57-65)."""

    _fields_ = [("frame_id", C.c_int64), ("cluster_id", C.c_int32), ("inlier_count", C.c_int32),
                ("v_x", C.c_double), ("v_y", C.c_double), ("heading", C.c_double),
                ("has_heading", C.c_int32), ("condition_ok", C.c_int32)]


ESTIMATE_DTYPE = np.dtype([("frame_id", "<i8"), ("cluster_id", "<i4"), ("inlier_count", "<i4"),
                           ("v_x", "<f8"), ("v_y", "<f8"), ("heading", "<f8"),
                           ("has_heading", "<i4"), ("condition_ok", "<i4")])
assert ESTIMATE_DTYPE.itemsize == C.sizeof(Estimate)


class CheckerError(RuntimeError):
    def __init__(self, status: int, msg: str, cluster: int = -1):
        super().__init__(msg)
        self.status, self.cluster = status, cluster


def _p(a, ctype):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class RansacResult:
    inlier_count: np.ndarray   # int32 [C]
    winning_trial: np.ndarray  # int32 [C]
    mask: np.ndarray           # uint8 [P]


def make_params(max_trials=256, threshold_scale=1.0, rng_seed=0) -> RansacParams:
    return RansacParams(int(max_trials), 0, float(threshold_scale), int(rng_seed) & (2**64 - 1))


def _csr(offsets, az, dop):
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    az = np.ascontiguousarray(az, dtype=np.float64)
    dop = np.ascontiguousarray(dop, dtype=np.float64)
    return offsets, az, dop


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.path = path

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, st):
        if st != RVK_OK:
            msg = self._fn("last_error")
            msg.restype = C.c_char_p
            raise CheckerError(st, msg().decode())


class _Clustering:
    """dbscan / extract_clusters (src/clustering.cpp:24-155) through a checker
    library that exports <prefix>dbscan and <prefix>extract_clusters."""

    def dbscan(self, x, y, z=None, eps=2.0, min_pts=3, features=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        z = None if z is None else np.ascontiguousarray(z, dtype=np.float64)
        labels = np.zeros(x.size, np.int32)
        f = self._fn("dbscan")
        f.argtypes = [C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.c_double, C.c_int32, C.c_int32,
                      C.POINTER(C.c_int32)]
        self._check(f(x.size, _p(x, C.c_double), _p(y, C.c_double), _p(z, C.c_double), eps,
                      min_pts, features, _p(labels, C.c_int32)))
        return labels

    def extract_clusters(self, labels, min_cluster_size=3):
        """-> (labels rewritten, offsets[m+1], point_indices[offsets[m]])."""
        labels = np.array(labels, dtype=np.int32)
        n = labels.size
        offsets = np.zeros(n + 2, np.int64)
        pi = np.zeros(max(n, 1), np.int32)
        m = C.c_int32(0)
        f = self._fn("extract_clusters")
        f.argtypes = [C.c_int64, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                      C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        self._check(f(n, _p(labels, C.c_int32), min_cluster_size, C.byref(m),
                      _p(offsets, C.c_int64), _p(pi, C.c_int32)))
        off = offsets[:m.value + 1].copy()
        return labels, off, pi[:int(off[-1])].copy()


def _combine(self, labels, mask_ids, mask_offsets, masks):
    labels = np.ascontiguousarray(labels, np.int32)
    ids = np.ascontiguousarray(mask_ids, np.int32)
    off = np.ascontiguousarray(mask_offsets, np.int64)
    m = np.ascontiguousarray(masks, np.uint8)
    out = np.zeros(labels.size, np.uint8)
    f = self._fn("combine_masks")
    f.argtypes = [C.c_int64, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                  C.POINTER(C.c_int64), C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]
    self._check(f(labels.size, _p(labels, C.c_int32), ids.size, _p(ids, C.c_int32),
                  _p(off, C.c_int64), _p(m, C.c_uint8), _p(out, C.c_uint8)))
    return out


_Clustering.combine_masks = _combine


class Oracle(_Lib, _Clustering):
    """The C restatement (oracle/rvk_oracle.c)."""

    prefix = "rvk_or_"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        self._fn("rng_u64").restype = C.c_uint64
        self._fn("prepare_cluster").restype = C.c_double
        self._fn("run_trial").restype = C.c_int32

    def rng_u64(self, seed, hi, lo, k):
        f = self._fn("rng_u64")
        f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32]
        return int(f(seed & (2**64 - 1), hi & (2**64 - 1), lo & (2**64 - 1), k))

    def seed_pair(self, seed, cluster, trial, n):
        i, j = C.c_int32(), C.c_int32()
        f = self._fn("seed_pair")
        f.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                      C.POINTER(C.c_int32)]
        self._check(f(seed & (2**64 - 1), cluster, trial, n, C.byref(i), C.byref(j)))
        return i.value, j.value

    def run_trial(self, xy, a, b, thr, want_mask=False):
        xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1)
        n = xy.size // 2
        mask = np.zeros(n, np.uint8) if want_mask else None
        f = self._fn("run_trial")
        f.argtypes = [C.c_int64, C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_double,
                      C.POINTER(C.c_uint8)]
        cnt = f(n, _p(xy, C.c_double), a, b, thr, _p(mask, C.c_uint8))
        return (cnt, mask) if want_mask else cnt

    def sequential_ransac(self, offsets, az, dop, params, key=None) -> RansacResult:
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        cnt = np.zeros(n, np.int32)
        tr = np.zeros(n, np.int32)
        mask = np.zeros(az.size, np.uint8)
        key = None if key is None else np.ascontiguousarray(key, np.int32)
        self._check(self._fn("sequential_ransac")(
            n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double), C.byref(params),
            _p(key, C.c_int32), _p(cnt, C.c_int32), _p(tr, C.c_int32), _p(mask, C.c_uint8)))
        return RansacResult(cnt, tr, mask)

    def trial_counts(self, offsets, az, dop, params, key=None):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        out = np.zeros(n * params.max_trials, np.int32)
        key = None if key is None else np.ascontiguousarray(key, np.int32)
        self._check(self._fn("trial_counts")(
            n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double), C.byref(params),
            _p(key, C.c_int32), _p(out, C.c_int32)))
        return out.reshape(n, params.max_trials)

    def cluster_thresholds(self, offsets, az, dop, scale):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        norm = np.zeros(4 * n)
        thr = np.zeros(n)
        xy = np.zeros(2 * az.size)
        f = self._fn("cluster_thresholds")
        f.argtypes = [C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._check(f(n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double), scale,
                      _p(norm, C.c_double), _p(thr, C.c_double), _p(xy, C.c_double)))
        return norm.reshape(n, 4), thr, xy.reshape(-1, 2)

    def estimate_all(self, offsets, az, dop, mask, frame_id=0, cluster_ids=None):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        out = np.zeros(n, ESTIMATE_DTYPE)
        mask = np.ascontiguousarray(mask, np.uint8)
        ids = None if cluster_ids is None else np.ascontiguousarray(cluster_ids, np.int32)
        f = self._fn("estimate_all")
        f.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                      C.c_void_p]
        self._check(f(frame_id, n, _p(offsets, C.c_int64), _p(az, C.c_double),
                      _p(dop, C.c_double), _p(ids, C.c_int32), _p(mask, C.c_uint8),
                      out.ctypes.data))
        return out

    def ransac_estimate_range(self, offsets, az, dop, params, c_begin, c_end, frame_id=0):
        """Sequential RANSAC + LSQ over clusters [c_begin, c_end) (bounded CPU samples)."""
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        cnt = np.zeros(n, np.int32)
        tr = np.zeros(n, np.int32)
        mask = np.zeros(az.size, np.uint8)
        out = np.zeros(n, ESTIMATE_DTYPE)
        f = self._fn("ransac_estimate_range")
        f.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(RansacParams),
                      C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                      C.POINTER(C.c_uint8), C.c_void_p]
        self._check(f(frame_id, n, _p(offsets, C.c_int64), _p(az, C.c_double),
                      _p(dop, C.c_double), None, C.byref(params), c_begin, c_end,
                      _p(cnt, C.c_int32), _p(tr, C.c_int32), _p(mask, C.c_uint8),
                      out.ctypes.data))
        return RansacResult(cnt, tr, mask), out


class Reference(_Lib, _Clustering):
    """The unmodified reference (oracle/_ref/librvk_ref.so, via oracle/ref_capi.cpp)."""

    prefix = "rvk_ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        self._fn("rng_u64").restype = C.c_uint64

    def _check(self, st):
        if st != RVK_OK:
            msg = self._fn("last_error")
            msg.restype = C.c_char_p
            cl = self._fn("last_error_cluster")()
            raise CheckerError(st, msg().decode(), cl)

    def rng_u64(self, seed, hi, lo, k):
        f = self._fn("rng_u64")
        f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32]
        return int(f(seed & (2**64 - 1), hi & (2**64 - 1), lo & (2**64 - 1), k))

    def seed_pair(self, seed, cluster, trial, n):
        i, j = C.c_int32(), C.c_int32()
        f = self._fn("seed_pair")
        f.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                      C.POINTER(C.c_int32)]
        self._check(f(seed & (2**64 - 1), cluster, trial, n, C.byref(i), C.byref(j)))
        return i.value, j.value

    def run_ransac(self, offsets, az, dop, params, workers=0) -> RansacResult:
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        cnt = np.zeros(n, np.int32)
        tr = np.zeros(n, np.int32)
        mask = np.zeros(az.size, np.uint8)
        f = self._fn("run_ransac")
        self._check(f(n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double),
                      C.byref(params), C.c_int32(workers), _p(cnt, C.c_int32),
                      _p(tr, C.c_int32), _p(mask, C.c_uint8)))
        return RansacResult(cnt, tr, mask)

    def sequential_ransac(self, offsets, az, dop, params) -> RansacResult:
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        cnt = np.zeros(n, np.int32)
        tr = np.zeros(n, np.int32)
        mask = np.zeros(az.size, np.uint8)
        self._check(self._fn("sequential_ransac")(
            n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double), C.byref(params),
            _p(cnt, C.c_int32), _p(tr, C.c_int32), _p(mask, C.c_uint8)))
        return RansacResult(cnt, tr, mask)

    def trial_counts(self, offsets, az, dop, params):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        out = np.zeros(n * params.max_trials, np.int32)
        self._check(self._fn("trial_counts")(
            n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double), C.byref(params),
            _p(out, C.c_int32)))
        return out.reshape(n, params.max_trials)

    def cluster_thresholds(self, offsets, az, dop, scale):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        norm = np.zeros(4 * n)
        thr = np.zeros(n)
        xy = np.zeros(2 * az.size)
        f = self._fn("cluster_thresholds")
        f.argtypes = [C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._check(f(n, _p(offsets, C.c_int64), _p(az, C.c_double), _p(dop, C.c_double), scale,
                      _p(norm, C.c_double), _p(thr, C.c_double), _p(xy, C.c_double)))
        return norm.reshape(n, 4), thr, xy.reshape(-1, 2)

    def _est(self, name, offsets, az, dop, mask, frame_id, cluster_ids, workers=None):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        out = np.zeros(n, ESTIMATE_DTYPE)
        mask = np.ascontiguousarray(mask, np.uint8)
        ids = None if cluster_ids is None else np.ascontiguousarray(cluster_ids, np.int32)
        args = [C.c_int64(frame_id), n, _p(offsets, C.c_int64), _p(az, C.c_double),
                _p(dop, C.c_double), _p(ids, C.c_int32), _p(mask, C.c_uint8)]
        if workers is not None:
            args.append(C.c_int32(workers))
        args.append(C.c_void_p(out.ctypes.data))
        self._check(self._fn(name)(*args))
        return out

    def estimate_all(self, offsets, az, dop, mask, frame_id=0, cluster_ids=None, workers=0):
        return self._est("estimate_all", offsets, az, dop, mask, frame_id, cluster_ids, workers)

    def sequential_lsq(self, offsets, az, dop, mask, frame_id=0, cluster_ids=None):
        return self._est("sequential_lsq", offsets, az, dop, mask, frame_id, cluster_ids)

    def ransac_estimate(self, offsets, az, dop, params, workers=0, frame_id=0, cluster_ids=None):
        offsets, az, dop = _csr(offsets, az, dop)
        n = offsets.size - 1
        cnt = np.zeros(n, np.int32)
        tr = np.zeros(n, np.int32)
        mask = np.zeros(az.size, np.uint8)
        out = np.zeros(n, ESTIMATE_DTYPE)
        ids = None if cluster_ids is None else np.ascontiguousarray(cluster_ids, np.int32)
        self._check(self._fn("ransac_estimate")(
            C.c_int64(frame_id), n, _p(offsets, C.c_int64), _p(az, C.c_double),
            _p(dop, C.c_double), _p(ids, C.c_int32), C.byref(params), C.c_int32(workers),
            _p(cnt, C.c_int32), _p(tr, C.c_int32), _p(mask, C.c_uint8),
            C.c_void_p(out.ctypes.data)))
        return RansacResult(cnt, tr, mask), out

    def write_frames(self, path, frames):
        """frames: list of (frame_id, x, y, z, doppler, azimuth) -> the reference's CSV."""
        ids = np.array([f[0] for f in frames], np.int64)
        sizes = [len(f[1]) for f in frames]
        off = np.zeros(len(frames) + 1, np.int64)
        np.cumsum(sizes, out=off[1:])
        cols = [np.ascontiguousarray(np.concatenate([f[k] for f in frames]) if frames
                                     else np.zeros(0), np.float64) for k in range(1, 6)]
        f = self._fn("write_frames")
        f.argtypes = [C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)] + \
            [C.POINTER(C.c_double)] * 5 + [C.c_char_p]
        self._check(f(len(frames), _p(ids, C.c_int64), _p(off, C.c_int64),
                      *[_p(c, C.c_double) for c in cols], path.encode()))

    def run_estimate_csv(self, frames_path, out_path, mode="parallel", eps=2.0, min_pts=3,
                         max_trials=256, threshold_scale=1.0, seed=0):
        f = self._fn("run_estimate_csv")
        f.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.c_double, C.c_int32, C.c_int32,
                      C.c_double, C.c_uint64]
        self._check(f(frames_path.encode(), out_path.encode(),
                      0 if mode == "parallel" else 2, eps, min_pts, max_trials, threshold_scale,
                      seed))

    def rng_units(self, seed, hi, lo, out):
        f = self._fn("rng_units")
        f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
        f.restype = None
        f(seed & (2**64 - 1), hi & (2**64 - 1), lo & (2**64 - 1), out.size,
          _p(out, C.c_double))
        return out

    def generate_frame(self, seed, objects, offset_range=(2.0, 5.0)):
        objects = np.ascontiguousarray(objects, np.float64).reshape(-1, 10)
        p = int(objects[:, 6].sum())
        x, y, d, a = (np.zeros(p) for _ in range(4))
        flag = np.zeros(p, np.int32)
        f = self._fn("generate_frame")
        f.argtypes = [C.c_uint64, C.c_int32, C.POINTER(C.c_double), C.c_double, C.c_double] + \
            [C.POINTER(C.c_double)] * 4 + [C.POINTER(C.c_int32)]
        self._check(f(seed, objects.shape[0], _p(objects, C.c_double), offset_range[0],
                      offset_range[1], _p(x, C.c_double), _p(y, C.c_double), _p(d, C.c_double),
                      _p(a, C.c_double), _p(flag, C.c_int32)))
        return x, y, d, a, flag


def build(reference: bool = True, quiet: bool = True) -> None:
    """Build the C oracle (always) and the reference library (when /root/reference exists)."""
    targets = ["oracle"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    out = subprocess.run(["make", "-C", HERE, "-j8", *targets], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
