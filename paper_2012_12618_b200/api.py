"""Python mirror of the reference's hot-path API, over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:

* ``run_ransac(clusters, params, workers=0)``   include/rvk/ransac.hpp:128-129
* ``estimate_all(frame, clusters, masks, workers=0)`` include/rvk/velocity.hpp:123-125
* ``gather_cluster_points(frame, clusters)``    include/rvk/ransac.hpp:133-134
* ``draw_seed_pair(seed, cluster_id, trial, n)`` include/rvk/ransac.hpp:105

``std::invalid_argument`` maps to ``ValueError``, ``rvk::ClusterTooSmall`` to
``ClusterTooSmall``; CUDA failures raise ``DeviceError`` (there is no CPU
fallback). The CSR entry points (``*_csr``) are the zero-copy form used by the
bench and the parity tests: ``offsets[C+1]`` (int64), ``azimuth[P]``,
``doppler[P]`` (float64), points of cluster c at ``offsets[c]:offsets[c+1]``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N


class ClusterTooSmall(RuntimeError):
    """rvk::ClusterTooSmall (include/rvk/ransac.hpp:47-49)."""

    def __init__(self, msg: str, cluster: int = -1):
        super().__init__(msg)
        self.cluster = cluster


class DeviceError(RuntimeError):
    """A CUDA error inside the native library."""


@dataclass
class RansacParams:
    """rvk::RansacParams (include/rvk/ransac.hpp:19-23)."""

    max_trials: int = 256
    threshold_scale: float = 1.0
    rng_seed: int = 0

    def c(self) -> N.RansacParamsC:
        return N.RansacParamsC(int(self.max_trials), 0, float(self.threshold_scale),
                               int(self.rng_seed) & (2**64 - 1))


@dataclass
class InlierMask:
    """rvk::InlierMask (include/rvk/types.hpp:50-55)."""

    cluster_id: int
    mask: np.ndarray          # bool [n]
    inlier_count: int
    winning_trial: int


@dataclass
class VelocityEstimate:
    """rvk::VelocityEstimate (include/rvk/types.hpp:57-65)."""

    frame_id: int
    cluster_id: int
    v_x: float
    v_y: float
    heading: Optional[float]
    inlier_count: int
    condition_ok: bool


@dataclass
class RadarPoint:
    """rvk::RadarPoint (include/rvk/types.hpp:27-33)."""

    x: float = 0.0
    y: float = 0.0
    z: float = 0.0
    doppler: float = 0.0
    azimuth: float = 0.0


@dataclass
class Frame:
    """rvk::Frame (include/rvk/types.hpp:35-40), struct-of-arrays: the
    RadarPoint fields x, y, z, doppler, azimuth as columns, plus labels
    once clustering has run."""

    frame_id: int = 0
    azimuth: np.ndarray = field(default_factory=lambda: np.zeros(0))
    doppler: np.ndarray = field(default_factory=lambda: np.zeros(0))
    x: np.ndarray = field(default_factory=lambda: np.zeros(0))
    y: np.ndarray = field(default_factory=lambda: np.zeros(0))
    z: np.ndarray = field(default_factory=lambda: np.zeros(0))
    labels: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))


@dataclass
class ClusteringParams:
    """rvk::ClusteringParams (include/rvk/clustering.hpp:13-17)."""

    eps: float = 2.0
    min_pts: int = 3
    features: str = "xy"  # "xy" | "xyz" (rvk::ClusterFeatures)

    def c(self) -> N.ClusteringParamsC:
        if self.features not in ("xy", "xyz"):
            raise ValueError("dbscan: unknown feature space")
        return N.ClusteringParamsC(float(self.eps), int(self.min_pts),
                                   1 if self.features == "xyz" else 0)


@dataclass
class Cluster:
    """rvk::Cluster (include/rvk/types.hpp:43-46)."""

    cluster_id: int
    point_indices: np.ndarray


@dataclass
class RansacResult:
    inlier_count: np.ndarray   # int32 [C]
    winning_trial: np.ndarray  # int32 [C]
    mask: np.ndarray           # uint8 [P]


def _raise(st: int) -> None:
    lib = N.gpu()
    msg = (lib.rvk_last_error() or b"").decode()
    if st == N.RVK_EINVAL:
        raise ValueError(msg)
    if st == N.RVK_ECLUSTER_TOO_SMALL:
        raise ClusterTooSmall(msg, lib.rvk_last_error_cluster())
    if st == N.RVK_ENOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


def _check(st: int) -> None:
    if st != N.RVK_OK:
        _raise(st)


def _csr(offsets, azimuth, doppler):
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    azimuth = np.ascontiguousarray(azimuth, dtype=np.float64)
    doppler = np.ascontiguousarray(doppler, dtype=np.float64)
    if offsets.ndim != 1 or offsets.size < 1:
        raise ValueError("offsets must be a 1-D array of n_clusters + 1 entries")
    if azimuth.shape != doppler.shape or azimuth.size < int(offsets[-1]):
        raise ValueError("azimuth/doppler must hold offsets[-1] points")
    return offsets, azimuth, doppler


def _opt_i32(a, n):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.int32)
    if a.size != n:
        raise ValueError("per-cluster array has the wrong length")
    return a


def clusters_to_csr(clusters: Sequence[np.ndarray]):
    """list of (n, 2) [azimuth, doppler] arrays (Eigen::ArrayX2d) -> CSR."""
    sizes = np.array([np.asarray(c).shape[0] for c in clusters], dtype=np.int64)
    offsets = np.zeros(len(clusters) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    if len(clusters):
        stacked = np.concatenate([np.asarray(c, dtype=np.float64).reshape(-1, 2)
                                  for c in clusters]) if offsets[-1] else np.zeros((0, 2))
    else:
        stacked = np.zeros((0, 2))
    return offsets, np.ascontiguousarray(stacked[:, 0]), np.ascontiguousarray(stacked[:, 1])


# ------------------------------------------------------------------ CSR API

def run_ransac_csr(offsets, azimuth, doppler, params: RansacParams,
                   rng_cluster_index=None) -> RansacResult:
    """rvk_run_ransac: bit-exact run_ransac over a CSR frame."""
    offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
    n = offsets.size - 1
    cnt = np.zeros(n, np.int32)
    tr = np.zeros(n, np.int32)
    mask = np.zeros(azimuth.size, np.uint8)
    keys = _opt_i32(rng_cluster_index, n)
    p = params.c()
    _check(N.gpu().rvk_run_ransac(n, N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler), C.addressof(p),
                                  N.ptr(keys), 0, N.ptr(cnt), N.ptr(tr), N.ptr(mask)))
    return RansacResult(cnt, tr, mask)


def ransac_estimate_csr(offsets, azimuth, doppler, params: RansacParams, frame_id: int = 0,
                        cluster_ids=None, rng_cluster_index=None, packed_mask: bool = False):
    """rvk_ransac_estimate: run_ransac + estimate_all in one device pass.
    packed_mask: the mask comes back as bits (rvk_ransac_estimate_packed,
    uint8 [ceil(P/8)], numpy.packbits(mask, bitorder="little"))."""
    offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
    n = offsets.size - 1
    cnt = np.zeros(n, np.int32)
    tr = np.zeros(n, np.int32)
    mask = np.zeros((azimuth.size + 7) // 8 if packed_mask else azimuth.size, np.uint8)
    est = np.zeros(n, N.ESTIMATE_DTYPE)
    ids = _opt_i32(cluster_ids, n)
    keys = _opt_i32(rng_cluster_index, n)
    p = params.c()
    fn = N.gpu().rvk_ransac_estimate_packed if packed_mask else N.gpu().rvk_ransac_estimate
    _check(fn(frame_id, n, N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler), N.ptr(ids),
              C.addressof(p), N.ptr(keys), N.ptr(cnt), N.ptr(tr), N.ptr(mask), N.ptr(est)))
    return RansacResult(cnt, tr, mask), est


def ransac_estimate_multi_csr(offsets, azimuth, doppler, params: RansacParams, devices,
                              frame_id: int = 0, cluster_ids=None, rng_cluster_index=None):
    """rvk_ransac_estimate_multi: one frame's clusters split over `devices`
    (CUDA ordinals, may repeat), byte-identical to ransac_estimate_csr."""
    offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
    n = offsets.size - 1
    cnt = np.zeros(n, np.int32)
    tr = np.zeros(n, np.int32)
    mask = np.zeros(azimuth.size, np.uint8)
    est = np.zeros(n, N.ESTIMATE_DTYPE)
    ids = _opt_i32(cluster_ids, n)
    keys = _opt_i32(rng_cluster_index, n)
    devs = np.ascontiguousarray(devices, np.int32)
    p = params.c()
    _check(N.gpu().rvk_ransac_estimate_multi(devs.size, N.ptr(devs), frame_id, n, N.ptr(offsets),
                                             N.ptr(azimuth), N.ptr(doppler), N.ptr(ids),
                                             C.addressof(p), N.ptr(keys), N.ptr(cnt), N.ptr(tr),
                                             N.ptr(mask), N.ptr(est)))
    return RansacResult(cnt, tr, mask), est


def estimate_all_csr(offsets, azimuth, doppler, mask, frame_id: int = 0, cluster_ids=None):
    """rvk_estimate_all: LSQ refit + heading for caller masks (uint8 [P])."""
    offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
    n = offsets.size - 1
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    if mask.size != azimuth.size:
        raise ValueError("estimate_all: mask size does not match cluster size")
    est = np.zeros(n, N.ESTIMATE_DTYPE)
    ids = _opt_i32(cluster_ids, n)
    _check(N.gpu().rvk_estimate_all(frame_id, n, N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler),
                                    N.ptr(ids), N.ptr(mask), 0, N.ptr(est)))
    return est


def trial_counts_csr(offsets, azimuth, doppler, params: RansacParams, rng_cluster_index=None):
    """Exact per-(cluster, trial) counts, [C, max_trials] (src/ransac.cpp:163-174)."""
    offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
    n = offsets.size - 1
    out = np.zeros(n * params.max_trials, np.int32)
    keys = _opt_i32(rng_cluster_index, n)
    p = params.c()
    _check(N.gpu().rvk_trial_counts(n, N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler),
                                    C.addressof(p), N.ptr(keys), N.ptr(out)))
    return out.reshape(n, params.max_trials)


def seed_pairs_csr(offsets, params: RansacParams, rng_cluster_index=None):
    """Device-drawn seed pairs, [C, max_trials, 2]."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    n = offsets.size - 1
    out = np.zeros(2 * n * params.max_trials, np.int32)
    keys = _opt_i32(rng_cluster_index, n)
    p = params.c()
    _check(N.gpu().rvk_seed_pairs(n, N.ptr(offsets), C.addressof(p), N.ptr(keys), N.ptr(out)))
    return out.reshape(n, params.max_trials, 2)


def cluster_thresholds_csr(offsets, azimuth, doppler, threshold_scale: float = 1.0):
    """(norm[C, 4] = offset_az, offset_dop, scale_az, scale_dop ; threshold[C])."""
    offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
    n = offsets.size - 1
    norm = np.zeros(4 * n)
    thr = np.zeros(n)
    _check(N.gpu().rvk_cluster_thresholds(n, N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler),
                                          float(threshold_scale), N.ptr(norm), N.ptr(thr)))
    return norm.reshape(n, 4), thr


def ransac_estimate_device(offsets, azimuth, doppler, params: RansacParams, out, stream=None,
                           frame_id: int = 0, cluster_ids=None, rng_cluster_index=None):
    """rvk_ransac_estimate_device on torch CUDA tensors (async on `stream`).

    out: dict with int32 'inlier_count'[C], 'winning_trial'[C], uint8 'mask'[P]
    and uint8 'est'[C*48] (rvk_estimate records) device tensors.
    """
    n = int(offsets.numel()) - 1
    p = params.c()
    s = None if stream is None else C.c_void_p(stream.cuda_stream)
    _check(N.gpu().rvk_ransac_estimate_device(
        frame_id, n, int(azimuth.numel()), N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler),
        N.ptr(cluster_ids), C.addressof(p), N.ptr(rng_cluster_index), N.ptr(out["inlier_count"]),
        N.ptr(out["winning_trial"]), N.ptr(out["mask"]), N.ptr(out["est"]), s))


class FrameStream:
    """rvk_stream_*: the reference's per-frame loop (tools/rvk_main.cpp:125-149)
    pipelined on the device, up to `depth` frames in flight.

    ``submit`` enqueues one CSR frame (or a batch of frames with frame-local
    ``rng_cluster_index``) and returns a ticket; ``result(ticket)`` waits and
    returns ``(RansacResult, estimates)``. Arrays handed to ``submit`` are kept
    alive by the stream until their ticket completes; pass pinned arrays
    (``pinned_empty``) to let the copy engines read/write them directly.
    """

    def __init__(self, params: RansacParams, depth: int = 3):
        self._lib = N.gpu()
        self._p = params.c()
        h = C.c_void_p()
        _check(self._lib.rvk_stream_create(C.addressof(self._p), int(depth), C.byref(h)))
        self._h = h
        self._inputs = {}
        self._outs = {}

    def submit(self, offsets, azimuth, doppler, frame_id: int = 0, cluster_ids=None,
               rng_cluster_index=None, out=None, packed_mask: bool = False) -> int:
        """packed_mask: the mask is delivered as bits (rvk_stream_submit_packed);
        `out`'s mask array then holds ceil(P/8) bytes."""
        offsets, azimuth, doppler = _csr(offsets, azimuth, doppler)
        n = offsets.size - 1
        if out is None:
            P = int(offsets[-1])
            out = (np.zeros(n, np.int32), np.zeros(n, np.int32),
                   np.zeros((P + 7) // 8 if packed_mask else P, np.uint8),
                   np.zeros(n, N.ESTIMATE_DTYPE))
        cnt, tr, mask, est = out
        ids = _opt_i32(cluster_ids, n)
        keys = _opt_i32(rng_cluster_index, n)
        t = C.c_int64(-1)
        fn = self._lib.rvk_stream_submit_packed if packed_mask else self._lib.rvk_stream_submit
        _check(fn(self._h, frame_id, n, N.ptr(offsets), N.ptr(azimuth), N.ptr(doppler),
                  N.ptr(ids), N.ptr(keys), N.ptr(cnt), N.ptr(tr), N.ptr(mask), N.ptr(est),
                  C.byref(t)))
        self._inputs[t.value] = (offsets, azimuth, doppler, ids, keys)
        self._outs[t.value] = out
        # tickets >= depth (<= 8) behind are complete: their inputs are free
        for k in [k for k in self._inputs if k < t.value - 8]:
            del self._inputs[k]
        return t.value

    def wait(self, ticket: int) -> None:
        _check(self._lib.rvk_stream_wait(self._h, int(ticket)))

    def result(self, ticket: int):
        self.wait(ticket)
        self._inputs.pop(ticket, None)
        cnt, tr, mask, est = self._outs.pop(ticket)
        return RansacResult(cnt, tr, mask), est

    def close(self) -> None:
        if self._h:
            st = self._lib.rvk_stream_destroy(self._h)
            self._h = None
            self._inputs.clear()
            _check(st)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            if self._h:
                self._lib.rvk_stream_destroy(self._h)
        except Exception:  # noqa: BLE001
            pass


def estimates_from_records(rec: np.ndarray):
    return [VelocityEstimate(int(r["frame_id"]), int(r["cluster_id"]), float(r["v_x"]),
                             float(r["v_y"]), float(r["heading"]) if r["has_heading"] else None,
                             int(r["inlier_count"]), bool(r["condition_ok"])) for r in rec]


# ------------------------------------------------------- reference-shaped API

def run_ransac(clusters: Sequence[np.ndarray], params: RansacParams = RansacParams(),
               workers: int = 0):
    """rvk::run_ransac (src/ransac.cpp:138-199). clusters: list of (n, 2)
    [azimuth, doppler] arrays. Returns one InlierMask per cluster, cluster_id
    = position. `workers` is accepted and ignored (the device grid replaces
    the thread team)."""
    del workers
    offsets, az, dop = clusters_to_csr(clusters)
    r = run_ransac_csr(offsets, az, dop, params)
    out = []
    for c in range(len(clusters)):
        m = r.mask[offsets[c]:offsets[c + 1]].astype(bool)
        out.append(InlierMask(c, m, int(r.inlier_count[c]), int(r.winning_trial[c])))
    return out


def gather_cluster_points(frame: Frame, clusters: Sequence[Cluster]):
    """rvk::gather_cluster_points (src/ransac.cpp:201-215)."""
    return [np.stack([frame.azimuth[np.asarray(cl.point_indices, dtype=np.int64)],
                      frame.doppler[np.asarray(cl.point_indices, dtype=np.int64)]], axis=1)
            for cl in clusters]


def estimate_all(frame: Frame, clusters: Sequence[Cluster], masks: Sequence[InlierMask],
                 workers: int = 0):
    """rvk::estimate_all (src/velocity.cpp:92-121)."""
    del workers
    if len(clusters) != len(masks):
        raise ValueError("estimate_all: one mask per cluster required")
    for cl, m in zip(clusters, masks):
        if len(m.mask) != len(cl.point_indices):
            raise ValueError("estimate_all: mask size does not match cluster size")
    pts = gather_cluster_points(frame, clusters)
    offsets, az, dop = clusters_to_csr(pts)
    mask = np.concatenate([np.asarray(m.mask, dtype=np.uint8) for m in masks]) if masks else \
        np.zeros(0, np.uint8)
    ids = np.array([cl.cluster_id for cl in clusters], dtype=np.int32)
    rec = estimate_all_csr(offsets, az, dop, mask, frame.frame_id, ids)
    return estimates_from_records(rec)


def draw_seed_pair(seed: int, cluster_id: int, trial: int, n: int):
    """rvk::draw_seed_pair (src/ransac.cpp:111-123), drawn on the device."""
    if n < 2:
        raise ValueError("draw_seed_pair: need at least 2 points")
    # Build a cluster of n points keyed `cluster_id`; trials 0..trial.
    offsets = np.array([0, n], np.int64)
    pairs = seed_pairs_csr(offsets, RansacParams(trial + 1, 1.0, seed),
                           rng_cluster_index=np.array([cluster_id], np.int32))
    i, j = pairs[0, trial]
    return int(i), int(j)


# ------------------------------------------------------------- clustering

def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ValueError("point arrays must have the same length")
    return a


def dbscan_points(x, y, z=None, params: ClusteringParams = ClusteringParams()) -> np.ndarray:
    """rvk_dbscan on SoA coordinates -> labels (int32, -1 = noise)."""
    x = _f64(x)
    y = _f64(y, x.size)
    z = None if z is None else _f64(z, x.size)
    labels = np.zeros(x.size, np.int32)
    p = params.c()
    _check(N.gpu().rvk_dbscan(x.size, N.ptr(x), N.ptr(y), N.ptr(z), C.addressof(p),
                              N.ptr(labels)))
    return labels


def extract_clusters_labels(labels, min_cluster_size: int = 3):
    """rvk_extract_clusters -> (labels rewritten, offsets[m+1], point_indices)."""
    labels = np.array(labels, dtype=np.int32)
    n = labels.size
    offsets = np.zeros(n + 2, np.int64)
    pi = np.zeros(max(n, 1), np.int32)
    m = C.c_int32(0)
    _check(N.gpu().rvk_extract_clusters(n, N.ptr(labels), int(min_cluster_size), C.byref(m),
                                        N.ptr(offsets), N.ptr(pi)))
    off = offsets[:m.value + 1].copy()
    return labels, off, pi[:int(off[-1])].copy()


def dbscan(frame: Frame, params: ClusteringParams = ClusteringParams()) -> None:
    """rvk::dbscan (src/clustering.cpp:24-114): fills frame.labels."""
    z = frame.z if params.features == "xyz" else None
    frame.labels = dbscan_points(frame.x, frame.y, z, params)


def extract_clusters(frame: Frame, min_cluster_size: int = 3):
    """rvk::extract_clusters (src/clustering.cpp:116-155): rewrites
    frame.labels and returns the surviving clusters (ascending members)."""
    if len(frame.labels) != len(frame.x):
        raise ValueError("extract_clusters: frame labels missing; run dbscan first")
    labels, off, pi = extract_clusters_labels(frame.labels, min_cluster_size)
    frame.labels = labels
    return [Cluster(c, pi[off[c]:off[c + 1]].copy()) for c in range(off.size - 1)]


def estimate_frame(frame: Frame, cparams: ClusteringParams = ClusteringParams(),
                   rparams: RansacParams = RansacParams(), min_cluster_size: int = 3):
    """One frame of run_estimate (tools/rvk_main.cpp:128-141) on the device:
    dbscan -> extract_clusters -> gather -> run_ransac -> estimate_all.
    Returns (labels, offsets, point_indices, RansacResult, estimates)."""
    x = _f64(frame.x)
    n = x.size
    y, dop, az = _f64(frame.y, n), _f64(frame.doppler, n), _f64(frame.azimuth, n)
    z = _f64(frame.z, n) if cparams.features == "xyz" else None
    cap = n // max(1, int(min_cluster_size)) + 1
    labels = np.zeros(n, np.int32)
    offsets = np.zeros(n + 2, np.int64)
    pi = np.zeros(max(n, 1), np.int32)
    cnt = np.zeros(cap, np.int32)
    tr = np.zeros(cap, np.int32)
    mask = np.zeros(max(n, 1), np.uint8)
    est = np.zeros(cap, N.ESTIMATE_DTYPE)
    m = C.c_int32(0)
    cp, rp = cparams.c(), rparams.c()
    _check(N.gpu().rvk_estimate_frame(
        int(frame.frame_id), n, N.ptr(x), N.ptr(y), N.ptr(z), N.ptr(dop), N.ptr(az),
        C.addressof(cp), int(min_cluster_size), C.addressof(rp), N.ptr(labels), C.byref(m),
        N.ptr(offsets), N.ptr(pi), N.ptr(cnt), N.ptr(tr), N.ptr(mask), N.ptr(est)))
    k = m.value
    off = offsets[:k + 1].copy()
    P = int(off[-1])
    frame.labels = labels
    return (labels, off, pi[:P].copy(), RansacResult(cnt[:k].copy(), tr[:k].copy(),
                                                     mask[:P].copy()), est[:k].copy())


def combine_masks_labels(labels, mask_ids, mask_offsets, masks) -> np.ndarray:
    """rvk_combine_masks: frame labels + CSR masks -> uint8 [n]."""
    labels = np.ascontiguousarray(labels, np.int32)
    ids = np.ascontiguousarray(mask_ids, np.int32)
    off = np.ascontiguousarray(mask_offsets, np.int64)
    m = np.ascontiguousarray(masks, np.uint8)
    if off.size != ids.size + 1:
        raise ValueError("combine_masks: mask_offsets must have n_masks + 1 entries")
    out = np.zeros(labels.size, np.uint8)
    _check(N.gpu().rvk_combine_masks(labels.size, N.ptr(labels), ids.size, N.ptr(ids),
                                     N.ptr(off), N.ptr(m), N.ptr(out)))
    return out


def combine_masks(frame: Frame, masks: Sequence[InlierMask]) -> np.ndarray:
    """rvk::combine_masks (src/ransac.cpp:217-242) -> bool [n points]."""
    n = len(frame.x) if len(frame.x) else len(frame.azimuth)
    if not masks or len(frame.labels) != n:
        return np.zeros(n, bool)
    ids = np.array([m.cluster_id for m in masks], np.int32)
    sizes = np.array([len(m.mask) for m in masks], np.int64)
    off = np.zeros(len(masks) + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    flat = np.concatenate([np.asarray(m.mask, np.uint8) for m in masks]) if off[-1] else \
        np.zeros(0, np.uint8)
    return combine_masks_labels(frame.labels, ids, off, flat).astype(bool)
