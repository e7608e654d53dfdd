"""Frame streams sharded over GPUs (BASELINE configs[4]: a stream of frames
over 1/2/4/8 B200, results gathered to the host).

The reference processes frames one after another on one host
(tools/rvk_main.cpp:125-149: for each frame, run_ransac then estimate_all).
Frames are independent and the RNG is keyed on the frame-local cluster index
(src/ransac.cpp:169), so the stream shards with no data-path collective:

* ``shard(n, world, rank)``     -- which frames a rank owns (round-robin).
* ``batch_frames(frames)``      -- concatenates frames into one CSR call; the
  per-cluster RNG key stays frame-local, so results are byte-identical to
  per-frame calls (the reference's worker-count invariance,
  include/rvk/ransac.hpp:124-125).
* ``estimate_stream(frames, params)`` -- this rank's frames through the
  device pipeline in batches: a ``FrameStream`` (rvk_stream_*) keeps up to
  ``depth`` batches in flight, so the H2D of batch k+1 overlaps the kernels
  of batch k.
* ``gather_to_root(results)``   -- the only cross-rank step: a host gather of
  the per-frame results to rank 0, in frame order; each rank sends one flat
  byte image (fixed-layout arrays, masks bit-packed; no pickling) through
  ``torch.distributed.gather`` (gloo: host tensors; NCCL: device tensors).
  Single-process multi-GPU streams gather into one pinned frame-indexed store
  instead (tools/stream_bench.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np


@dataclass
class FrameResult:
    """Per-frame output of run_ransac + estimate_all."""

    frame: int                 # global frame index in the stream
    inlier_count: np.ndarray   # int32 [C]
    winning_trial: np.ndarray  # int32 [C]
    mask: np.ndarray           # uint8 [P]
    estimates: np.ndarray      # rvk_estimate records [C]


def shard(n_frames: int, world: int, rank: int) -> List[int]:
    """Frames owned by `rank`: round-robin, so per-rank work stays balanced
    for a stream of statistically identical frames."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: need 0 <= rank < world")
    return list(range(rank, n_frames, world))


def batch_frames(frames: Sequence) -> tuple:
    """(offsets, azimuth, doppler, rng_keys, cluster_ranges, point_ranges)
    for a list of CSR frames (objects with offsets/azimuth/doppler)."""
    offs = [np.zeros(1, np.int64)]
    az, dop, keys, cr, pr = [], [], [], [], []
    base = 0
    c0 = 0
    for w in frames:
        n = int(w.offsets.size - 1)
        p = int(w.offsets[-1])
        offs.append(np.asarray(w.offsets[1:], np.int64) + base)
        az.append(np.asarray(w.azimuth, np.float64))
        dop.append(np.asarray(w.doppler, np.float64))
        keys.append(np.arange(n, dtype=np.int32))
        cr.append((c0, c0 + n))
        pr.append((base, base + p))
        base += p
        c0 += n
    return (np.concatenate(offs), np.concatenate(az) if az else np.zeros(0),
            np.concatenate(dop) if dop else np.zeros(0),
            np.concatenate(keys) if keys else np.zeros(0, np.int32), cr, pr)


def _device_estimator(params):
    from . import api

    def run(offsets, azimuth, doppler, keys):
        r, est = api.ransac_estimate_csr(offsets, azimuth, doppler, params,
                                         rng_cluster_index=keys)
        return r.inlier_count, r.winning_trial, r.mask, est
    return run


def estimate_stream(frames: Sequence, params, frame_ids: Optional[Sequence[int]] = None,
                    batch: int = 8, estimator: Optional[Callable] = None,
                    depth: int = 3) -> List[FrameResult]:
    """run_ransac + estimate_all for each frame, `batch` frames per device
    call, `depth` calls in flight. `estimator(offsets, az, dop, keys) ->
    (count, trial, mask, est)` replaces the sm_100a pipeline (tests inject
    the CPU oracle)."""
    ids = list(frame_ids) if frame_ids is not None else list(range(len(frames)))
    out: List[FrameResult] = []
    batches = []
    for b0 in range(0, len(frames), batch):
        batches.append((b0, batch_frames(frames[b0:b0 + batch])))
    if estimator is not None:
        results = [estimator(off, az, dop, keys) for _, (off, az, dop, keys, _, _) in batches]
    else:
        from .api import FrameStream
        results = []
        with FrameStream(params, depth=depth) as fs:
            tickets = [fs.submit(off, az, dop, rng_cluster_index=keys)
                       for _, (off, az, dop, keys, _, _) in batches]
            for t in tickets:
                r, est = fs.result(t)
                results.append((r.inlier_count, r.winning_trial, r.mask, est))
    for (b0, (_, _, _, _, cr, pr)), (cnt, tr, mask, est) in zip(batches, results):
        for k, ((ca, cb), (pa, pb)) in enumerate(zip(cr, pr)):
            e = est[ca:cb].copy()
            e["frame_id"] = ids[b0 + k]
            e["cluster_id"] = np.arange(cb - ca, dtype=np.int32)
            out.append(FrameResult(ids[b0 + k], cnt[ca:cb].copy(), tr[ca:cb].copy(),
                                   mask[pa:pb].copy(), e))
    return out


_HDR = np.dtype([("frame", "<i8"), ("C", "<i4"), ("P", "<i4")])


def pack_results(results: List[FrameResult]) -> np.ndarray:
    """Flat uint8 image of a rank's results (no pickling): [n][headers]
    [counts][trials][estimates][masks, 1 bit per point]."""
    from ._native import ESTIMATE_DTYPE
    hdr = np.zeros(len(results), _HDR)
    for k, r in enumerate(results):
        hdr[k] = (r.frame, r.inlier_count.size, r.mask.size)
    parts = [np.array([len(results)], "<i8").view(np.uint8), hdr.view(np.uint8)]
    parts += [np.ascontiguousarray(r.inlier_count, "<i4").view(np.uint8) for r in results]
    parts += [np.ascontiguousarray(r.winning_trial, "<i4").view(np.uint8) for r in results]
    parts += [np.ascontiguousarray(r.estimates, ESTIMATE_DTYPE).view(np.uint8) for r in results]
    parts += [np.packbits(np.asarray(r.mask, np.uint8) != 0, bitorder="little") for r in results]
    return np.concatenate(parts) if parts else np.zeros(0, np.uint8)


def unpack_results(buf: np.ndarray) -> List[FrameResult]:
    from ._native import ESTIMATE_DTYPE
    n = int(buf[:8].view("<i8")[0])
    pos = 8
    hdr = buf[pos:pos + n * _HDR.itemsize].view(_HDR)
    pos += n * _HDR.itemsize

    def take(nbytes):
        nonlocal pos
        a = buf[pos:pos + nbytes]
        pos += nbytes
        return a
    cnt = [take(4 * int(h["C"])).view("<i4").copy() for h in hdr]
    tr = [take(4 * int(h["C"])).view("<i4").copy() for h in hdr]
    est = [take(ESTIMATE_DTYPE.itemsize * int(h["C"])).view(ESTIMATE_DTYPE).copy() for h in hdr]
    masks = [np.unpackbits(take((int(h["P"]) + 7) // 8), count=int(h["P"]),
                           bitorder="little") for h in hdr]
    return [FrameResult(int(h["frame"]), cnt[k], tr[k], masks[k], est[k])
            for k, h in enumerate(hdr)]


def gather_to_root(results: List[FrameResult], group=None) -> Optional[List[FrameResult]]:
    """Host gather of every rank's results to rank 0, ordered by frame index
    (None on the other ranks). Each rank's results travel as one flat byte
    image (pack_results: fixed-layout arrays, masks bit-packed -- no object
    pickling) through torch.distributed.gather: CPU tensors over gloo, device
    tensors over NCCL (NVLink/NVSwitch to GPU 0, then one D2H). Single-process
    runs return the input sorted."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return sorted(results, key=lambda r: r.frame)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    img = pack_results(results)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([img.size], dtype=torch.int64, device=dev), group=group)
    sizes = [int(x.item()) for x in sizes]
    cap = max(sizes)
    mine = torch.zeros(cap, dtype=torch.uint8, device=dev)
    mine[:img.size] = torch.from_numpy(img).to(dev)
    bucket = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(world)] \
        if rank == 0 else None
    dist.gather(mine, bucket, dst=0, group=group)
    if rank != 0:
        return None
    merged = []
    for b, n in zip(bucket, sizes):
        merged += unpack_results(b[:n].cpu().numpy())
    return sorted(merged, key=lambda r: r.frame)
