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
  the per-frame results to rank 0, in frame order (torch.distributed
  ``gather_object``; gloo or NCCL process group).
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


def gather_to_root(results: List[FrameResult], group=None) -> Optional[List[FrameResult]]:
    """Host gather of every rank's results to rank 0, ordered by frame index
    (None on the other ranks). Single-process runs return the input sorted."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return sorted(results, key=lambda r: r.frame)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bucket = [None] * world if rank == 0 else None
    dist.gather_object(results, bucket, dst=0, group=group)
    if rank != 0:
        return None
    merged = [r for part in bucket for r in part]
    return sorted(merged, key=lambda r: r.frame)
