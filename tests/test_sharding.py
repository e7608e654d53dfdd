"""Frame-stream sharding and the host gather (paper_2012_12618_b200/stream.py).

CPU tests run the N>1 path with world_size-2 gloo process groups; the
estimator is injected (the C oracle) so the sharding, batching with
frame-local RNG keys and the gather are checked without a GPU: a stream
split over 2 ranks and gathered on rank 0 must equal the 1-rank result
byte for byte. The GPU test checks the same invariance through the sm_100a
pipeline.
"""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_12618_b200 import stream as S
from tools import workloads as W


def _frames(n):
    rng = np.random.default_rng(2024)
    out = []
    for _ in range(n):
        off, az, dop = W.random_clusters(rng, int(rng.integers(1, 5)), lo=5, hi=60)
        out.append(W.Workload("r", off, az, dop, np.zeros(az.size, np.int32),
                              np.zeros((off.size - 1, 2)), 48))
    return out


def _oracle_estimator(params):
    from oracle.binding import Oracle, make_params
    o = Oracle()
    p = make_params(params.max_trials, params.threshold_scale, params.rng_seed)

    def run(offsets, az, dop, keys):
        r = o.sequential_ransac(offsets, az, dop, p, key=keys)
        est = o.estimate_all(offsets, az, dop, r.mask)
        return r.inlier_count, r.winning_trial, r.mask, est
    return run


def _params():
    import paper_2012_12618_b200 as rvk
    return rvk.RansacParams(48, 1.0, 99)


def _same(a, b):
    assert [r.frame for r in a] == [r.frame for r in b]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.inlier_count, y.inlier_count)
        np.testing.assert_array_equal(x.winning_trial, y.winning_trial)
        np.testing.assert_array_equal(x.mask, y.mask)
        assert x.estimates.tobytes() == y.estimates.tobytes()


def test_shard_is_a_balanced_partition():
    for n, world in [(10, 1), (10, 2), (10_000, 8), (3, 4)]:
        parts = [S.shard(n, world, r) for r in range(world)]
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(n))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        S.shard(4, 2, 2)


def test_batching_keeps_frame_local_rng_keys(oracle):
    frames = _frames(7)
    p = _params()
    est = _oracle_estimator(p)
    one = S.estimate_stream(frames, p, batch=1, estimator=est)
    many = S.estimate_stream(frames, p, batch=5, estimator=est)
    _same(one, many)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = _frames(n_frames)
        mine = S.shard(n_frames, world, rank)
        p = _params()
        res = S.estimate_stream([frames[i] for i in mine], p, frame_ids=mine, batch=3,
                                estimator=_oracle_estimator(p))
        gathered = S.gather_to_root(res)
        if rank == 0:
            with open(out_path, "wb") as f:
                pickle.dump(gathered, f)
        else:
            assert gathered is None
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_stream_equals_one_rank(oracle):
    n = 9
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "gathered.pkl")
        mp.start_processes(_worker, args=(2, _free_port(), n, path), nprocs=2,
                           start_method="spawn")
        with open(path, "rb") as f:
            gathered = pickle.load(f)
    p = _params()
    single = S.estimate_stream(_frames(n), p, batch=4, estimator=_oracle_estimator(p))
    _same(gathered, single)


@pytest.mark.gpu
def test_device_stream_matches_per_frame_calls(gpu_lib):
    import paper_2012_12618_b200 as rvk
    frames = [W.automotive(seed=50 + i, n_clusters=20) for i in range(5)]
    p = rvk.RansacParams(1024, 1.0, 3)
    res = S.estimate_stream(frames, p, batch=3)
    for r, w in zip(res, frames):
        one, est = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
        np.testing.assert_array_equal(r.mask, one.mask)
        np.testing.assert_array_equal(r.winning_trial, one.winning_trial)
        for f in ("v_x", "v_y", "heading", "inlier_count", "condition_ok"):
            np.testing.assert_array_equal(r.estimates[f], est[f])


def test_result_image_round_trip():
    """pack_results / unpack_results (the gather's wire format): every field
    back bit for bit, masks through the 1-bit packing, empty frames too."""
    from paper_2012_12618_b200 import _native
    rng = np.random.default_rng(2)
    res = []
    for f, (C_, P_) in enumerate([(3, 17), (0, 0), (5, 64), (1, 3)]):
        est = np.zeros(C_, _native.ESTIMATE_DTYPE)
        est["v_x"] = rng.normal(size=C_)
        est["cluster_id"] = np.arange(C_)
        res.append(S.FrameResult(10 + f, rng.integers(0, 99, C_).astype(np.int32),
                                 rng.integers(0, 99, C_).astype(np.int32),
                                 (rng.uniform(size=P_) < 0.5).astype(np.uint8), est))
    back = S.unpack_results(S.pack_results(res))
    assert len(back) == len(res)
    for a, b in zip(res, back):
        assert a.frame == b.frame
        np.testing.assert_array_equal(a.inlier_count, b.inlier_count)
        np.testing.assert_array_equal(a.winning_trial, b.winning_trial)
        np.testing.assert_array_equal(a.mask, b.mask)
        assert a.estimates.tobytes() == b.estimates.tobytes()
