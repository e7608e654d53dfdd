"""GPU parity on the exact calls bench.py times, every cluster.

For BASELINE configs 1-4 (config 4 at T=256 and T=1024) the first step of the
bench -- 16 frames batched into ONE rvk_ransac_estimate_device call with
frame-local RNG keys (bench.batch, bench.py step()) -- is compared with the
unmodified reference (oracle/_ref: rvk::run_ransac + estimate_all with all
host threads, src/ransac.cpp:138-199, src/velocity.cpp:92-121) run frame by
frame, the C3 pattern of tests/acceptance_test.cpp:257-330 (and the first 16
frames of the config-5 stream batched the same way): for EVERY cluster
the inlier count, winning trial and mask bit-exact, the estimates within the
north_star tolerance (assert_estimates_close). No sampling budget.
"""
import os

import numpy as np
import pytest

from conftest import assert_estimates_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,T", [(1, 0), (2, 0), (3, 0), (4, 256), (4, 1024), (5, 0)],
                         ids=["config1", "config2", "config3", "config4_T256", "config4_T1024",
                              "config5_stream_frames"])
def test_bench_batches_every_cluster_vs_reference(gpu_lib, reference, cfg, T):
    import torch

    import bench
    import paper_2012_12618_b200 as rvk
    from oracle.binding import make_params
    from paper_2012_12618_b200 import _native

    if cfg == 5:  # the stream's frames (tools/stream_bench.make_pool: seed = index)
        from tools import workloads as W
        frames = [W.stream_frame(i) for i in range(16)]
    else:
        frames = bench.make_frames(cfg, range(16), T)  # rank 0's first step
    off, az, dop, keys = bench.batch(frames)
    w0 = frames[0]
    p = rvk.RansacParams(w0.max_trials, w0.threshold_scale, w0.rng_seed)
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(v).to(dev) for k, v in
         (("off", off), ("az", az), ("dop", dop), ("keys", keys))}
    Cn, Pn = off.size - 1, int(off[-1])
    o = {"inlier_count": torch.zeros(Cn, dtype=torch.int32, device=dev),
         "winning_trial": torch.zeros(Cn, dtype=torch.int32, device=dev),
         "mask": torch.zeros(Pn, dtype=torch.uint8, device=dev),
         "est": torch.zeros(Cn * 48, dtype=torch.uint8, device=dev)}
    s = torch.cuda.Stream(device=dev)
    rvk.ransac_estimate_device(d["off"], d["az"], d["dop"], p, o, stream=s,
                               rng_cluster_index=d["keys"])
    s.synchronize()
    cnt = o["inlier_count"].cpu().numpy()
    tr = o["winning_trial"].cpu().numpy()
    mask = o["mask"].cpu().numpy()
    est = o["est"].cpu().numpy().view(_native.ESTIMATE_DTYPE)
    mp = make_params(p.max_trials, p.threshold_scale, p.rng_seed)
    workers = os.cpu_count() or 1
    c0 = p0 = 0
    for i, w in enumerate(frames):
        cs = slice(c0, c0 + w.n_clusters)
        ps = slice(p0, p0 + w.n_points)
        r, e = reference.ransac_estimate(w.offsets, w.azimuth, w.doppler, mp, workers=workers,
                                         frame_id=0,
                                         cluster_ids=np.arange(c0, c0 + w.n_clusters,
                                                               dtype=np.int32))
        np.testing.assert_array_equal(cnt[cs], r.inlier_count, err_msg=f"frame {i} counts")
        np.testing.assert_array_equal(tr[cs], r.winning_trial, err_msg=f"frame {i} trials")
        np.testing.assert_array_equal(mask[ps], r.mask, err_msg=f"frame {i} masks")
        assert_estimates_close(est[cs], e, label=f"config {cfg} frame {i}",
                               frame=(w.offsets, w.azimuth, r.mask))
        c0 += w.n_clusters
        p0 += w.n_points
    assert c0 == Cn and p0 == Pn
