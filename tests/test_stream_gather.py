"""Config 5 (BASELINE configs[4]): the sharded frame stream with the host
gather (tools/stream_bench.py). The store gathered from N GPU threads is
byte-identical to N = 1 (frame-local RNG keys, canonical refit order), and
every frame equals a standalone rvk_ransac_estimate_packed call. On a 1-GPU
box the 2- and 3-thread runs share the device (functional check of the
sharding and the gather)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_stream_gather_independent_of_gpu_count(gpu_lib):
    import paper_2012_12618_b200 as rvk
    from tools import stream_bench as SB
    frames = SB.make_pool(5, max_trials=256)
    F = 23
    s1, _, c1 = SB.run_stream(1, frames, F)
    s2, _, c2 = SB.run_stream(2, frames, F)
    s3, _, c3 = SB.run_stream(3, frames, F, depth=2)
    assert sum(c1) == sum(c2) == sum(c3) == F and c2 == [12, 11]
    assert s1.digest() == s2.digest() == s3.digest()
    w0 = frames[0]
    p = rvk.RansacParams(w0.max_trials, w0.threshold_scale, w0.rng_seed)
    for f in (0, 7, 22):
        w = frames[f % len(frames)]
        r, e = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p, frame_id=f,
                                       packed_mask=True)
        cnt, tr, bits, est = s2.slices(f)
        np.testing.assert_array_equal(cnt, r.inlier_count)
        np.testing.assert_array_equal(tr, r.winning_trial)
        np.testing.assert_array_equal(bits, r.mask)
        assert est.tobytes() == e.tobytes()
