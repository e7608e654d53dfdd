"""GPU parity: the sm_100a path (through the C-ABI) against the oracle and the
reference's golden vectors.

Bar (BASELINE.json north_star): seed pairs, thresholds, per-trial counts,
inlier counts, winning trials and masks bit-exact; v_x, v_y, speed within
1e-4 relative and heading within 1e-3 rad, condition_ok / heading presence
exact (assert_estimates_close).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2012_12618_b200 as rvk
from tools import workloads as W
from conftest import EXTREME_PARAMS, ROOT, assert_estimates_close, extreme_value_clusters
from oracle.binding import make_params

pytestmark = pytest.mark.gpu


def _params(g):
    return rvk.RansacParams(g["max_trials"], g["threshold_scale"], g["seed"])


def _oracle_params(p):
    return make_params(p.max_trials, p.threshold_scale, p.rng_seed)


def test_native_library_is_the_cuda_one(gpu_lib):
    assert gpu_lib.rvk_abi_version() == 1
    gpu_lib.rvk_reset_kernel_launches()
    off = np.array([0, 5], np.int64)
    rvk.run_ransac_csr(off, np.linspace(0, 1, 5), np.linspace(1, 2, 5), rvk.RansacParams(8))
    # the fused warp-per-cluster kernel alone (the host knows every cluster
    # fits), or prep (+ the persistent CTA prep of large clusters), score, select
    assert gpu_lib.rvk_kernel_launches() in (1, 3, 4)


def test_seed_pairs_vs_oracle(gpu_lib, oracle):
    rng = np.random.default_rng(1)
    for _ in range(20):
        k = int(rng.integers(1, 8))
        sizes = rng.choice([2, 3, 5, 64, 100, 2048, 70000], size=k)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        keys = rng.integers(0, 10000, size=k).astype(np.int32)
        p = rvk.RansacParams(int(rng.integers(1, 300)), 1.0, int(rng.integers(0, 2**63)) * 2 + 1)
        got = rvk.seed_pairs_csr(off, p, rng_cluster_index=keys)
        for c in range(k):
            for t in range(0, p.max_trials, 7):
                assert tuple(got[c, t]) == oracle.seed_pair(p.rng_seed, int(keys[c]), t,
                                                            int(sizes[c]))


def test_seed_pairs_golden(gpu_lib, golden_rng):
    ins, outs = golden_rng["seed_pair_in"], golden_rng["seed_pair_out"]
    for (s, c, t, n), want in list(zip(ins, outs))[:300]:
        got = rvk.draw_seed_pair(int(s), int(c), int(t), int(n))
        assert got == tuple(int(v) for v in want)


def test_thresholds_golden(gpu_lib, golden_cases):
    for g in golden_cases:
        norm, thr = rvk.cluster_thresholds_csr(g["offsets"], g["az"], g["dop"],
                                               g["threshold_scale"])
        np.testing.assert_array_equal(norm, g["norm"], err_msg=g["name"])
        np.testing.assert_array_equal(thr, g["threshold"], err_msg=g["name"])


def test_trial_counts_golden(gpu_lib, golden_cases):
    for g in golden_cases:
        got = rvk.trial_counts_csr(g["offsets"], g["az"], g["dop"], _params(g))
        np.testing.assert_array_equal(got, g["trial_counts"], err_msg=g["name"])


def test_ransac_golden(gpu_lib, golden_cases):
    for g in golden_cases:
        r = rvk.run_ransac_csr(g["offsets"], g["az"], g["dop"], _params(g))
        np.testing.assert_array_equal(r.inlier_count, g["inlier_count"], err_msg=g["name"])
        np.testing.assert_array_equal(r.winning_trial, g["winning_trial"], err_msg=g["name"])
        np.testing.assert_array_equal(r.mask, g["mask"], err_msg=g["name"])


def test_ransac_estimate_golden(gpu_lib, golden_cases):
    for g in golden_cases:
        n = g["offsets"].size - 1
        r, est = rvk.ransac_estimate_csr(g["offsets"], g["az"], g["dop"], _params(g),
                                         frame_id=g["frame_id"],
                                         cluster_ids=np.arange(n, dtype=np.int32) + 100)
        np.testing.assert_array_equal(r.mask, g["mask"], err_msg=g["name"])
        fr = (g["offsets"], g["az"], g["mask"])
        assert_estimates_close(est, g["estimates"], label=g["name"], frame=fr)
        # estimate_all on the reference's masks too
        est2 = rvk.estimate_all_csr(g["offsets"], g["az"], g["dop"], g["mask"],
                                    frame_id=g["frame_id"],
                                    cluster_ids=np.arange(n, dtype=np.int32) + 100)
        assert_estimates_close(est2, g["estimates"], label=g["name"] + "/estimate_all", frame=fr)


def test_c3_thousand_random_frames(gpu_lib, oracle):
    """Acceptance C3 (acceptance_test.cpp:257-330) against the GPU: 1000
    frames, 1-4 clusters x 5-40 points, T in [16, 96], random 64-bit seed."""
    rng = np.random.default_rng(303)
    for f in range(1000):
        off, az, dop = W.random_clusters(rng, int(rng.integers(1, 5)))
        p = rvk.RansacParams(int(rng.integers(16, 97)), 1.0, int(rng.integers(0, 2**63)))
        r, est = rvk.ransac_estimate_csr(off, az, dop, p, frame_id=f)
        o = oracle.sequential_ransac(off, az, dop, _oracle_params(p))
        np.testing.assert_array_equal(r.mask, o.mask, err_msg=f"frame {f}")
        np.testing.assert_array_equal(r.winning_trial, o.winning_trial, err_msg=f"frame {f}")
        np.testing.assert_array_equal(r.inlier_count, o.inlier_count, err_msg=f"frame {f}")
        oe = oracle.estimate_all(off, az, dop, o.mask, frame_id=f)
        assert_estimates_close(est, oe, label=f"frame {f}", frame=(off, az, o.mask))


@pytest.mark.parametrize("scale", [1.0, 0.25, 1e-3, 3.0])
def test_radar_frames_all_trial_counts(gpu_lib, oracle, scale):
    """Per-trial counts exact for every trial (not only the verified ones)."""
    w = W.automotive(seed=5, n_clusters=12, max_trials=96, lo_pts=16, hi_pts=400)
    p = rvk.RansacParams(96, scale, 99)
    got = rvk.trial_counts_csr(w.offsets, w.azimuth, w.doppler, p)
    want = oracle.trial_counts(w.offsets, w.azimuth, w.doppler, _oracle_params(p))
    np.testing.assert_array_equal(got, want)
    r = rvk.run_ransac_csr(w.offsets, w.azimuth, w.doppler, p)
    o = oracle.sequential_ransac(w.offsets, w.azimuth, w.doppler, _oracle_params(p))
    np.testing.assert_array_equal(r.mask, o.mask)
    np.testing.assert_array_equal(r.winning_trial, o.winning_trial)


def test_config1_full(gpu_lib, oracle):
    w = W.single_frame()
    p = rvk.RansacParams(w.max_trials, w.threshold_scale, w.rng_seed)
    r, est = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
    o, oe = oracle.ransac_estimate_range(w.offsets, w.azimuth, w.doppler, _oracle_params(p), 0,
                                         w.n_clusters)
    np.testing.assert_array_equal(r.mask, o.mask)
    np.testing.assert_array_equal(r.winning_trial, o.winning_trial)
    np.testing.assert_array_equal(r.inlier_count, o.inlier_count)
    assert_estimates_close(est, oe, frame=(w.offsets, w.azimuth, o.mask))


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_full_size_configs_sampled(gpu_lib, oracle, cfg):
    """Full-size frames on the GPU; the oracle checks a bounded sample of
    clusters (the largest ones and a spread of others) bit-exactly."""
    w = W.CONFIGS[cfg]()
    p = rvk.RansacParams(w.max_trials, w.threshold_scale, w.rng_seed)
    r, est = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
    sizes = np.diff(w.offsets)
    budget = 1.5e8  # oracle evals
    order = np.argsort(-sizes, kind="stable")
    picks = list(order[:2]) + list(range(0, w.n_clusters, max(1, w.n_clusters // 12)))
    done = 0
    for c in sorted(set(int(c) for c in picks)):
        if done + sizes[c] * w.max_trials > budget:
            continue
        done += sizes[c] * w.max_trials
        o, oe = oracle.ransac_estimate_range(w.offsets, w.azimuth, w.doppler,
                                             _oracle_params(p), c, c + 1)
        sl = slice(w.offsets[c], w.offsets[c + 1])
        np.testing.assert_array_equal(r.mask[sl], o.mask[sl], err_msg=f"cfg {cfg} cluster {c}")
        assert r.winning_trial[c] == o.winning_trial[c]
        assert r.inlier_count[c] == o.inlier_count[c]
        assert_estimates_close(est[c:c + 1], oe[c:c + 1], label=f"cfg {cfg} cluster {c}",
                               frame=(w.offsets[c:c + 2] - w.offsets[c], w.azimuth[sl], o.mask[sl]))
    # size-independent properties over every cluster
    per = np.add.reduceat(r.mask.astype(np.int64), w.offsets[:-1])
    np.testing.assert_array_equal(per, r.inlier_count)
    np.testing.assert_array_equal(est["inlier_count"], r.inlier_count)
    assert (r.winning_trial >= 0).all() and (r.winning_trial < w.max_trials).all()
    pairs = rvk.seed_pairs_csr(w.offsets, p)
    idx = np.arange(w.n_clusters)
    a = pairs[idx, r.winning_trial, 0] + w.offsets[:-1]
    b = pairs[idx, r.winning_trial, 1] + w.offsets[:-1]
    assert r.mask[a].all() and r.mask[b].all()  # the winner contains its seeds


def test_batch_composition_invariance(gpu_lib):
    """Splitting a frame into batches with frame-local RNG keys gives
    byte-identical results (the reference's worker-count invariance; both
    halves use the same CTA shapes, so the velocities are byte-identical too)."""
    w = W.imaging(n_clusters=600, total=120_000)
    p = rvk.RansacParams(256, 1.0, 12345)
    full, est = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
    h = w.n_clusters // 3
    for lo, hi in [(0, h), (h, w.n_clusters)]:
        off = w.offsets[lo:hi + 1] - w.offsets[lo]
        sl = slice(w.offsets[lo], w.offsets[hi])
        r, e = rvk.ransac_estimate_csr(off, w.azimuth[sl], w.doppler[sl], p,
                                       rng_cluster_index=np.arange(lo, hi, dtype=np.int32))
        np.testing.assert_array_equal(r.mask, full.mask[sl])
        np.testing.assert_array_equal(r.winning_trial, full.winning_trial[lo:hi])
        for f in ("v_x", "v_y", "heading"):
            np.testing.assert_array_equal(e[f], est[f][lo:hi])


def test_concurrent_host_threads(gpu_lib):
    """The reference's run_ransac may be called from several host threads;
    the C-ABI keeps one context (stream, workspace) per thread: concurrent
    calls on different frames give the sequential results byte for byte."""
    import threading
    frames = [W.automotive(seed=500 + i, n_clusters=60) for i in range(8)]
    p = rvk.RansacParams(512, 1.0, 99)
    want = [rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p) for w in frames]
    got = [None] * len(frames)
    errors = []

    def work(k):
        try:
            for i in range(k, len(frames), 4):
                w = frames[i]
                for _ in range(3):
                    got[i] = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (r0, e0), (r1, e1) in zip(want, got):
        np.testing.assert_array_equal(r0.mask, r1.mask)
        np.testing.assert_array_equal(r0.winning_trial, r1.winning_trial)
        np.testing.assert_array_equal(r0.inlier_count, r1.inlier_count)
        for f in ("v_x", "v_y", "heading"):
            np.testing.assert_array_equal(e0[f], e1[f])


def test_frame_alone_vs_in_batch(gpu_lib):
    """A frame scored alone (a small call: 512-thread prep, 256-thread select,
    small scoring units) and inside a 16-frame batch (512-point units, the
    throughput CTA shapes) gives byte-identical results, velocities included
    (the refit's canonical summation order, RefitAcc)."""
    frames = [W.automotive(seed=900 + i) for i in range(16)]
    p = rvk.RansacParams(1024, 1.0, 4242)
    offs, az, dop, keys = [np.zeros(1, np.int64)], [], [], []
    base = 0
    for w in frames:
        offs.append(w.offsets[1:] + base)
        base += w.n_points
        az.append(w.azimuth)
        dop.append(w.doppler)
        keys.append(np.arange(w.n_clusters, dtype=np.int32))
    r_all, e_all = rvk.ransac_estimate_csr(np.concatenate(offs), np.concatenate(az),
                                           np.concatenate(dop), p,
                                           rng_cluster_index=np.concatenate(keys))
    c0, p0 = 0, 0
    for w in frames:
        r, e = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
        cs, ps = slice(c0, c0 + w.n_clusters), slice(p0, p0 + w.n_points)
        np.testing.assert_array_equal(r.mask, r_all.mask[ps])
        np.testing.assert_array_equal(r.winning_trial, r_all.winning_trial[cs])
        np.testing.assert_array_equal(r.inlier_count, r_all.inlier_count[cs])
        for f in ("v_x", "v_y", "heading", "condition_ok", "has_heading", "inlier_count"):
            np.testing.assert_array_equal(e[f], e_all[f][cs])
        c0 += w.n_clusters
        p0 += w.n_points


_SHAPE_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2012_12618_b200 as rvk
from tools import workloads as W
h = hashlib.sha256()
for w in (W.automotive(seed=77, n_clusters=40), W.imaging(seed=78, n_clusters=300, total=60_000)):
    r, e = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, rvk.RansacParams(512, 1.0, 5))
    m = rvk.estimate_all_csr(w.offsets, w.azimuth, w.doppler, r.mask)
    assert e.tobytes() == m.tobytes(), "select's refit != estimate_all's refit"
    for a in (r.mask, r.winning_trial, r.inlier_count, e.tobytes(), m.tobytes()):
        h.update(np.asarray(a).tobytes() if not isinstance(a, bytes) else a)
print(h.hexdigest())
"""


def test_launch_shapes_bit_identical(gpu_lib):
    """Every launch shape -- CTA or warp select, 64..256-thread CTAs, warp or
    CTA prep, unit sizes -- gives the same bytes for every output, velocities
    included (counts/masks by the exact scheme, velocities by the canonical
    refit order), as the reference's worker-count invariance demands."""
    digests = {}
    ps0 = {"RVK_PREP_SCORE": "0"}
    for env in ({}, dict(ps0, RVK_SELECT_WARP="1"), dict(ps0, RVK_SELECT_WARP="0"),
                dict(ps0, RVK_SELECT_WARP="0", RVK_SELECT_THREADS="64"),
                dict(ps0, RVK_SELECT_WARP="0", RVK_SELECT_THREADS="256"),
                dict(ps0, RVK_PREP_WARP="1"), dict(ps0, RVK_PREP_WARP="0", RVK_PREP_THREADS="512"),
                {"RVK_SCORE_PPT": "64"}, {"RVK_FUSED": "1"}, {"RVK_FUSED": "0"},
                {"RVK_FUSED": "0", "RVK_PREP_SCORE": "1"}, {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0"}):
        r = subprocess.run([sys.executable, "-c", _SHAPE_SCRIPT, ROOT], capture_output=True,
                           text=True, env=dict(os.environ, **env), cwd=ROOT, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests[str(env)] = r.stdout.strip()
    assert len(set(digests.values())) == 1, digests


def test_randomised_sweep(gpu_lib):
    """A short run of tools/fuzz_parity.py (random clustered / uniform /
    quantised / tiny-spread / near-degenerate frames, random T, scale and
    seed): masks, trials, counts bit-exact, estimates within tolerance."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"),
                        "--frames", "400", "--seed", "21"],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert '"mismatches": 0' in r.stdout


def test_randomised_sweep_stress(gpu_lib):
    """The config-3 regime of tools/fuzz_parity.py: T in {2048, 4096},
    threshold_scale 0.25, exactly 50% outliers, 64-2048-point clusters."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"),
                        "--frames", "60", "--seed", "22", "--stress"],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert '"mismatches": 0' in r.stdout


def test_edge_cases(gpu_lib, oracle):
    rng = np.random.default_rng(11)
    cases = []
    # huge cluster (> shared-memory chunk), odd sizes, odd base offsets
    cases.append([rng.uniform(-1, 1, (9001, 2)) * [1, 10]])
    cases.append([rng.uniform(-1, 1, (3, 2)), rng.uniform(-1, 1, (4, 2)),
                  rng.uniform(-1, 1, (4097, 2))])
    # zero spread in azimuth (all degenerate), in doppler (zero MAD)
    cases.append([np.stack([np.full(20, 0.3), rng.uniform(-5, 5, 20)], 1)])
    cases.append([np.stack([rng.uniform(-1, 1, 20), np.full(20, 2.0)], 1)])
    # duplicates + quantized ties
    q = np.round(rng.uniform(-1, 1, (200, 2)) * 4) / 4
    cases.append([q, q[:50].copy()])
    for cl in cases:
        off, az, dop = rvk.clusters_to_csr(cl)
        for T, scale in [(1, 1.0), (513, 1.0), (64, 1e-6), (300, 0.25)]:
            p = rvk.RansacParams(T, scale, 77)
            r = rvk.run_ransac_csr(off, az, dop, p)
            o = oracle.sequential_ransac(off, az, dop, _oracle_params(p))
            np.testing.assert_array_equal(r.mask, o.mask)
            np.testing.assert_array_equal(r.winning_trial, o.winning_trial)
            np.testing.assert_array_equal(r.inlier_count, o.inlier_count)


def test_edge_cases_extreme_values(gpu_lib, oracle):
    """conftest.extreme_value_clusters (three-point clusters, signed zeros,
    FP64-extreme magnitudes, subnormal spreads): every decision bit-exact."""
    for cl in extreme_value_clusters():
        off, az, dop = rvk.clusters_to_csr(cl)
        for T, scale in EXTREME_PARAMS:
            p = rvk.RansacParams(T, scale, 5)
            r, est = rvk.ransac_estimate_csr(off, az, dop, p)
            o = oracle.sequential_ransac(off, az, dop, _oracle_params(p))
            np.testing.assert_array_equal(r.mask, o.mask)
            np.testing.assert_array_equal(r.winning_trial, o.winning_trial)
            np.testing.assert_array_equal(r.inlier_count, o.inlier_count)
            oe = oracle.estimate_all(off, az, dop, o.mask)
            assert_estimates_close(est, oe, label=f"T={T} scale={scale}", frame=(off, az, o.mask))


def test_errors_and_reference_shaped_api(gpu_lib, oracle):
    with pytest.raises(rvk.ClusterTooSmall, match="cluster 0 has 2 points"):
        rvk.run_ransac([np.zeros((2, 2))])
    masks = rvk.run_ransac([np.array([[0.0, 1.0], [0.1, 1.2], [0.2, 1.4], [0.3, 1.6],
                                      [0.4, 1.8]])], rvk.RansacParams(32))
    assert masks[0].inlier_count == 5 and masks[0].winning_trial == 0 and masks[0].mask.all()
    assert rvk.run_ransac([], rvk.RansacParams()) == []


def test_device_api_matches_host_api(gpu_lib):
    import torch
    w = W.automotive(seed=3, n_clusters=50)
    p = rvk.RansacParams(w.max_trials, 1.0, 5)
    r, est = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
    dev = torch.device("cuda")
    off = torch.from_numpy(w.offsets).to(dev)
    az = torch.from_numpy(w.azimuth).to(dev)
    dp = torch.from_numpy(w.doppler).to(dev)
    out = {"inlier_count": torch.zeros(w.n_clusters, dtype=torch.int32, device=dev),
           "winning_trial": torch.zeros(w.n_clusters, dtype=torch.int32, device=dev),
           "mask": torch.zeros(w.n_points, dtype=torch.uint8, device=dev),
           "est": torch.zeros(w.n_clusters * 48, dtype=torch.uint8, device=dev)}
    s = torch.cuda.current_stream()
    rvk.ransac_estimate_device(off, az, dp, p, out, stream=s)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["mask"].cpu().numpy(), r.mask)
    np.testing.assert_array_equal(out["winning_trial"].cpu().numpy(), r.winning_trial)
    e = out["est"].cpu().numpy().view(est.dtype)
    for f in ("v_x", "v_y", "heading", "inlier_count"):
        np.testing.assert_array_equal(e[f], est[f])


def _run_binary(name, extra=()):
    path = os.path.join(ROOT, "oracle", "_ref", name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    out = subprocess.run([path, *extra], capture_output=True, text=True, timeout=900)
    return out.returncode, out.stdout + out.stderr


def test_reference_unit_suites_against_dropin(gpu_lib):
    """The reference's own gtest suites (test_ransac, test_baseline,
    test_velocity, test_clustering, ...) linked against the GPU drop-in
    (run_ransac, estimate_all, dbscan and extract_clusters on the device).

    Excluded: SequentialLsq.ExactlyMatchesParallelEstimates
    (test_baseline.cpp:84-110) asserts that the reference's two CPU LSQ
    engines produce bitwise-equal doubles ("same arithmetic"). The device
    refit reduces in a different order and uses CUDA's sin/cos, so it is held
    to the north_star tolerance instead (test_ransac_estimate_golden,
    test_c3_thousand_random_frames); its discrete outputs must still match."""
    code, log = _run_binary("rvk_dropin_tests",
                            ["--gtest_filter=-SequentialLsq.ExactlyMatchesParallelEstimates"])
    assert code == 0, log[-4000:]


def test_reference_acceptance_against_dropin(gpu_lib):
    """Acceptance C1, C2, C3 (1000 frames), C5-C7 of the reference against the
    GPU drop-in (C7: the reference's brute-force DBSCAN oracle vs rvk::dbscan,
    now the device grid-hash DBSCAN). C4 (CPU thread-scaling trend) is about the CPU engine and is
    excluded."""
    code, log = _run_binary("rvk_dropin_acceptance", ["--gtest_filter=-C4ScalingTrend"])
    assert code == 0, log[-4000:]
    for crit in ("C1", "C2", "C3", "C5", "C6", "C7"):
        assert f"[ACCEPTANCE] {crit}" in log and ": PASS" in log


def test_reference_bench_harness_gpu_arm(gpu_lib, tmp_path):
    """The reference's own bench harness (src/bench.cpp run_bench, compiled
    unmodified) linked against the drop-in: its parallel_* columns time the
    sm_100a path, the sequential_* columns the reference's 1-core CPU
    baselines -- the GPU arm of `rvk bench`."""
    out = tmp_path / "bench.csv"
    code, log = _run_binary("rvk_dropin_bench", ["--grid", "default", "--reps", "5",
                                                 "--warmups", "2", "-o", str(out)])
    assert code == 0, log[-4000:]
    lines = out.read_text().strip().splitlines()
    assert lines[0] == ("n_clusters,points_per_cluster,parallel_ransac_ms,sequential_ransac_ms,"
                        "parallel_lsq_ms,sequential_lsq_ms")
    rows = [list(map(float, ln.split(","))) for ln in lines[1:]]
    assert [(int(r[0]), int(r[1])) for r in rows] == [(c, p) for c in (8, 16, 32, 64)
                                                      for p in (100, 150)]
    assert all(np.isfinite(r[2:]).all() and min(r[2:]) > 0 for r in rows)
    print(log)


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_frame_stream_matches_host_api(gpu_lib, depth):
    """rvk_stream_*: pipelined frames give the same bytes as one-shot calls,
    for pinned and pageable inputs, any depth, waits in any order."""
    import torch
    frames = [W.automotive(seed=70 + i, n_clusters=30) for i in range(7)]
    p = rvk.RansacParams(256, 1.0, 11)
    want = [rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p, frame_id=i)
            for i, w in enumerate(frames)]
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    with rvk.FrameStream(p, depth=depth) as fs:
        tickets = []
        for i, w in enumerate(frames):
            if i % 2:
                az, dop = pin(w.azimuth), pin(w.doppler)
                out = (pin(np.zeros(w.n_clusters, np.int32)), pin(np.zeros(w.n_clusters, np.int32)),
                       pin(np.zeros(w.n_points, np.uint8)), np.zeros(w.n_clusters, est_dtype()))
            else:
                az, dop, out = w.azimuth, w.doppler, None
            tickets.append(fs.submit(w.offsets, az, dop, frame_id=i, out=out))
        assert tickets == list(range(len(frames)))
        order = list(reversed(tickets)) if depth > 1 else tickets
        got = {t: fs.result(t) for t in order}
        fs.wait(tickets[0])  # idempotent
        with pytest.raises(ValueError, match="unknown ticket"):
            fs.wait(len(frames) + 5)
        with pytest.raises(rvk.ClusterTooSmall):
            fs.submit(np.array([0, 2], np.int64), np.zeros(2), np.zeros(2))
    for t, (r, est) in zip(tickets, want):
        g, ge = got[t]
        np.testing.assert_array_equal(g.mask, r.mask)
        np.testing.assert_array_equal(g.winning_trial, r.winning_trial)
        np.testing.assert_array_equal(g.inlier_count, r.inlier_count)
        for f in ("frame_id", "cluster_id", "v_x", "v_y", "heading", "inlier_count",
                  "condition_ok", "has_heading"):
            np.testing.assert_array_equal(ge[f], est[f])


def est_dtype():
    from paper_2012_12618_b200 import _native
    return _native.ESTIMATE_DTYPE


@pytest.mark.parametrize("env", [{"RVK_FUSED": "1"}, {"RVK_FUSED": "0"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "1"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_PREP_THREADS": "256",
                                  "RVK_SELECT_THREADS": "256"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_PREP_THREADS": "64",
                                  "RVK_SELECT_THREADS": "64"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_PREP_WARP": "1"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_PREP_WARP": "0"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_SELECT_WARP": "1"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_SELECT_WARP": "0"},
                                 {"RVK_SCORE_PPT": "64"}, {"RVK_SCORE_PPT": "512"},
                                 {"RVK_FUSED": "0", "RVK_PREP_SCORE": "0", "RVK_PREP_THREADS": "512",
                                  "RVK_PREP_WARP": "0"}],
                         ids=["fused", "unfused", "prep_score", "no_prep_score", "cta256",
                              "cta64", "warp_prep", "cta_prep",
                              "warp_select", "cta_select", "units_64", "units_512",
                              "cta512_prep"])
def test_alternative_kernel_shapes_parity(gpu_lib, env):
    """Every kernel variant must give the same bytes: the fused
    warp-per-cluster kernel forced on/off for every call (normally chosen from
    the mean cluster size; clusters > 512 points then take the CTA path), the
    per-cluster CTA shapes of prep/select, the warp-per-cluster prep and
    select, the scoring unit sizes. The golden, C3 and full-size parity tests
    re-run in a child process with the variant selected (selections are read
    once per process)."""
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         os.path.join(ROOT, "tests", "test_gpu_parity.py"),
         "-k", "golden or c3 or config1 or full_size or edge or batch_composition or radar or "
         "device_api"],
        capture_output=True, text=True, env=dict(os.environ, **env), cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_packed_masks(gpu_lib):
    """rvk_ransac_estimate_packed / rvk_stream_submit_packed:
    the bits are numpy.packbits(mask, bitorder="little") of the byte mask, every
    other output identical; odd point counts, chunked host calls (> 2^18 points)
    and single points past a byte boundary included."""
    cases = [W.single_frame(), W.automotive(seed=3, n_clusters=40),
             W.imaging(seed=5, n_clusters=1500, total=300_001)]
    for w in cases:
        p = rvk.RansacParams(w.max_trials, w.threshold_scale, 3)
        r, e = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
        rb, eb = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p, packed_mask=True)
        assert rb.mask.size == (w.n_points + 7) // 8
        np.testing.assert_array_equal(rb.mask, np.packbits(r.mask, bitorder="little"))
        np.testing.assert_array_equal(rb.inlier_count, r.inlier_count)
        np.testing.assert_array_equal(rb.winning_trial, r.winning_trial)
        assert eb.tobytes() == e.tobytes()
        with rvk.FrameStream(p, depth=2) as fs:
            t1 = fs.submit(w.offsets, w.azimuth, w.doppler, packed_mask=True)
            t2 = fs.submit(w.offsets, w.azimuth, w.doppler)
            rs, es = fs.result(t1)
            rs2, _ = fs.result(t2)
        np.testing.assert_array_equal(rs.mask, rb.mask)
        np.testing.assert_array_equal(rs2.mask, r.mask)
        assert es.tobytes() == e.tobytes()


@pytest.mark.parametrize("env", [{}, {"RVK_FUSED": "1"}, {"RVK_PREP_WARP": "0",
                                                         "RVK_SELECT_WARP": "0"}],
                         ids=["default", "fused", "cta"])
def test_device_api_too_small_clusters(gpu_lib, env):
    """rvk_ransac_estimate_device does no host-side size check: clusters of 0,
    1 and 2 points get the sentinel (count = trial = -1, zero mask, zero
    estimate) and never disturb their neighbours, whose outputs equal the
    host API's on the valid clusters alone (same RNG keys)."""
    r = subprocess.run([sys.executable, "-c", _TOO_SMALL_SCRIPT, ROOT], capture_output=True,
                       text=True, env=dict(os.environ, **env), cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "ok" in r.stdout


_TOO_SMALL_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import paper_2012_12618_b200 as rvk
from paper_2012_12618_b200 import _native
rng = np.random.default_rng(5)
sizes = np.array([40, 1, 0, 300, 2, 7, 600, 2, 3])
off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
P = int(off[-1])
az = rng.uniform(-1, 1, P); dop = rng.uniform(-5, 5, P)
keys = np.arange(sizes.size, dtype=np.int32)
p = rvk.RansacParams(200, 1.0, 9)
dev = torch.device("cuda", 0)
d = {k: torch.from_numpy(v).to(dev) for k, v in (("off", off), ("az", az), ("dop", dop), ("keys", keys))}
C_ = sizes.size
o = {"inlier_count": torch.full((C_,), 77, dtype=torch.int32, device=dev),
     "winning_trial": torch.full((C_,), 77, dtype=torch.int32, device=dev),
     "mask": torch.full((P,), 9, dtype=torch.uint8, device=dev),
     "est": torch.full((C_ * 48,), 7, dtype=torch.uint8, device=dev)}
rvk.ransac_estimate_device(d["off"], d["az"], d["dop"], p, o, rng_cluster_index=d["keys"])
torch.cuda.synchronize()
cnt = o["inlier_count"].cpu().numpy(); tr = o["winning_trial"].cpu().numpy()
mask = o["mask"].cpu().numpy(); est = o["est"].cpu().numpy().view(_native.ESTIMATE_DTYPE)
ok = sizes >= 3
for c in np.nonzero(~ok)[0]:
    assert cnt[c] == -1 and tr[c] == -1, (c, cnt[c], tr[c])
    assert (mask[off[c]:off[c + 1]] == 0).all()
    e = est[c]
    assert e["inlier_count"] == 0 and e["v_x"] == 0 and e["v_y"] == 0
    assert e["has_heading"] == 0 and e["condition_ok"] == 0 and e["cluster_id"] == c
vc = np.nonzero(ok)[0]
voff = np.concatenate([[0], np.cumsum(sizes[vc])]).astype(np.int64)
vaz = np.concatenate([az[off[c]:off[c + 1]] for c in vc])
vdop = np.concatenate([dop[off[c]:off[c + 1]] for c in vc])
r, e = rvk.ransac_estimate_csr(voff, vaz, vdop, p, rng_cluster_index=keys[vc],
                               cluster_ids=vc.astype(np.int32))
np.testing.assert_array_equal(cnt[vc], r.inlier_count)
np.testing.assert_array_equal(tr[vc], r.winning_trial)
np.testing.assert_array_equal(np.concatenate([mask[off[c]:off[c + 1]] for c in vc]), r.mask)
assert est[vc].tobytes() == e.tobytes()
print("ok")
"""


_MIXED_BATCH_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import paper_2012_12618_b200 as rvk
from paper_2012_12618_b200 import _native
from tools import workloads as W
# > 6144 small clusters (the fused prep + score path) with large clusters
# (> 384 and > 508 points: the CTA path) interleaved, T = 300
wi = W.imaging(seed=31, n_clusters=7000, total=1_400_000)
wa = W.automotive(seed=32, n_clusters=30, lo_pts=300, hi_pts=1800)
cl = []
for c in range(wi.n_clusters):
    s = slice(wi.offsets[c], wi.offsets[c + 1])
    cl.append(np.stack([wi.azimuth[s], wi.doppler[s]], 1))
    if c % 250 == 0 and c // 250 < wa.n_clusters:
        a = c // 250
        s2 = slice(wa.offsets[a], wa.offsets[a + 1])
        cl.append(np.stack([wa.azimuth[s2], wa.doppler[s2]], 1))
off, az, dop = rvk.clusters_to_csr(cl)
p = rvk.RansacParams(300, 1.0, 12)
h = hashlib.sha256()
r, e = rvk.ransac_estimate_csr(off, az, dop, p)
for a in (r.inlier_count, r.winning_trial, r.mask, e.tobytes()):
    h.update(np.asarray(a).tobytes() if not isinstance(a, bytes) else a)
dev = torch.device("cuda", 0)
d = [torch.from_numpy(a).to(dev) for a in (off, az, dop)]
C_, P_ = off.size - 1, int(off[-1])
o = {"inlier_count": torch.zeros(C_, dtype=torch.int32, device=dev),
     "winning_trial": torch.zeros(C_, dtype=torch.int32, device=dev),
     "mask": torch.zeros(P_, dtype=torch.uint8, device=dev),
     "est": torch.zeros(C_ * 48, dtype=torch.uint8, device=dev)}
rvk.ransac_estimate_device(d[0], d[1], d[2], p, o)
torch.cuda.synchronize()
assert (o["inlier_count"].cpu().numpy() == r.inlier_count).all()
assert (o["mask"].cpu().numpy() == r.mask).all()
assert o["est"].cpu().numpy().tobytes() == e.tobytes()
np.save(sys.argv[2], np.concatenate([[0], np.cumsum([len(x) for x in cl])]))
if len(sys.argv) > 3:  # the large clusters (the CTA path) against the C oracle
    from oracle.binding import Oracle, make_params
    orc = Oracle()
    big = np.nonzero(np.diff(off) > 384)[0]
    assert big.size >= 10
    for c in big:
        ro, _ = orc.ransac_estimate_range(off, az, dop, make_params(300, 1.0, 12), int(c),
                                          int(c) + 1)
        s = slice(off[c], off[c + 1])
        assert (ro.mask[s] == r.mask[s]).all(), c
        assert ro.winning_trial[c] == r.winning_trial[c] and ro.inlier_count[c] == r.inlier_count[c]
print(h.hexdigest())
"""


def test_mixed_batch_small_and_large_clusters(gpu_lib, oracle, tmp_path):
    """A batch of > 6144 small clusters (the fused prep + score path) with
    clusters of 300-1800 points interleaved (the CTA path: listed by the
    fused kernel, prepared by persistent CTAs, scored by score_kernel,
    selected by select_warp_kernel): host and device API agree, every path
    (default, fused prep+score off, whole-path fused forced) gives the same
    bytes, and the large clusters match the oracle."""
    digests = {}
    for name, env in (("default", {}), ("no_prep_score", {"RVK_PREP_SCORE": "0"}),
                      ("cta", {"RVK_PREP_SCORE": "0", "RVK_PREP_WARP": "0",
                               "RVK_SELECT_WARP": "0"})):
        r = subprocess.run([sys.executable, "-c", _MIXED_BATCH_SCRIPT, ROOT,
                            str(tmp_path / "off.npy")] + (["check"] if name == "default" else []),
                           capture_output=True, text=True,
                           env=dict(os.environ, **env), cwd=ROOT, timeout=900)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        digests[name] = r.stdout.strip().splitlines()[-1]
    assert len(set(digests.values())) == 1, digests
    sizes = np.diff(np.load(tmp_path / "off.npy"))
    assert (sizes > 508).any() and (sizes.size > 6144)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0, 0]])
def test_multi_device_split_is_byte_identical(gpu_lib, devices):
    """rvk_ransac_estimate_multi (single-frame latency): the frame
    split into point-balanced cluster ranges, one host worker per entry of
    `devices` (the one GPU repeated here); RNG keys and ids stay frame-positional,
    so every output equals the single call byte for byte -- with and without
    caller keys/ids, and more parts than clusters."""
    cases = [W.single_frame(), W.automotive(seed=8, n_clusters=60),
             W.imaging(seed=9, n_clusters=900, total=200_000)]
    for w in cases:
        p = rvk.RansacParams(w.max_trials, w.threshold_scale, 5)
        C_ = w.offsets.size - 1
        for ids, keys in [(None, None), (np.arange(C_)[::-1] + 7, (np.arange(C_) * 3) % 1000)]:
            r, e = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p, frame_id=4,
                                           cluster_ids=ids, rng_cluster_index=keys)
            for _ in range(2):  # the second call reuses the workers' contexts
                rm, em = rvk.ransac_estimate_multi_csr(w.offsets, w.azimuth, w.doppler, p,
                                                       devices, frame_id=4, cluster_ids=ids,
                                                       rng_cluster_index=keys)
                np.testing.assert_array_equal(rm.mask, r.mask)
                np.testing.assert_array_equal(rm.inlier_count, r.inlier_count)
                np.testing.assert_array_equal(rm.winning_trial, r.winning_trial)
                assert em.tobytes() == e.tobytes()
