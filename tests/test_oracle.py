"""CPU: the C oracle (oracle/rvk_oracle.c) pinned against the reference.

1. Bit-exact against every golden vector produced by the UNMODIFIED reference
   (tests/golden/make_golden.py -> oracle/_ref/librvk_ref.so).
2. Live cross-check against the reference build when it is present.
3. The reference's own known-answer tests, restated
   (tests/test_ransac.cpp, tests/test_velocity.cpp in /root/reference/proj).
"""
import math

import numpy as np
import pytest

from conftest import assert_estimates_close
from oracle.binding import CheckerError, make_params


def test_rng_streams_match_reference_vectors(oracle, golden_rng):
    for (seed, hi, lo), row in zip(golden_rng["keys"], golden_rng["rng_u64"]):
        got = [oracle.rng_u64(int(seed), int(hi), int(lo), k) for k in range(8)]
        assert got == [int(v) for v in row]


def test_seed_pairs_match_reference_vectors(oracle, golden_rng):
    for (s, c, t, n), (i, j) in zip(golden_rng["seed_pair_in"], golden_rng["seed_pair_out"]):
        assert oracle.seed_pair(int(s), int(c), int(t), int(n)) == (int(i), int(j))


def test_thresholds_and_normalization_bit_exact(oracle, golden_cases):
    for g in golden_cases:
        norm, thr, xy = oracle.cluster_thresholds(g["offsets"], g["az"], g["dop"],
                                                  g["threshold_scale"])
        np.testing.assert_array_equal(norm, g["norm"], err_msg=g["name"])
        np.testing.assert_array_equal(thr, g["threshold"], err_msg=g["name"])
        np.testing.assert_array_equal(xy, g["normalized"], err_msg=g["name"])


def test_trial_counts_bit_exact(oracle, golden_cases):
    for g in golden_cases:
        p = make_params(g["max_trials"], g["threshold_scale"], g["seed"])
        got = oracle.trial_counts(g["offsets"], g["az"], g["dop"], p)
        np.testing.assert_array_equal(got, g["trial_counts"], err_msg=g["name"])


def test_sequential_ransac_bit_exact(oracle, golden_cases):
    for g in golden_cases:
        p = make_params(g["max_trials"], g["threshold_scale"], g["seed"])
        r = oracle.sequential_ransac(g["offsets"], g["az"], g["dop"], p)
        np.testing.assert_array_equal(r.inlier_count, g["inlier_count"], err_msg=g["name"])
        np.testing.assert_array_equal(r.winning_trial, g["winning_trial"], err_msg=g["name"])
        np.testing.assert_array_equal(r.mask, g["mask"], err_msg=g["name"])


def test_lsq_matches_reference(oracle, golden_cases):
    for g in golden_cases:
        n = g["offsets"].size - 1
        est = oracle.estimate_all(g["offsets"], g["az"], g["dop"], g["mask"],
                                  frame_id=g["frame_id"],
                                  cluster_ids=np.arange(n, dtype=np.int32) + 100)
        # Same sequential reduction order as the reference build with the
        # Eigen stand-in: bit-identical.
        for f in ("v_x", "v_y", "heading", "has_heading", "condition_ok", "inlier_count"):
            np.testing.assert_array_equal(est[f], g["estimates"][f], err_msg=g["name"] + f)
        assert_estimates_close(est, g["estimates"], label=g["name"],
                               frame=(g["offsets"], g["az"], g["mask"]))


def test_live_against_reference_random(oracle, reference):
    rng = np.random.default_rng(7)
    for _ in range(40):
        k = int(rng.integers(1, 6))
        sizes = rng.integers(3, 60, size=k)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        az = rng.uniform(-1.3, 1.3, off[-1])
        dop = rng.uniform(-25, 25, off[-1])
        p = make_params(int(rng.integers(1, 80)), float(rng.uniform(0.1, 3)),
                        int(rng.integers(0, 2**63)))
        a = oracle.sequential_ransac(off, az, dop, p)
        b = reference.run_ransac(off, az, dop, p, workers=3)
        np.testing.assert_array_equal(a.mask, b.mask)
        np.testing.assert_array_equal(a.winning_trial, b.winning_trial)
        np.testing.assert_array_equal(a.inlier_count, b.inlier_count)


def test_live_against_reference_extreme_values(oracle, reference):
    import paper_2012_12618_b200 as rvk
    from conftest import EXTREME_PARAMS, extreme_value_clusters
    for cl in extreme_value_clusters():
        off, az, dop = rvk.clusters_to_csr(cl)
        for T, scale in EXTREME_PARAMS:
            p = make_params(T, scale, 5)
            a = oracle.sequential_ransac(off, az, dop, p)
            b = reference.run_ransac(off, az, dop, p, workers=2)
            np.testing.assert_array_equal(a.mask, b.mask)
            np.testing.assert_array_equal(a.winning_trial, b.winning_trial)
            np.testing.assert_array_equal(a.inlier_count, b.inlier_count)


# ---- the reference's own known-answer tests, restated ----

def test_kat_mad_one_third(oracle):
    # test_ransac.cpp:91-100 / :120-127: MAD of (0, .5, 1) = 1/3.
    off = np.array([0, 3], np.int64)
    _, thr, _ = oracle.cluster_thresholds(off, np.array([0.0, 1.0, 2.0]),
                                          np.array([0.0, 0.5, 1.0]), 1.0)
    assert thr[0] == 0.3333333333333333
    _, thr3, _ = oracle.cluster_thresholds(off, np.array([0.0, 1.0, 2.0]),
                                           np.array([0.0, 0.5, 1.0]), 3.0)
    assert thr3[0] == 3.0 * 0.3333333333333333


def test_kat_zero_threshold_keeps_seeds(oracle):
    # test_ransac.cpp:160-171
    xy = np.array([[0.0, 0.0], [1.0, 0.5], [0.25, 0.8], [0.7, 0.3]])
    cnt, mask = oracle.run_trial(xy, 0, 1, 0.0, want_mask=True)
    assert cnt == 2 and list(mask) == [1, 1, 0, 0]


def test_kat_degenerate_seeds_score_zero(oracle):
    # test_ransac.cpp:173-181
    xy = np.array([[0.5, 0.0], [0.5, 1.0], [0.0, 0.5], [1.0, 0.5]])
    cnt, mask = oracle.run_trial(xy, 0, 1, 10.0, want_mask=True)
    assert cnt == 0 and not mask.any()


def test_kat_seed_pair_coverage(oracle):
    # test_ransac.cpp:213-229: all 6 ordered pairs of 3 indices show up.
    seen = {oracle.seed_pair(9, 2, t, 3) for t in range(200)}
    assert len(seen) == 6 and all(a != b for a, b in seen)
    with pytest.raises(CheckerError):
        oracle.seed_pair(9, 0, 0, 1)


def test_kat_collinear_first_trial_wins(oracle):
    # test_ransac.cpp:231-246
    off = np.array([0, 5], np.int64)
    az = np.array([0.0, 0.1, 0.2, 0.3, 0.4])
    dop = np.array([1.0, 1.2, 1.4, 1.6, 1.8])
    r = oracle.sequential_ransac(off, az, dop, make_params(32, 1.0, 0))
    assert r.inlier_count[0] == 5 and r.winning_trial[0] == 0 and r.mask.all()


def test_kat_heading_and_degenerate_lsq(oracle):
    # test_velocity.cpp:197-203 (heading KATs) and :255-288.
    off = np.array([0, 1], np.int64)
    for (vx, vy, want) in [(1.0, 0.0, 0.0), (0.0, 1.0, math.pi / 2), (-1.0, 0.0, math.pi),
                           (-1.0, -1.0, -2.356194490192345)]:
        az = np.array([math.atan2(vy, vx)])
        d = np.array([math.hypot(vx, vy)])
        e = oracle.estimate_all(off, az, d, np.array([1], np.uint8))
        assert e["has_heading"][0] == 1
        assert abs(e["heading"][0] - want) < 1e-15
    off3 = np.array([0, 3], np.int64)
    az = np.array([0.2, 0.4, 0.6])
    dp = np.array([5.0, 6.0, 7.0])
    e0 = oracle.estimate_all(off3, az, dp, np.zeros(3, np.uint8))
    assert e0["inlier_count"][0] == 0 and e0["condition_ok"][0] == 0 and e0["has_heading"][0] == 0
    e1 = oracle.estimate_all(off3, az, dp, np.array([0, 1, 0], np.uint8))
    assert abs(e1["v_x"][0] - 6.0 * math.cos(0.4)) < 1e-12
    assert e1["condition_ok"][0] == 0
    offn = np.array([0, 10], np.int64)
    ef = oracle.estimate_all(offn, np.full(10, 0.3), np.full(10, 12.0), np.ones(10, np.uint8))
    assert ef["condition_ok"][0] == 0
    assert abs(ef["v_x"][0] - 12.0 * math.cos(0.3)) < 1e-12
    assert abs(ef["v_y"][0] - 12.0 * math.sin(0.3)) < 1e-12


def test_validation_errors(oracle):
    off = np.array([0, 2], np.int64)
    with pytest.raises(CheckerError) as e:
        oracle.sequential_ransac(off, np.zeros(2), np.zeros(2), make_params())
    assert e.value.status == 2 and "cluster 0 has 2 points, need 3" in str(e.value)
    off = np.array([0, 8], np.int64)
    with pytest.raises(CheckerError) as e:
        oracle.sequential_ransac(off, np.zeros(8), np.zeros(8), make_params(max_trials=0))
    assert "max_trials must be at least 1" in str(e.value)
    with pytest.raises(CheckerError) as e:
        oracle.sequential_ransac(off, np.zeros(8), np.zeros(8), make_params(threshold_scale=0.0))
    assert "threshold_scale must be positive" in str(e.value)
