"""Randomised GPU-vs-oracle parity sweep (development tool, B200).

    python tools/fuzz_parity.py [--frames 3000] [--seed 1]

Random frames (1-12 clusters of 3-3000 points, clustered / uniform /
quantised / near-degenerate coordinates, random T, threshold scale and RNG
seed) through ransac_estimate_csr, compared with the C oracle: masks,
winning trials and counts bit-exact, estimates within the parity tolerance.
Prints one JSON line with the totals."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2012_12618_b200 as rvk  # noqa: E402
from conftest import assert_estimates_close  # noqa: E402
from oracle.binding import Oracle, make_params  # noqa: E402


def cluster(rng, n, stress=False):
    kind = 0 if stress else rng.integers(0, 5)
    if kind == 0:  # a moving object + outliers (stress: exactly 50%, micro-Doppler-like)
        th = rng.uniform(-1.2, 1.2) + rng.normal(0, rng.uniform(0.001, 0.3), n)
        v = rng.uniform(-30, 30, 2)
        d = v[0] * np.cos(th) + v[1] * np.sin(th) + rng.normal(0, 0.05, n)
        out = (rng.permutation(n) < n // 2) if stress else \
            rng.uniform(size=n) < rng.uniform(0, 0.5)
        d[out] = rng.uniform(-40, 40, out.sum())
        return np.stack([th, d], 1)
    if kind == 1:  # uniform
        return rng.uniform(-1, 1, (n, 2)) * rng.uniform(0.01, 100, 2)
    if kind == 2:  # quantised: ties everywhere
        q = rng.integers(2, 16)
        return np.round(rng.uniform(-1, 1, (n, 2)) * q) / q
    if kind == 3:  # tiny spread
        return 0.5 + rng.uniform(-1, 1, (n, 2)) * 10.0 ** rng.uniform(-12, -3)
    a = np.full(n, rng.uniform(-1, 1))  # near-degenerate azimuths (|dx| ~ 1e-12 after scaling)
    j = rng.uniform(size=n) < 0.3
    a[j] += rng.normal(0, 1e-3, j.sum())
    return np.stack([a + rng.normal(0, 1e-13, n), rng.uniform(-5, 5, n)], 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=3000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--stress", action="store_true",
                    help="config-3 regime: T in {2048, 4096}, threshold_scale 0.25, "
                         "50%% outliers, clusters of 64-2048 points")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    o = Oracle()
    t0 = time.time()
    n_clusters = n_points = 0
    for f in range(args.frames):
        if args.stress:
            k = int(rng.integers(1, 5))
            sizes = np.rint(64 * 32 ** rng.uniform(size=k)).astype(int)
            cl = [cluster(rng, int(s), stress=True) for s in sizes]
            T = int(rng.choice([2048, 4096]))
            scale = 0.25
        else:
            k = int(rng.integers(1, 13))
            sizes = np.minimum(3000, np.maximum(3, (10 ** rng.uniform(0.5, 3.5, k)).astype(int)))
            cl = [cluster(rng, int(s)) for s in sizes]
            T = int(rng.choice([1, 7, 64, 256, 257, 1024, 1500, 2048, 4096]))
            scale = float(10 ** rng.uniform(-3, 0.7))
        off, az, dop = rvk.clusters_to_csr(cl)
        p = rvk.RansacParams(T, scale, int(rng.integers(0, 2**63)))
        r, est = rvk.ransac_estimate_csr(off, az, dop, p, frame_id=f)
        ro = o.sequential_ransac(off, az, dop, make_params(p.max_trials, p.threshold_scale,
                                                           p.rng_seed))
        np.testing.assert_array_equal(r.mask, ro.mask, err_msg=f"frame {f}")
        np.testing.assert_array_equal(r.winning_trial, ro.winning_trial, err_msg=f"frame {f}")
        np.testing.assert_array_equal(r.inlier_count, ro.inlier_count, err_msg=f"frame {f}")
        oe = o.estimate_all(off, az, dop, ro.mask, frame_id=f)
        assert_estimates_close(est, oe, label=f"frame {f}", frame=(off, az, ro.mask))
        n_clusters += k
        n_points += int(off[-1])
    print(json.dumps({"frames": args.frames, "clusters": n_clusters, "points": n_points,
                      "mismatches": 0, "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
