"""Generate the golden parity fixtures from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/librvk_ref.so, built by
`make -C oracle ref` from /root/reference/proj/src). Every output array is
produced by the reference's own functions through oracle/ref_capi.cpp; the
inputs are stored next to them so the tests never need the reference:

  rng.npz        KeyedRng next_u64 streams and draw_seed_pair vectors
                 (test_rng.cpp has properties only, no golden values)
  cases.npz      RANSAC + LSQ cases: inputs, per-trial counts, thresholds,
                 normalization, winning trial / count / mask, estimates
  scene.npz      generate_frame outputs for a few specs (workload generator pin)

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.binding import Reference, make_params  # noqa: E402


def cases(rng: np.random.Generator):
    """(name, offsets, az, dop, max_trials, threshold_scale, seed) tuples."""
    out = []

    def add(name, clusters, T, scale, seed):
        sizes = [len(c) for c in clusters]
        off = np.zeros(len(clusters) + 1, np.int64)
        np.cumsum(sizes, out=off[1:])
        pts = np.concatenate([np.asarray(c, np.float64).reshape(-1, 2) for c in clusters])
        out.append((name, off, pts[:, 0].copy(), pts[:, 1].copy(), T, scale, seed))

    # Known-answer shapes from tests/test_ransac.cpp.
    add("collinear5", [[(0.0, 1.0), (0.1, 1.2), (0.2, 1.4), (0.3, 1.6), (0.4, 1.8)]], 32, 1.0, 0)
    add("dyadic_collinear", [[(0.0, 1.0), (0.25, 1.5), (0.5, 2.0), (0.75, 2.5), (1.0, 3.0)]],
        16, 1.0, 3)
    add("degenerate_x", [[(0.5, 0.0), (0.5, 1.0), (0.5, 0.5), (0.5, 0.25)]], 16, 1.0, 1)
    add("all_identical", [[(3.0, 7.0)] * 6], 8, 1.0, 2)
    add("min_size3", [[(0.1, 2.0), (0.4, -1.0), (0.9, 0.5)]], 64, 1.0, 9)
    add("duplicates", [[(0.1, 1.0), (0.1, 1.0), (0.2, 1.5), (0.2, 1.5), (0.3, 2.0), (0.9, -4.0)]],
        48, 1.0, 5)
    add("zero_mad", [[(0.0, 1.0), (0.1, 1.0), (0.2, 1.0), (0.3, 1.0), (0.4, 3.0)]], 32, 1.0, 4)
    # Random clusters, C3 style (acceptance_test.cpp:264-279), varied T/scale/seed.
    for f in range(60):
        k = int(rng.integers(1, 5))
        cl = []
        for _ in range(k):
            n = int(rng.integers(5, 41))
            cl.append(np.stack([rng.uniform(-1.3, 1.3, n), rng.uniform(-25, 25, n)], 1))
        add(f"c3_{f}", cl, int(rng.integers(16, 97)), 1.0, int(rng.integers(0, 2**63)))
    # Radar-like: Doppler = v . (cos, sin) + noise, with outliers; several scales.
    for f in range(24):
        k = int(rng.integers(1, 6))
        cl = []
        for _ in range(k):
            n = int(rng.integers(20, 300))
            th0 = rng.uniform(-1.0, 1.0)
            az = th0 + rng.uniform(-0.05, 0.05, n)
            vx, vy = rng.uniform(-20, 20, 2)
            d = vx * np.cos(az) + vy * np.sin(az) + rng.normal(0, 0.1, n)
            out_mask = rng.random(n) < rng.uniform(0.0, 0.5)
            d[out_mask] += rng.choice([-1, 1], out_mask.sum()) * rng.uniform(2, 5, out_mask.sum())
            cl.append(np.stack([az, d], 1))
        scale = float(rng.choice([1.0, 0.25, 0.5, 2.0, 3.0]))
        add(f"radar_{f}", cl, int(rng.choice([64, 128, 256])), scale, int(rng.integers(0, 2**63)))
    # Quantized values: many exact ties and boundary points.
    for f in range(12):
        n = int(rng.integers(8, 120))
        az = np.round(rng.uniform(-1, 1, n) * 8) / 8
        d = np.round(rng.uniform(-4, 4, n) * 4) / 4
        add(f"quant_{f}", [np.stack([az, d], 1)], int(rng.integers(32, 200)),
            float(rng.choice([1.0, 0.5, 0.25])), int(rng.integers(0, 2**63)))
    return out


def main():
    ref = Reference()
    rng = np.random.default_rng(20201223)

    # ---- RNG vectors
    keys = [(0, 0, 0), (42, 7, 3), (2**64 - 1, 123456, 987654), (5, 1, 0), (5, 2, 0),
            (9, 2, 17), (2024, 3, 127)]
    rng_u64 = np.array([[ref.rng_u64(s, h, l, k) for k in range(8)] for (s, h, l) in keys],
                       dtype=np.uint64)
    sp_in = []
    for _ in range(4000):
        seed = int(rng.integers(0, 2**63)) * int(rng.integers(1, 3))
        sp_in.append((seed % 2**64, int(rng.integers(0, 5000)), int(rng.integers(0, 4096)),
                      int(rng.choice([2, 3, 5, 64, 100, 2048, 100000]))))
    sp_in = np.array(sp_in, dtype=np.uint64)
    sp_out = np.array([ref.seed_pair(int(s), int(c), int(t), int(n)) for s, c, t, n in sp_in],
                      dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), keys=np.array(keys, dtype=np.uint64),
                        rng_u64=rng_u64, seed_pair_in=sp_in, seed_pair_out=sp_out)

    # ---- RANSAC / LSQ cases
    blob = {}
    names = []
    for (name, off, az, dop, T, scale, seed) in cases(rng):
        p = make_params(T, scale, seed)
        res = ref.sequential_ransac(off, az, dop, p)
        par = ref.run_ransac(off, az, dop, p, workers=4)
        assert (res.mask == par.mask).all() and (res.winning_trial == par.winning_trial).all()
        counts = ref.trial_counts(off, az, dop, p)
        norm, thr, xy = ref.cluster_thresholds(off, az, dop, scale)
        est = ref.sequential_lsq(off, az, dop, res.mask, frame_id=len(names),
                                 cluster_ids=np.arange(off.size - 1, dtype=np.int32) + 100)
        pre = f"{name}/"
        blob.update({pre + "offsets": off, pre + "az": az, pre + "dop": dop,
                     pre + "params": np.array([T, scale, 0], np.float64),
                     pre + "seed": np.array([seed], np.uint64),
                     pre + "inlier_count": res.inlier_count, pre + "winning_trial": res.winning_trial,
                     pre + "mask": res.mask, pre + "trial_counts": counts, pre + "norm": norm,
                     pre + "threshold": thr, pre + "normalized": xy, pre + "estimates": est})
        names.append(name)
    blob["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **blob)

    # ---- scene generator
    specs = []
    for s in range(4):
        k = int(rng.integers(1, 9))
        objs = np.zeros((k, 10))
        for i in range(k):
            objs[i] = [16.0 + 11.0 * (i % 4), -26.0 + 13.0 * (i // 4), rng.uniform(0.5, 8),
                       rng.uniform(0.5, 8), rng.uniform(-15, 15), rng.uniform(-15, 15),
                       int(rng.integers(3, 300)), rng.choice([0.0, 0.2, 0.3, 0.49]),
                       rng.choice([0.0, 0.05, 0.1]), 0.0]
        specs.append((int(rng.integers(0, 2**63)), objs))
    sc = {}
    for i, (seed, objs) in enumerate(specs):
        x, y, d, a, flag = ref.generate_frame(seed, objs)
        sc.update({f"{i}/seed": np.array([seed], np.uint64), f"{i}/objects": objs, f"{i}/x": x,
                   f"{i}/y": y, f"{i}/doppler": d, f"{i}/azimuth": a, f"{i}/outlier": flag})
    sc["n"] = np.array([len(specs)])
    np.savez_compressed(os.path.join(HERE, "scene.npz"), **sc)
    print("wrote", len(names), "cases")


if __name__ == "__main__":
    main()
