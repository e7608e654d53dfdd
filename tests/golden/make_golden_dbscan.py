"""Golden DBSCAN + extract_clusters fixtures from the UNMODIFIED reference
(rvk::dbscan, rvk::extract_clusters, src/clustering.cpp:24-155, through
oracle/ref_capi.cpp). Build container only:

    python tests/golden/make_golden_dbscan.py      -> tests/golden/dbscan.npz

Cases: blobs + uniform noise, quantized coordinates (equal distances, so
border ties and exactly-eps neighbours occur), duplicates, a chain of points
exactly eps apart, min_pts 1, XYZ features, and radar frames from the
reference's own generate_frame.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.binding import Reference  # noqa: E402


def main():
    ref = Reference()
    rng = np.random.default_rng(20121218)
    cases = []  # (name, x, y, z, eps, min_pts, features, min_cluster_size)

    def blobs(n_blobs, size, n_noise, spread, span):
        c = rng.uniform(-span, span, (n_blobs, 2))
        pts = [c[b] + rng.normal(0, spread, (size, 2)) for b in range(n_blobs)]
        pts.append(rng.uniform(-span, span, (n_noise, 2)))
        p = np.concatenate(pts)
        return p[rng.permutation(len(p))]

    for k in range(6):
        p = blobs(int(rng.integers(1, 6)), int(rng.integers(5, 60)), int(rng.integers(0, 40)),
                  rng.uniform(0.3, 1.5), 30.0)
        cases.append((f"blobs{k}", p[:, 0], p[:, 1], None, float(rng.uniform(0.8, 3.0)),
                      int(rng.integers(1, 6)), 0, int(rng.integers(1, 5))))
    for k in range(4):  # quantized: equal distances, ties, exactly-eps pairs
        p = np.round(blobs(3, 40, 30, 1.0, 12.0) * 2) / 2
        cases.append((f"grid{k}", p[:, 0], p[:, 1], None, [0.5, 1.0, 1.5, 2.0][k],
                      int(rng.integers(2, 6)), 0, 3))
    dup = np.repeat(rng.uniform(-5, 5, (20, 2)), 3, axis=0)
    cases.append(("duplicates", dup[:, 0], dup[:, 1], None, 0.25, 3, 0, 3))
    chain = np.arange(50, dtype=np.float64) * 0.75
    cases.append(("chain_exact_eps", chain, np.zeros(50), None, 0.75, 2, 0, 3))
    cases.append(("min_pts_1", *blobs(2, 10, 10, 1.0, 10.0).T, None, 1.0, 1, 0, 1))
    cases.append(("all_noise", *(rng.uniform(-100, 100, (60, 2)).T), None, 0.5, 3, 0, 3))
    for k in range(3):
        p = blobs(4, 50, 40, 1.0, 15.0)
        z = rng.normal(0, [0.2, 1.0, 3.0][k], len(p))
        cases.append((f"xyz{k}", p[:, 0], p[:, 1], z, 2.0, 3, 1, 3))
    for k in range(4):  # radar frames (generate_frame, scene.cpp:105-189)
        n_obj = int(rng.integers(3, 30))
        objs = np.zeros((n_obj, 10))
        for i in range(n_obj):
            objs[i] = [10.0 + 9.0 * (i % 6), -30.0 + 12.0 * (i // 6), rng.uniform(0.5, 3),
                       rng.uniform(0.5, 6), rng.uniform(-15, 15), rng.uniform(-15, 15),
                       int(rng.integers(3, 120)), 0.25, 0.1, 0.0]
        x, y, _, _, _ = ref.generate_frame(int(rng.integers(0, 2**62)), objs)
        cases.append((f"radar{k}", x, y, None, 2.0, 3, 0, 3))
    big = blobs(60, 80, 400, 0.8, 80.0)
    cases.append(("large5200", big[:, 0], big[:, 1], None, 1.2, 4, 0, 3))

    blob = {"names": np.array([c[0] for c in cases])}
    for i, (name, x, y, z, eps, mp, feat, mcs) in enumerate(cases):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        lab = ref.dbscan(x, y, z, eps, mp, feat)
        lab2, off, pi = ref.extract_clusters(lab, mcs)
        blob.update({f"{i}/x": x, f"{i}/y": y, f"{i}/params": np.array([eps, mp, feat, mcs]),
                     f"{i}/labels": lab, f"{i}/extracted": lab2, f"{i}/offsets": off,
                     f"{i}/point_indices": pi})
        if z is not None:
            blob[f"{i}/z"] = np.ascontiguousarray(z, np.float64)
    np.savez_compressed(os.path.join(HERE, "dbscan.npz"), **blob)
    print("wrote", len(cases), "dbscan cases")


if __name__ == "__main__":
    main()
