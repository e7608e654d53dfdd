"""Clustering + whole-frame-path timing.

Config-4-shaped frames (imaging radar: 5000 objects, 1M points) through
  rvk.dbscan_points       (rvk_dbscan: H2D x,y -> grid-hash DBSCAN -> D2H labels)
  rvk.estimate_frame      (rvk_estimate_frame: dbscan -> extract -> gather ->
                           run_ransac -> estimate_all, one call per frame)
and the unmodified reference's rvk::dbscan (O(N^2)) on a bounded prefix.
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_12618_b200 as rvk  # noqa: E402
from tools import workloads as W  # noqa: E402


def timeit(f, reps):
    f()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts))


def main():
    w = W.imaging(seed=4000)
    n = w.n_points
    cp = rvk.ClusteringParams(2.0, 3)
    t_db = timeit(lambda: rvk.dbscan_points(w.x, w.y, None, cp), 10)
    fr = rvk.Frame(frame_id=0, x=w.x, y=w.y, z=np.zeros(n), doppler=w.doppler, azimuth=w.azimuth)
    rp = rvk.RansacParams(256, 1.0, 0)
    t_fr = timeit(lambda: rvk.estimate_frame(fr, cp, rp), 10)
    labels = rvk.dbscan_points(w.x, w.y, None, cp)
    out = {"workload": f"imaging frame (config 4): {w.n_clusters} objects, {n} points, eps 2 m, "
                       "min_pts 3, T=256",
           "gpu_dbscan_ms": t_db * 1e3, "gpu_dbscan_points_per_sec": n / t_db,
           "gpu_estimate_frame_ms": t_fr * 1e3, "gpu_frames_per_sec": 1.0 / t_fr,
           "clusters_found": int(labels.max()) + 1,
           "note": "host API wall time incl. H2D of the frame and D2H of all outputs"}
    try:
        from oracle.binding import Reference
        ref = Reference()
        k = 40_000
        t0 = time.perf_counter()
        rl = ref.dbscan(w.x[:k], w.y[:k], None, 2.0, 3, 0)
        t_ref = time.perf_counter() - t0
        gl = rvk.dbscan_points(w.x[:k], w.y[:k], None, cp)
        out["cpu_reference_dbscan"] = {
            "sample_points": k, "ms": t_ref * 1e3, "points_per_sec": k / t_ref,
            "identical_labels": bool((rl == gl).all()),
            "note": "unmodified rvk::dbscan (O(N^2) neighbour lists), 1 thread; the full 1M-point "
                    "frame would take ~(1e6/4e4)^2 = 625x the sample"}
    except Exception as e:  # noqa: BLE001
        out["cpu_reference_dbscan"] = {"unavailable": str(e)[:200]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
