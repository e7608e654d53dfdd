"""Small end-to-end workload for compute-sanitizer runs: every kernel path
(CTA and warp prep, FFMA2 scoring, select/refit, the fused warp-per-cluster
kernel, packed masks, the device API's too-small-cluster sentinel, frame
stream, DBSCAN + extract + estimate_frame, combine_masks) on tiny frames.
Run it once with RVK_FUSED=0 and once with RVK_FUSED=1.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_12618_b200 as rvk  # noqa: E402
from tools import workloads as W  # noqa: E402


def main():
    w = W.automotive(seed=1, n_clusters=6, lo_pts=16, hi_pts=700)
    p = rvk.RansacParams(300, 1.0, 3)
    r, est = rvk.ransac_estimate_csr(w.offsets, w.azimuth, w.doppler, p)
    off, az, dop = rvk.clusters_to_csr([np.stack([w.azimuth[:40], w.doppler[:40]], 1)] * 3)
    rvk.run_ransac_csr(off, az, dop, rvk.RansacParams(64, 0.5, 1))
    rvk.trial_counts_csr(w.offsets, w.azimuth, w.doppler, rvk.RansacParams(40, 1.0, 2))
    rvk.seed_pairs_csr(w.offsets, rvk.RansacParams(40, 1.0, 2))
    rvk.cluster_thresholds_csr(w.offsets, w.azimuth, w.doppler)
    rvk.estimate_all_csr(w.offsets, w.azimuth, w.doppler, r.mask)
    with rvk.FrameStream(p, depth=2) as fs:
        t = [fs.submit(w.offsets, w.azimuth, w.doppler) for _ in range(3)]
        for k in t:
            fs.result(k)
    fr = rvk.Frame(frame_id=1, x=w.x, y=w.y, z=np.zeros(w.n_points), doppler=w.doppler,
                   azimuth=w.azimuth)
    labels, o2, pi, res, e2 = rvk.estimate_frame(fr, rvk.ClusteringParams(2.0, 3), p)
    rvk.combine_masks_labels(labels, np.arange(o2.size - 1, dtype=np.int32), o2, res.mask)
    rvk.dbscan_points(w.x, w.y, np.zeros(w.n_points), rvk.ClusteringParams(1.5, 4, "xyz"))
    # imaging-like small clusters (warp prep / fused path), packed masks
    wi = W.imaging(seed=9, n_clusters=40, total=8000)
    rvk.ransac_estimate_csr(wi.offsets, wi.azimuth, wi.doppler, p, packed_mask=True)
    with rvk.FrameStream(p, depth=2) as fs:
        fs.result(fs.submit(wi.offsets, wi.azimuth, wi.doppler, packed_mask=True))
    # one frame split over two workers (the multi-GPU latency API, one device here)
    rvk.ransac_estimate_multi_csr(wi.offsets, wi.azimuth, wi.doppler, p, [0, 0])
    # device API with clusters below the minimum (sentinel path)
    import torch
    sizes = np.array([30, 1, 0, 2, 600, 5])
    o3 = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    P3 = int(o3[-1])
    rng = np.random.default_rng(3)
    dev = torch.device("cuda", 0)
    d = [torch.from_numpy(a).to(dev) for a in (o3, rng.uniform(-1, 1, P3), rng.uniform(-5, 5, P3))]
    out = {"inlier_count": torch.zeros(6, dtype=torch.int32, device=dev),
           "winning_trial": torch.zeros(6, dtype=torch.int32, device=dev),
           "mask": torch.zeros(P3, dtype=torch.uint8, device=dev),
           "est": torch.zeros(6 * 48, dtype=torch.uint8, device=dev)}
    rvk.ransac_estimate_device(d[0], d[1], d[2], p, out)
    torch.cuda.synchronize()
    print("sanitize workload done:", w.n_clusters, "clusters,", w.n_points, "points")


if __name__ == "__main__":
    main()
