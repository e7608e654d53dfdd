"""Host -> host single-frame latency breakdown through rvk_ransac_estimate
(development probe): pinned inputs/outputs, RVK_TRACE timings per call.

    RVK_TRACE=1 python tools/e2e_latency.py [--config 4] [--packed]
"""
import argparse
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--packed", action="store_true")
    a = ap.parse_args()
    import torch
    import bench
    import paper_2012_12618_b200 as rvk
    from paper_2012_12618_b200 import _native
    lib = _native.gpu()
    w = bench.make_frames(a.config, [0])[0]
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa
    off, az, dop = pin(w.offsets), pin(w.azimuth), pin(w.doppler)
    Cn, Pn = w.n_clusters, w.n_points
    cnt, tr = pin(np.zeros(Cn, np.int32)), pin(np.zeros(Cn, np.int32))
    mask = pin(np.zeros((Pn + 7) // 8 if a.packed else Pn, np.uint8))
    est = pin(np.zeros(Cn * 48, np.uint8))
    p = rvk.RansacParams(w.max_trials, w.threshold_scale, 0).c()
    fn = lib.rvk_ransac_estimate_packed if a.packed else lib.rvk_ransac_estimate
    lat = []
    for j in range(a.reps + 3):
        t0 = time.perf_counter()
        st = fn(0, Cn, off.ctypes.data, az.ctypes.data, dop.ctypes.data, None, C.addressof(p),
                None, cnt.ctypes.data, tr.ctypes.data, mask.ctypes.data, est.ctypes.data)
        assert st == 0, lib.rvk_last_error()
        if j >= 3:
            lat.append((time.perf_counter() - t0) * 1e3)
    h2d = 16 * Pn + 8 * Cn
    print(f"config {a.config}: p50 {statistics.median(lat):.3f} ms min {min(lat):.3f} ms; "
          f"H2D {h2d / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
