"""Development helper: one device-API call of a bench batch (for ncu).

    python tools/one_call.py --config 4 --frames 4 [--max-trials T] [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--max-trials", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2012_12618_b200 as rvk
    frames = bench.make_frames(a.config, range(a.frames))
    off, az, dop, keys = bench.batch(frames)
    T = a.max_trials or frames[0].max_trials
    p = rvk.RansacParams(T, frames[0].threshold_scale, 0)
    dev = torch.device("cuda", 0)
    d = {k: torch.from_numpy(v).to(dev) for k, v in
         (("off", off), ("az", az), ("dop", dop), ("keys", keys))}
    C_, P_ = off.size - 1, int(off[-1])
    o = {"inlier_count": torch.zeros(C_, dtype=torch.int32, device=dev),
         "winning_trial": torch.zeros(C_, dtype=torch.int32, device=dev),
         "mask": torch.zeros(P_, dtype=torch.uint8, device=dev),
         "est": torch.zeros(C_ * 48, dtype=torch.uint8, device=dev)}
    for _ in range(a.reps):
        rvk.ransac_estimate_device(d["off"], d["az"], d["dop"], p, o, rng_cluster_index=d["keys"])
    torch.cuda.synchronize()
    print("ok", C_, P_, T)


if __name__ == "__main__":
    main()
