"""Single-frame latency breakdown (development probe, B200).

    python tools/frame_latency.py [--config 2]

Prints, for one frame per call through rvk_ransac_estimate_device with
device-resident inputs: the p50 call latency (CUDA events around the call),
the per-frame time of 32 back-to-back calls (GPU-bound when the host enqueues
faster than the device drains), and the per-stage device times
(rvk_profile_*)."""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2012_12618_b200 as rvk  # noqa: E402
from paper_2012_12618_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    lib = _native.gpu()
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    w = bench.make_frames(args.config, [0])[0]
    off, az, dop, keys = bench.batch([w])
    d = {k: torch.from_numpy(v).to(dev) for k, v in
         (("off", off), ("az", az), ("dop", dop), ("keys", keys))}
    C_, P = off.size - 1, int(off[-1])
    outs = {"cnt": torch.zeros(C_, dtype=torch.int32, device=dev),
            "trial": torch.zeros(C_, dtype=torch.int32, device=dev),
            "mask": torch.zeros(P, dtype=torch.uint8, device=dev),
            "est": torch.zeros(C_ * 48, dtype=torch.uint8, device=dev)}
    p = rvk.RansacParams(w.max_trials, w.threshold_scale, 0)
    pc = p.c()

    def call():
        st = lib.rvk_ransac_estimate_device(
            0, C_, P, d["off"].data_ptr(), d["az"].data_ptr(), d["dop"].data_ptr(), None,
            C.addressof(pc), d["keys"].data_ptr(), outs["cnt"].data_ptr(),
            outs["trial"].data_ptr(), outs["mask"].data_ptr(), outs["est"].data_ptr(),
            C.c_void_p(stream.cuda_stream))
        assert st == 0, st

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    lat = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        call()
        b.record(stream)
        b.synchronize()
        lat.append(a.elapsed_time(b))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(32):
        call()
    b.record(stream)
    b.synchronize()
    lib.rvk_profile_enable(1)
    for _ in range(20):
        call()
    lib.rvk_profile_enable(0)
    ms = (C.c_double * 4)()
    n = (C.c_int64 * 4)()
    lib.rvk_profile_read(ms, n, 4)
    print(json.dumps({
        "config": args.config, "clusters": C_, "points": P, "max_trials": w.max_trials,
        "p50_call_latency_ms": statistics.median(lat),
        "back_to_back_ms_per_frame": a.elapsed_time(b) / 32,
        "stage_ms": {k: ms[i] / max(1, n[i]) for i, k in
                     ((0, "prep"), (2, "score"), (3, "select"))}}))


if __name__ == "__main__":
    main()
