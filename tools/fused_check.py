"""Development A/B check of a kernel-path switch: the same inputs through
two settings of an environment variable (default RVK_FUSED=1 vs 0) must give
byte-identical outputs; prints a rough per-call timing of each. Runs itself
in child processes (path selections are read once per process).

    python tools/fused_check.py [--var RVK_FUSED] [--a 1] [--b 0]
"""
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import numpy as np
    import torch
    import bench
    import paper_2012_12618_b200 as rvk
    from tools import workloads as W
    out = {}
    dev = torch.device("cuda", 0)
    cases = [("cfg1", [W.single_frame()], 256),
             ("cfg4_1frame", bench.make_frames(4, range(1)), 256),
             ("cfg2_1frame", bench.make_frames(2, range(1)), 1024),
             ("cfg4_T256", bench.make_frames(4, range(4)), 256),
             ("cfg4_T1024", bench.make_frames(4, range(2)), 1024),
             ("mixed", [W.automotive(seed=5, n_clusters=60, lo_pts=3, hi_pts=1500)], 300),
             ("cfg2", bench.make_frames(2, range(4)), 1024)]
    for name, frames, T in cases:
        off, az, dop, keys = bench.batch(frames)
        p = rvk.RansacParams(T, frames[0].threshold_scale, 0)
        C_, P_ = off.size - 1, int(off[-1])
        d = {k: torch.from_numpy(v).to(dev) for k, v in
             (("off", off), ("az", az), ("dop", dop), ("keys", keys))}
        o = {"inlier_count": torch.zeros(C_, dtype=torch.int32, device=dev),
             "winning_trial": torch.zeros(C_, dtype=torch.int32, device=dev),
             "mask": torch.zeros(P_, dtype=torch.uint8, device=dev),
             "est": torch.zeros(C_ * 48, dtype=torch.uint8, device=dev)}
        run = lambda: rvk.ransac_estimate_device(d["off"], d["az"], d["dop"], p, o,  # noqa
                                                 rng_cluster_index=d["keys"])
        run()
        torch.cuda.synchronize()
        h = hashlib.sha256()
        for k in ("inlier_count", "winning_trial", "mask", "est"):
            h.update(o[k].cpu().numpy().tobytes())
        # host API (knows the largest cluster) too
        r, e = rvk.ransac_estimate_csr(off, az, dop, p, rng_cluster_index=keys)
        h2 = hashlib.sha256()
        for a in (r.inlier_count, r.winning_trial, r.mask, e.tobytes()):
            h2.update(np.asarray(a).tobytes() if not isinstance(a, bytes) else a)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            run()
        a.record()
        for _ in range(10):
            run()
        b.record()
        b.synchronize()
        out[name] = {"dev": h.hexdigest()[:16], "host": h2.hexdigest()[:16],
                     "ms": a.elapsed_time(b) / 10, "evals": P_ * T}
    print(json.dumps(out))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--var", default="RVK_FUSED")
    ap.add_argument("--a", default="1")
    ap.add_argument("--b", default="0")
    args = ap.parse_args()
    res = {}
    for val, key in ((args.a, "1"), (args.b, "0")):
        r = subprocess.run([sys.executable, __file__, "--child"], capture_output=True, text=True,
                           env=dict(os.environ, **{args.var: val}), cwd=ROOT, timeout=900)
        if r.returncode != 0:
            print(r.stdout[-3000:], r.stderr[-3000:])
            sys.exit(1)
        res[key] = json.loads(r.stdout.strip().splitlines()[-1])
    ok = True
    for name in res["1"]:
        a, b = res["1"][name], res["0"][name]
        same = a["dev"] == b["dev"] and a["host"] == b["host"] and a["dev"] == a["host"]
        ok &= same
        print(f"{name:12s} identical={same} {args.var}={args.a} {a['ms']:.3f} ms "
              f"({a['evals'] / a['ms'] / 1e9:.2f} Tev/s)  {args.var}={args.b} {b['ms']:.3f} ms "
              f"({b['evals'] / b['ms'] / 1e9:.2f} Tev/s)")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        main()
