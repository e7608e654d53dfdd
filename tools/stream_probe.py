"""FrameStream throughput vs depth, pinned inputs, config-2 batches of 8 frames."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_12618_b200 as rvk
from paper_2012_12618_b200 import _native, stream as S
from tools import workloads as W
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
hb = []
for j in range(4):
    off, az, dop, keys, _, _ = S.batch_frames([W.automotive(seed=1000 + 8 * j + i) for i in range(8)])
    hb.append((pin(off), pin(az), pin(dop), pin(keys)))
P = max(int(h[0][-1]) for h in hb); Cn = max(h[0].size - 1 for h in hb)
p = rvk.RansacParams(1024, 1.0, 0)
for depth in (1, 2, 3, 4, 6):
    outs = [(pin(np.zeros(Cn, np.int32)), pin(np.zeros(Cn, np.int32)), pin(np.zeros(P, np.uint8)),
             np.zeros(Cn, _native.ESTIMATE_DTYPE)) for _ in range(depth)]
    fs = rvk.FrameStream(p, depth=depth)
    def run(n):
        ts, sub = [], 0.0
        for j in range(n):
            off, az, dop, keys = hb[j % len(hb)]
            nc, npt = off.size - 1, int(off[-1]); o = outs[j % depth]
            t = time.perf_counter()
            ts.append(fs.submit(off, az, dop, rng_cluster_index=keys,
                                out=(o[0][:nc], o[1][:nc], o[2][:npt], o[3][:nc])))
            sub += time.perf_counter() - t
        for t in ts: fs.wait(t)
        return sub
    run(12)
    t0 = time.perf_counter(); sub = run(40); dt = time.perf_counter() - t0
    print(f"depth {depth}: {dt / 40 * 1e3:.3f} ms/step, submit {sub / 40 * 1e3:.3f} ms/step", flush=True)
    fs.close()
os.environ["RVK_TRACE"] = "1"
