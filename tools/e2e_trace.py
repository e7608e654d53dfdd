"""Host-API latency breakdown (RVK_TRACE=1) for one 8-frame automotive batch."""
import ctypes as C, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_12618_b200 as rvk
from paper_2012_12618_b200 import _native, stream as S
from tools import workloads as W
frames = [W.automotive(seed=1000 + i) for i in range(8)]
off, az, dop, keys, _, _ = S.batch_frames(frames)
pin = lambda a: torch.from_numpy(a).pin_memory()
t_off, t_az, t_dop, t_keys = pin(off), pin(az), pin(dop), pin(keys)
P, Cn = int(off[-1]), off.size - 1
cnt = torch.zeros(Cn, dtype=torch.int32).pin_memory()
tr = torch.zeros(Cn, dtype=torch.int32).pin_memory()
mask = torch.zeros(P, dtype=torch.uint8).pin_memory()
est = np.zeros(Cn, _native.ESTIMATE_DTYPE)
x = torch.empty(14_400_000 // 4, dtype=torch.float32).pin_memory()
dx = torch.empty_like(x, device="cuda")
for _ in range(3): dx.copy_(x, non_blocking=True)
torch.cuda.synchronize()
ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ea.record(); [dx.copy_(x, non_blocking=True) for _ in range(10)]; eb.record(); eb.synchronize()
print(f"H2D {10 * x.numel() * 4 / (ea.elapsed_time(eb) / 1e3) / 1e9:.1f} GB/s (pinned, 14.4 MB)")
lib = _native.gpu()
p = rvk.RansacParams(1024, 1.0, 0).c()
for i in range(12):
    t = time.perf_counter()
    st = lib.rvk_ransac_estimate(0, Cn, t_off.data_ptr(), t_az.data_ptr(), t_dop.data_ptr(), None,
                                 C.addressof(p), t_keys.data_ptr(), cnt.data_ptr(), tr.data_ptr(),
                                 mask.data_ptr(), est.ctypes.data)
    print(f"call {i}: {(time.perf_counter() - t) * 1e3:.3f} ms st={st}", flush=True)
