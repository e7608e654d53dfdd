"""e2e pipeline-chunking sweep + H2D bandwidth (development tool)."""
import json, os, subprocess, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
x = torch.empty(14_400_000 // 4, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); [d.copy_(x, non_blocking=True) for _ in range(10)]; b.record(); b.synchronize()
print(json.dumps({"h2d_GBps": 10 * x.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9}))
y = torch.empty_like(x); 
a.record(); [y.copy_(d, non_blocking=True) for _ in range(10)]; b.record(); b.synchronize()
print(json.dumps({"d2h_GBps": 10 * x.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9}))
for chunk, mx in [(1 << 17, 8), (1 << 18, 4), (1 << 19, 2), (1 << 16, 16), (1 << 20, 1), (200000, 4)]:
    env = dict(os.environ, RVK_PIPE_CHUNK=str(chunk), RVK_PIPE_MAX=str(mx))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "20", "--warmup", "3",
                          "--no-cpu-baseline", "--resident-frames", "16", "--e2e-steps", "40"],
                         env=env, capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if l.startswith("{")]
    if line:
        e = json.loads(line[-1])["e2e"]
        print(json.dumps({"chunk": chunk, "max": mx, "e2e": e["value"], "p50_ms": e["p50_step_latency_ms"]}))
