"""Pinned H2D bandwidth: one copy stream vs several concurrent ones (15 MB/step)."""
import torch, time, json
n = 15_000_000 // 4
res = {}
for k in (1, 2, 3, 4):
    hs = [torch.empty(n // k, dtype=torch.float32).pin_memory() for _ in range(k)]
    ds = [torch.empty_like(h, device="cuda") for h in hs]
    ss = [torch.cuda.Stream() for _ in range(k)]
    for _ in range(3):
        for h, d, s in zip(hs, ds, ss):
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 40
    for _ in range(reps):
        for h, d, s in zip(hs, ds, ss):
            with torch.cuda.stream(s):
                d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    res[f"streams{k}"] = reps * n * 4 / dt / 1e9
# H2D while D2H runs
h = torch.empty(n, dtype=torch.float32).pin_memory(); d = torch.empty_like(h, device="cuda")
h2 = torch.empty(n, dtype=torch.float32).pin_memory(); d2 = torch.empty_like(h2, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(40):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
res["h2d_with_concurrent_d2h"] = 40 * n * 4 / dt / 1e9
print(json.dumps(res))
