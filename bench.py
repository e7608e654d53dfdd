"""Benchmark: per-cluster RANSAC + LSQ velocity-profile estimation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1|2|3|4|5] [--max-trials T]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Metric (BASELINE.json): hypothesis x point inlier evaluations per second,
whole job (all ranks); also clusters/s and p50 frame latency.

Workload at N=1: BASELINE configs[3], the largest single-GPU configuration --
the imaging-radar frame, 5000 clusters / 1,000,000 points (n_i ~ U[50, 350]),
25% outliers, T = 256 (`--max-trials 1024` for its T=1024 variant, SURVEY
8(d)). Synthetic frames of the generate_frame recipe (tools/workloads.py). A
step = 16 frames batched into one call with frame-local RNG keys, through the
whole path: prep (normalize, median, MAD, hypotheses) -> FP32 upper-bound
scoring -> exact argmax / mask -> LSQ refit + heading. 96 distinct frames stay
resident in HBM and steps cycle through them, so the inputs touched between
reuses (1.5 GB) exceed the 126 MB L2. Multi-GPU: each rank scores its own
frames (weak scaling, no collective on the data path); elapsed = max over
ranks of CUDA-event time. `--config 5` runs BASELINE configs[4] instead: a
stream of config-2 frames sharded over the GPUs with the results gathered to
host memory (tools/stream_bench.py).

--impl reference times the reference's own CPU implementation
(oracle/_ref/librvk_ref.so: the unmodified rvk::run_ransac + estimate_all with
all host threads) on the same step (16 frames, drawn by the reference's own
generate_frame), rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hypothesis_point_evals_per_sec"
UNIT = "evals/s"
FLOP_PER_EVAL = 4  # 1 mul + 2 add + 1 div (ref form) == 2 FMA (affine form)
# SURVEY.md 8(d) algorithmic HBM bytes: ingest reads the f64 (az, dop) and
# writes the f32 normalized (x, y), plus the offsets; refit reads the f64
# (az, dop), a mask bit, and writes the 40 B estimate per cluster.
INGEST_B_PT, INGEST_B_CL = 16 + 8, 4
REFIT_B_PT, REFIT_B_CL = 16 + 1 / 8, 40
HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--max-trials", type=int, default=0, help="override the config's T")
    ap.add_argument("--frames-per-step", type=int, default=16)
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--resident-frames", type=int, default=96)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--latency-reps", type=int, default=100)
    ap.add_argument("--stream-frames", type=int, default=10_000, help="config 5: frames")
    ap.add_argument("--stream-pool", type=int, default=64,
                    help="config 5: distinct frames generated and cycled")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def physical_cores():
    """Unique (package, core) pairs of /sys cpu topology, as the reference's
    acceptance test counts them (tests/acceptance_test.cpp:69-92)."""
    cores = set()
    cpu = 0
    while True:
        base = f"/sys/devices/system/cpu/cpu{cpu}/topology/"
        try:
            with open(base + "physical_package_id") as f:
                p = int(f.read())
            with open(base + "core_id") as f:
                c = int(f.read())
        except (OSError, ValueError):
            break
        cores.add((p, c))
        cpu += 1
    return len(cores) or (os.cpu_count() or 1)


def hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, "fallback of /opt/skills/guides/B200_PROFILING.md"


def h2d_link_probe(step_bytes, dev):
    """Best pinned host-to-device copy rate (GB/s): 5 bursts of 10 copies of
    max(one step's input, 64 MB)."""
    import torch
    hbuf = torch.empty(max(step_bytes, 64 << 20) // 4 + 1, dtype=torch.float32).pin_memory()
    dbuf = torch.empty_like(hbuf, device=dev)
    for _ in range(3):
        dbuf.copy_(hbuf, non_blocking=True)
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best_ms = float("inf")
    for _ in range(5):
        ea.record()
        for _ in range(10):
            dbuf.copy_(hbuf, non_blocking=True)
        eb.record()
        eb.synchronize()
        best_ms = min(best_ms, ea.elapsed_time(eb))
    return 10 * hbuf.numel() * 4 / (best_ms / 1e3) / 1e9


def make_frames(cfg, indices, max_trials=0):
    """Frames of config `cfg` (scene seed = 1000 cfg + index)."""
    from tools import workloads as W
    out = []
    for i in indices:
        if cfg == 2:
            w = W.automotive(seed=1000 + i)
        elif cfg == 3:
            w = W.stress(seed=3000 + i)
        elif cfg == 4:
            w = W.imaging(seed=4000 + i)
        else:
            w = W.single_frame(seed=7 + i)
        if max_trials:
            w.max_trials = max_trials
        out.append(w)
    return out


def batch(frames):
    """Concatenate frames into one CSR call; RNG keys stay frame-local."""
    offs, az, dop, keys = [np.zeros(1, np.int64)], [], [], []
    base = 0
    for w in frames:
        offs.append(w.offsets[1:] + base)
        base += w.n_points
        az.append(w.azimuth)
        dop.append(w.doppler)
        keys.append(np.arange(w.n_clusters, dtype=np.int32))
    return (np.concatenate(offs), np.concatenate(az), np.concatenate(dop), np.concatenate(keys))


def config_desc(cfg, w, args, world):
    """Identical for both arms (the driver compares them)."""
    T = w.max_trials
    names = {1: "single frame: 8 clusters x 128 points, 20%% outliers, T=%d (configs[0])" % T,
             2: "automotive frame: 200 clusters x 64-2048 points (log-uniform), 25%% outliers, "
                "T=%d (configs[1])" % T,
             3: "micro-Doppler stress: automotive shapes, 50%% outliers, T=%d, "
                "threshold_scale 0.25 (configs[2])" % T,
             4: "imaging frame: 5000 clusters, 1M points (n_i ~ U[50,350]), 25%% outliers, "
                "T=%d (configs[3]: the largest single-GPU configuration)" % T}
    resident_mb = w.n_points * 16 * args.resident_frames / 1e6
    return {"workload": names[cfg], "clusters_per_frame": w.n_clusters,
            "points_per_frame": w.n_points, "max_trials": T,
            "threshold_scale": w.threshold_scale, "frames_per_step": args.frames_per_step,
            "resident_frames_per_rank": args.resident_frames,
            "l2": "inputs larger than L2: steps cycle through %d resident frames "
                  "(~%.0f MB of f64 azimuth/doppler per rank > 126 MB L2)"
                  % (args.resident_frames, resident_mb),
            "parallelism": f"frame shards x{world} (weak, no data-path collective)",
            "rng_seed": w.rng_seed}


class ClockSampler:
    """Polls SM clock + throttle reasons through NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def fp32_peak(torch, stream):
    """In-run FP32 FMA-pipe peak (MEASURED_PEAKS.json has no FP32 entry)."""
    from paper_2012_12618_b200 import _native
    lib = _native.probe()
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(256, device="cuda")
    best = {}
    for kind, name in ((0, "ffma2"), (1, "ffma")):
        blocks, iters = n_sm * 8, 20000
        for _ in range(2):
            lib.rvk_probe_fp32(kind, blocks, 200, out.data_ptr(), C.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            a.record(stream)
            lib.rvk_probe_fp32(kind, blocks, iters, out.data_ptr(), C.c_void_p(stream.cuda_stream))
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        best[name] = lib.rvk_probe_flops(blocks, iters) / min(ts) / 1e12
    return max(best.values()), best, n_sm


# --------------------------------------------------------------- CPU arms

def _median_time(fn, reps, warmups):
    """src/bench.cpp:68-87: median of `reps` after `warmups`."""
    for _ in range(warmups):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def _prefix(w, k):
    off = w.offsets[:k + 1]
    return off, w.azimuth[:off[-1]], w.doppler[:off[-1]]


def _sized_prefix(run_k, w, T, rep_budget_s):
    """Largest cluster prefix of frame w whose one run fits rep_budget_s."""
    k = w.n_clusters
    dt = run_k(k)
    if dt <= rep_budget_s:
        return k, dt
    rate = int(w.offsets[k]) * T / dt
    want_points = rep_budget_s * rate / T
    k = max(1, min(w.n_clusters, int(np.searchsorted(w.offsets, want_points))))
    return k, run_k(k)


def cpu_baseline(w, p, budget_s, reps=20, warmups=3):
    """The reference's CPU path on the box's host cores, on frame w:
    run_ransac + estimate_all with all logical cores, and the 1-core
    sequential_ransac + sequential_lsq (src/baseline.cpp:11-79); median of
    `reps` after `warmups` each (src/bench.cpp:68-87), on the whole frame or the
    largest cluster prefix that keeps each arm inside half the budget."""
    from oracle.binding import REF_SO, Oracle, Reference, make_params
    mp = make_params(p.max_trials, p.threshold_scale, p.rng_seed)
    logical = os.cpu_count() or 1
    phys = physical_cores()
    per_rep = budget_s / 2 / (reps + warmups)
    out = {"unit": UNIT, "cores_logical": logical, "cores_physical": phys,
           "reps": reps, "warmups": warmups}
    if os.path.exists(REF_SO):
        ref = Reference()

        def par(k):
            off, az, dop = _prefix(w, k)
            t0 = time.perf_counter()
            ref.ransac_estimate(off, az, dop, mp, workers=logical)
            return time.perf_counter() - t0

        def seq(k):
            off, az, dop = _prefix(w, k)
            t0 = time.perf_counter()
            r = ref.sequential_ransac(off, az, dop, mp)
            ref.sequential_lsq(off, az, dop, r.mask)
            return time.perf_counter() - t0
        kind = "reference"
    else:  # the C restatement (single-threaded) where the reference was never built
        ref = Oracle()

        def par(k):
            off, az, dop = _prefix(w, k)
            t0 = time.perf_counter()
            ref.ransac_estimate_range(off, az, dop, mp, 0, k)
            return time.perf_counter() - t0
        seq = par
        kind, logical = "port", 1
    kp, _ = _sized_prefix(par, w, p.max_trials, per_rep)
    tp = _median_time(lambda: par(kp), reps, warmups)
    ks, _ = _sized_prefix(seq, w, p.max_trials, per_rep)
    ts = _median_time(lambda: seq(ks), reps, warmups)
    ev_p = int(w.offsets[kp]) * p.max_trials
    ev_s = int(w.offsets[ks]) * p.max_trials

    def desc(k):
        if k == w.n_clusters:
            return "the whole frame"
        return f"the first {k} of {w.n_clusters} clusters ({int(w.offsets[k])} points)"
    out.update({"value": ev_p / tp, "cores": logical, "kind": kind,
                "sample": f"{desc(kp)} of one frame ({ev_p / 1e6:.1f} M evals), "
                          f"rvk::run_ransac + estimate_all, workers={logical}, "
                          f"median of {reps} after {warmups} warm-ups",
                "sequential_1core": {"value": ev_s / ts, "unit": UNIT, "cores": 1,
                                     "sample": f"{desc(ks)} ({ev_s / 1e6:.1f} M evals), "
                                               "sequential_ransac + sequential_lsq, "
                                               f"median of {reps} after {warmups} warm-ups"}})
    return out


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on the same
    step as our arm -- frames_per_step frames, each through rvk::run_ransac +
    estimate_all with all host threads -- rank 0 only. Frames come from the
    reference's own generate_frame (oracle/_ref), so this arm maps no repo
    library; config 3's 50% outliers are beyond generate_frame's check
    (scene.cpp:39), so that config uses tools/rvk_scene.c."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if args.config == 5:
        print(json.dumps({"impl": "reference", "unavailable":
                          "config 5 (multi-GPU frame stream) has no CPU-reference arm; "
                          "run bench.py --impl reference --config 2 for its per-frame rate"}))
        return
    from tools import workloads as W
    from oracle.binding import REF_SO, Oracle, Reference, make_params
    if args.config != 3:
        W.set_generator("reference")
    B = args.frames_per_step
    frames = make_frames(args.config, range(B), args.max_trials)
    w0 = frames[0]
    T, scale, seed = w0.max_trials, w0.threshold_scale, w0.rng_seed
    mp = make_params(T, scale, seed)
    cores = os.cpu_count() or 1
    kind = "reference" if os.path.exists(REF_SO) else "port"
    cpu = Reference() if kind == "reference" else Oracle()
    workers = cores if kind == "reference" else 1

    def run(f, k):
        off, az, dop = _prefix(f, k)
        if kind == "reference":
            cpu.ransac_estimate(off, az, dop, mp, workers=workers)
        else:
            cpu.ransac_estimate_range(off, az, dop, mp, 0, k)
        return int(off[-1]) * T

    # the whole step when (warmup + steps) x step fits ~150 s, else the same
    # cluster fraction of every frame (stated in the line)
    t0 = time.perf_counter()
    run(w0, w0.n_clusters)
    est_step = (time.perf_counter() - t0) * B
    k_frac = min(1.0, 150.0 / max(1e-9, est_step * (args.steps + args.warmup)))
    ks = [max(1, int(round(f.n_clusters * k_frac))) for f in frames]
    ev_total, t_total, step_ms = 0, 0.0, []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ev = sum(run(f, k) for f, k in zip(frames, ks))
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            ev_total += ev
            t_total += dt
            step_ms.append(dt * 1e3)
    value = ev_total / t_total
    whole = all(k == f.n_clusters for f, k in zip(frames, ks))
    sample = (f"per step: {B} frames, " +
              ("every cluster" if whole else
               f"the first {ks[0]} of {w0.n_clusters} clusters of each") +
              f" (rvk::run_ransac + estimate_all, workers={workers}; frames from " +
              ("oracle/_ref generate_frame)" if args.config != 3 else "tools/rvk_scene.c)"))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(step_ms), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_frame recipe)",
            "config": config_desc(args.config, w0, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
                             "cores_logical": cores, "cores_physical": physical_cores(),
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm

def load_capture(cfg, T):
    """Per-launch DRAM bytes of the committed `ncu --set full` capture of this
    configuration (profiles/ncu_capture.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_capture.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"config{cfg}_T{T}")
    except (OSError, ValueError):
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == 5:
        from tools import stream_bench
        stream_bench.run(args)
        return
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        # one rank per GPU (ranks beyond the device count share devices: only
        # for functional runs of the multi-rank path on a smaller box)
        torch.cuda.set_device(local % torch.cuda.device_count())
        backend = os.environ.get("RVK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2012_12618_b200 as rvk
    from paper_2012_12618_b200 import _native
    lib = _native.gpu()

    # ---- resident frames (distinct per rank)
    F = args.resident_frames
    B = args.frames_per_step
    n_batches = max(1, F // B)
    frames = make_frames(args.config, range(rank * F, rank * F + n_batches * B), args.max_trials)
    w0 = frames[0]
    p = rvk.RansacParams(w0.max_trials, w0.threshold_scale, w0.rng_seed)
    batches = []
    for j in range(n_batches):
        off, az, dop, keys = batch(frames[j * B:(j + 1) * B])
        d = {"offsets": torch.from_numpy(off).to(dev), "az": torch.from_numpy(az).to(dev),
             "dop": torch.from_numpy(dop).to(dev), "keys": torch.from_numpy(keys).to(dev),
             "C": off.size - 1, "P": int(off[-1]), "evals": int(off[-1]) * p.max_trials}
        batches.append(d)
    Cmax = max(b["C"] for b in batches)
    Pmax = max(b["P"] for b in batches)
    S = max(1, args.streams)
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]
    outs = [{"inlier_count": torch.zeros(Cmax, dtype=torch.int32, device=dev),
             "winning_trial": torch.zeros(Cmax, dtype=torch.int32, device=dev),
             "mask": torch.zeros(Pmax, dtype=torch.uint8, device=dev),
             "est": torch.zeros(Cmax * 48, dtype=torch.uint8, device=dev)} for _ in range(S)]
    stream = streams[0]
    pc = p.c()

    def step(j, si=None):
        """One step (a batch of frames) on stream j % S (or stream si)."""
        si = j % S if si is None else si
        b = batches[j % n_batches]
        out = outs[si]
        st = lib.rvk_ransac_estimate_device(
            0, b["C"], b["P"], b["offsets"].data_ptr(), b["az"].data_ptr(), b["dop"].data_ptr(),
            None, C.addressof(pc), b["keys"].data_ptr(), out["inlier_count"].data_ptr(),
            out["winning_trial"].data_ptr(), out["mask"].data_ptr(), out["est"].data_ptr(),
            C.c_void_p(streams[si].cuda_stream))
        if st != 0:
            raise RuntimeError(lib.rvk_last_error().decode())
        return b["evals"], b["C"]

    peak, peaks, n_sm = fp32_peak(torch, stream)

    for j in range(args.warmup):
        step(j)
    torch.cuda.synchronize()

    # ---- timed region
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    lib.rvk_reset_kernel_launches()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    s_end = [torch.cuda.Event() for _ in range(S)]
    evals = clusters = 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        t_start.record(streams[0])
        for s_ in streams[1:]:
            s_.wait_event(t_start)
        for j in range(args.steps):
            e, c = step(args.warmup + j)
            evals += e
            clusters += c
        for si, s_ in enumerate(streams):
            s_end[si].record(s_)
            streams[0].wait_event(s_end[si])
        t_end.record(streams[0])
        t_end.synchronize()
        torch.cuda.synchronize()
    launches = lib.rvk_kernel_launches()
    elapsed = t_start.elapsed_time(t_end) / 1e3

    # isolated single-stream pass: per-step latency and per-stage durations
    # without cross-stream overlap (the rooflines of the kernels)
    n_iso = min(args.steps, 40)
    lib.rvk_profile_enable(1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_iso + 1)]
    iso_evals = iso_points = iso_clusters = 0
    ev[0].record(stream)
    for j in range(n_iso):
        e, c = step(j, 0)
        iso_evals += e
        iso_clusters += c
        iso_points += batches[j % n_batches]["P"]
        ev[j + 1].record(stream)
    ev[-1].synchronize()
    lib.rvk_profile_enable(0)
    stage_ms = (C.c_double * 4)()
    stage_n = (C.c_int64 * 4)()
    lib.rvk_profile_read(stage_ms, stage_n, 4)
    per_step = [ev[j].elapsed_time(ev[j + 1]) for j in range(n_iso)]

    # single-frame latency: device-resident (CUDA events) and host -> host
    # through the public API (pinned buffers: H2D, kernels, D2H of every output)
    f_off, f_az, f_dop, f_keys = batch(frames[:1])
    one = {"offsets": torch.from_numpy(f_off).to(dev), "az": torch.from_numpy(f_az).to(dev),
           "dop": torch.from_numpy(f_dop).to(dev), "keys": torch.from_numpy(f_keys).to(dev)}
    frame_lat = []
    for j in range(args.latency_reps + 3):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        lib.rvk_ransac_estimate_device(
            0, f_off.size - 1, int(f_off[-1]), one["offsets"].data_ptr(), one["az"].data_ptr(),
            one["dop"].data_ptr(), None, C.addressof(pc), one["keys"].data_ptr(),
            outs[0]["inlier_count"].data_ptr(), outs[0]["winning_trial"].data_ptr(),
            outs[0]["mask"].data_ptr(), outs[0]["est"].data_ptr(), C.c_void_p(stream.cuda_stream))
        b_.record(stream)
        b_.synchronize()
        if j >= 3:
            frame_lat.append(a.elapsed_time(b_))
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    h_off, h_az, h_dop = pin(f_off), pin(f_az), pin(f_dop)
    Cf, Pf = f_off.size - 1, int(f_off[-1])
    h_cnt, h_tr = pin(np.zeros(Cf, np.int32)), pin(np.zeros(Cf, np.int32))
    h_mask, h_est = pin(np.zeros(Pf, np.uint8)), np.zeros(Cf, _native.ESTIMATE_DTYPE)
    e2e_lat = []
    for j in range(args.latency_reps + 3):
        t1 = time.perf_counter()
        st = lib.rvk_ransac_estimate(0, Cf, h_off.ctypes.data, h_az.ctypes.data,
                                     h_dop.ctypes.data, None, C.addressof(pc), None,
                                     h_cnt.ctypes.data, h_tr.ctypes.data, h_mask.ctypes.data,
                                     h_est.ctypes.data)
        if st != 0:
            raise RuntimeError(lib.rvk_last_error().decode())
        if j >= 3:
            e2e_lat.append((time.perf_counter() - t1) * 1e3)

    if world > 1:
        import torch.distributed as dist
        rdev = dev if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([elapsed], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        tot = torch.tensor([evals, clusters], device=rdev, dtype=torch.float64)
        dist.all_reduce(tot)
        evals_all, clusters_all = float(tot[0]), float(tot[1])
    else:
        evals_all, clusters_all = float(evals), float(clusters)

    # ---- rooflines. Stage ids (rvk_profile_read): 0 = prep (normalize,
    # median, MAD, hypotheses: the ingest), 1 = a fused warp-per-cluster
    # kernel (the whole path for calls of at most one small-cluster frame,
    # e.g. config 1; prep + score for batches of small clusters at T <= 512,
    # e.g. config 4), 2 = score, 3 = select + refit.
    fused = stage_n[1] > 0 and stage_ms[1] > stage_ms[2]
    sc = 1 if fused else 2
    whole_path = fused and stage_ms[3] < 0.05 * stage_ms[1]
    score_ms = stage_ms[sc] / max(1, stage_n[sc])
    evals_per_launch = iso_evals / max(1, stage_n[sc])
    achieved = evals_per_launch * FLOP_PER_EVAL / (score_ms / 1e3) / 1e12
    clk = clk.summary()
    sm_max = clk.get("sm_max_mhz") or 1965
    nominal = n_sm * 128 * 2 * sm_max * 1e6 / 1e12
    cap = load_capture(args.config, w0.max_trials) or {}
    total_ms = sum(stage_ms)
    kname = ("fused_warp_kernel (whole path, scoring inside)" if whole_path else
             "fused_warp_kernel<prep + score> (normalize, median, MAD, hypotheses and the "
             "FFMA2 scoring loop in one warp per cluster)" if fused else "score_kernel")
    roofline = {"bound": "fp32", "kernel": kname, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": "in-run FP32 FMA-pipe probe (max of FFMA2 %.1f / FFMA %.1f "
                               "TFLOP/s); MEASURED_PEAKS.json has no FP32 entry"
                               % (peaks["ffma2"], peaks["ffma"]),
                "frac_of_nominal": achieved / nominal, "nominal_peak": nominal,
                "flop_per_eval": FLOP_PER_EVAL, "evals_per_launch": evals_per_launch,
                "avg_launch_ms": score_ms,
                "traffic": cap.get("fused" if fused else "score", {}).get("dram_bytes"),
                "traffic_source": cap.get("source"),
                "share_of_step": stage_ms[sc] / total_ms if total_ms else None,
                "stage_ms_per_step": {"prep_ingest": stage_ms[0] / n_iso,
                                      "fused_prep_score_or_whole": stage_ms[1] / n_iso,
                                      "score": stage_ms[2] / n_iso,
                                      "select_refit": stage_ms[3] / n_iso},
                "measured": "isolated single-stream pass (%d steps) right after the timed "
                            "region, CUDA events around each stage's launches" % n_iso}
    hbm, hbm_src = hbm_peak()

    def hbm_line(kernel, stage, b_pt, b_cl, ncu_key):
        ms = stage_ms[stage] / max(1, n_iso)
        byts = (iso_points * b_pt + iso_clusters * b_cl) / max(1, n_iso)
        ach = byts / (ms / 1e3) / 1e9 if ms > 0 else None
        return {"bound": "hbm", "kernel": kernel, "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm if ach else None, "peak_source": hbm_src,
                "algorithmic_bytes_per_step": byts,
                "bytes_model": f"{b_pt:g} B/point + {b_cl} B/cluster (SURVEY.md 8(d))",
                "avg_ms_per_step": ms,
                "traffic": cap.get(ncu_key, {}).get("dram_bytes")}
    roofline["hbm"] = None if whole_path else {
        "ingest": hbm_line("fused prep + score kernel: the ingest shares the kernel (and its "
                           "time) with the scoring loop, so this is a lower bound of the "
                           "ingest rate", 1, INGEST_B_PT, INGEST_B_CL, "fused")
        if fused else hbm_line("prep kernels (normalize, median, MAD, hypotheses)", 0,
                               INGEST_B_PT, INGEST_B_CL, "prep"),
        "refit": hbm_line("select kernel (exact winner, mask, LSQ refit + heading)", 3,
                          REFIT_B_PT, REFIT_B_CL, "select")}

    # ---- e2e through the public host API (pinned host buffers, H2D + D2H per
    # step), on every rank at once
    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def reduce_max_sum(t, n):
        if world == 1:
            return t, n
        import torch.distributed as dist
        rdev = dev if dist.get_backend() == "nccl" else "cpu"
        v = torch.tensor([t], device=rdev, dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        c = torch.tensor([float(n)], device=rdev, dtype=torch.float64)
        dist.all_reduce(c)
        return float(v.item()), float(c.item())

    hb = []
    for j in range(min(n_batches, 4)):
        off, az, dop, keys = batch(frames[j * B:(j + 1) * B])
        hb.append((pin(off), pin(az), pin(dop), pin(keys)))
    C_ = hb[0][0].size - 1
    P_ = int(hb[0][0][-1])
    h2d = (C_ + 1) * 8 + 2 * P_ * 8 + 2 * C_ * 4  # offsets, az, dop, keys, cluster ids
    # counts, trials, estimates, mask bits (rvk_stream_submit_packed: 1 bit/pt)
    d2h = C_ * 4 * 2 + C_ * 48 + (P_ + 7) // 8
    depth = 3
    outsets = [(pin(np.zeros(Cmax, np.int32)), pin(np.zeros(Cmax, np.int32)),
                pin(np.zeros((Pmax + 7) // 8, np.uint8)), np.zeros(Cmax, _native.ESTIMATE_DTYPE))
               for _ in range(depth)]
    fs = rvk.FrameStream(p, depth=depth)

    def stream_run(n):
        tickets, ev_ = [], 0
        for j in range(n):
            off, az, dop, keys = hb[j % len(hb)]
            nc, npt = off.size - 1, int(off[-1])
            o = outsets[j % depth]
            tickets.append(fs.submit(off, az, dop, frame_id=j, rng_cluster_index=keys,
                                     out=(o[0][:nc], o[1][:nc], o[2][:(npt + 7) // 8],
                                          o[3][:nc]), packed_mask=True))
            ev_ += npt * p.max_trials
        for t in tickets:
            fs.wait(t)
        return ev_

    h2d_probe_gbs = h2d_link_probe(h2d, dev)
    stream_run(len(hb) + depth)  # every batch through every slot: buffers sized
    barrier()  # all ranks stream concurrently; the job time is the slowest rank's
    t0 = time.perf_counter()
    e2e_evals = stream_run(args.e2e_steps)
    e2e_t = time.perf_counter() - t0
    fs.close()
    e2e_t, e2e_evals = reduce_max_sum(e2e_t, e2e_evals)
    h2d_peak = max(h2d_probe_gbs, h2d_link_probe(h2d, dev))
    h2d_ach = h2d / (e2e_t / args.e2e_steps) / 1e9
    e2e = {"value": e2e_evals / e2e_t, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_t * 1e3 / args.e2e_steps,
           "api": "FrameStream / rvk_stream_submit_packed+wait (pinned host buffers, masks "
                  "as bits, depth %d: H2D of step k+1 overlaps the kernels of step k)" % depth,
           "roofline": {"bound": "pcie_h2d" if h2d_ach / h2d_peak > 0.8 else
                                 "device (kernels; the H2D of the next step overlaps)",
                        "achieved": h2d_ach, "peak": h2d_peak,
                        "unit": "GB/s", "frac": h2d_ach / h2d_peak,
                        "peak_source": "in-run pinned H2D copy bandwidth, best of 5 bursts "
                                       "of 10 copies of max(step input, 64 MB), probed "
                                       "before and after the e2e run"},
           "note": "all %d ranks concurrently: evals summed over ranks / the slowest rank's "
                   "wall time" % world}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(w0, p, args.cpu_seconds)
        result = {
            "metric": METRIC, "value": evals_all / elapsed, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 scoring + f64 exact decisions/refit",
            "data": "synthetic (generate_frame recipe, KeyedRng; no network datasets)",
            "config": config_desc(args.config, w0, args, world),
            "clusters_per_sec": clusters_all / elapsed,
            "p50_step_latency_ms": statistics.median(per_step),
            "p50_frame_latency_ms": statistics.median(frame_lat),
            "p50_frame_latency_e2e_ms": statistics.median(e2e_lat),
            "frame_latency_note": "one frame per call, p50 of %d: device-resident inputs with "
                                  "CUDA events (p50_frame_latency_ms); host -> host through "
                                  "rvk_ransac_estimate with pinned buffers, wall clock, H2D "
                                  "of the f64 input and D2H of counts, trials, mask and "
                                  "estimates included (p50_frame_latency_e2e_ms)"
                                  % args.latency_reps,
            "streams": S, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
