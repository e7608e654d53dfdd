"""Summarise ncu --set full captures of the pipeline kernels.

    python tools/ncu_extract.py gpurun_out/<tag> [--write-profiles]

Prints per kernel: duration, FMA / ALU pipe activity, issue activity,
occupancy, DRAM bytes; with --write-profiles also updates
profiles/score_kernel_ncu.json (read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        k = {"kernel": d.get("Kernel Name", "")[:60]}
        for m, name in METRICS.items():
            if m in d:
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                if name.startswith("dram") or name == "duration_us":
                    v *= SCALE.get(u.get(m, ""), 1.0)
                k[name] = v
        res.append(k)
    return res


def main():
    d = sys.argv[1]
    write = "--write-profiles" in sys.argv
    prof = {}
    for c in (2, 3, 4):
        rep = os.path.join(d, f"prof_c{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        ks = kernels(rep)
        print(f"== config {c}")
        for k in ks:
            print(json.dumps(k))
        sc = [k for k in ks if "score_kernel" in k["kernel"]]
        if sc:
            k = sc[-1]
            prof[f"config{c}"] = {
                "dram_bytes_per_launch": k.get("dram_read", 0) + k.get("dram_write", 0),
                "fma_pipe_active_pct": k.get("fma_pipe_pct"),
                "alu_pipe_active_pct": k.get("alu_pipe_pct"),
                "issue_active_pct": k.get("issue_pct"),
                "ncu_duration_us": k.get("duration_us"),
                "source": f"ncu --set full --clock-control none, one launch ({os.path.basename(rep)})",
            }
    if write and prof:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "profiles", "score_kernel_ncu.json"), "w") as f:
            json.dump(prof, f, indent=1)
        print("wrote profiles/score_kernel_ncu.json")


if __name__ == "__main__":
    main()
