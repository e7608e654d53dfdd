"""profiles/ncu_capture.json from `ncu --set full` reports of one bench step per
configuration (tools/profile_r2.sh): per kernel, DRAM bytes, duration, pipe
activity and issue rate, normalized to bytes / microseconds.

    python tools/ncu_capture.py gpurun_out/r2_c4_t256.ncu-rep:4:256 ... > profiles/ncu_capture.json
"""
import csv
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6, "%": 1, "": 1}
KEYS = {"dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "gpu__time_duration.sum": "duration_us",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_pct",
        "smsp__warps_active.avg.per_cycle_active": "warps_per_smsp",
        "launch__registers_per_thread": "registers"}


def role(name):
    if "fused_warp" in name:
        return "fused"
    if "score_kernel" in name:
        return "score"
    if "prep" in name:
        return "prep"
    if "select" in name:
        return "select"
    return name


def parse(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        k = {}
        for m, name in KEYS.items():
            try:
                k[name] = float(d[m].replace(",", "")) * SCALE.get(u.get(m, ""), 1)
            except (KeyError, ValueError):
                pass
        k["dram_bytes"] = k.get("dram_read", 0) + k.get("dram_write", 0)
        r = role(d.get("Kernel Name", ""))
        prev = res.get(r)
        if prev:  # e.g. prep_warp + prep_hyp: one stage, summed
            for f in ("dram_read", "dram_write", "dram_bytes", "duration_us"):
                prev[f] = prev.get(f, 0) + k.get(f, 0)
            prev["kernels"].append(d.get("Kernel Name", "")[:80])
        else:
            k["kernels"] = [d.get("Kernel Name", "")[:80]]
            res[r] = k
    return res


def main():
    cap = {}
    for spec in sys.argv[1:]:
        rep, cfg, T = spec.split(":")
        d = parse(rep)
        d["source"] = ("ncu --set full --clock-control none, one bench step (16 frames, "
                       "tools/one_call.py) -- %s" % rep.split("/")[-1])
        cap[f"config{cfg}_T{T}"] = d
    print(json.dumps(cap, indent=1))


if __name__ == "__main__":
    main()
