"""One-screen summary of bench.py JSON lines (development helper).

    python tools/summarize_bench.py gpurun_out/r2e_*.json
"""
import json
import sys


def main():
    for f in sys.argv[1:]:
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            print(f, "unparsable:", e)
            continue
        if d.get("impl") == "reference":
            print(f"{f}: reference {d.get('value', 0):.3e} evals/s, {d.get('ms_per_step', 0):.0f} ms/step,"
                  f" {d.get('cpu_baseline', {}).get('sample', d.get('unavailable'))}")
            continue
        r = d.get("roofline") or {}
        line = f"{f}: value {d['value']:.3e} ms/step {d['ms_per_step']:.3f}"
        if "e2e" in d:
            line += f" e2e {d['e2e']['value']:.3e}"
        if r:
            line += f" score frac {r['frac']:.3f} ({r['achieved']:.1f}/{r['peak']:.1f} TF)"
            st = r.get("stage_ms_per_step", {})
            line += " stages " + " ".join(f"{k}={v:.3f}" for k, v in st.items())
            for k, v in (r.get("hbm") or {}).items():
                if not v:
                    continue
                line += f" {k} {v['achieved']:.0f} GB/s ({v['frac']:.3f})"
        for k in ("p50_frame_latency_ms", "p50_frame_latency_e2e_ms", "frames_per_sec"):
            if k in d:
                line += f" {k}={d[k]:.3f}"
        cpu = d.get("cpu_baseline")
        if cpu:
            line += f" cpu {cpu['value']:.3e} ({cpu['cores']} thr)"
            if cpu.get("sequential_1core"):
                line += f" 1core {cpu['sequential_1core']['value']:.3e}"
        if "clocks" in d:
            line += f" clk {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}"
        print(line)


if __name__ == "__main__":
    main()
