"""Prints the key numbers of bench.py JSON lines (development helper)."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            if "Error" in line or "error" in line:
                print(f, line.strip()[:300])
            continue
        d = json.loads(line)
        r = d.get("roofline", {})
        st = {k: round(v, 4) for k, v in r.get("stage_ms_per_step", {}).items()}
        print(f"{f}: value {d['value']:.3e} ms/step {d['ms_per_step']:.4f} "
              f"e2e {d.get('e2e', {}).get('value', 0):.3e} frac {r.get('frac', 0):.3f} "
              f"live_score_ms {r.get('live_avg_launch_ms', 0):.4f} stages {st} "
              f"p50 frame {d.get('p50_frame_latency_ms', 0):.4f} ms clk {d.get('clocks', {}).get('sm_mhz')} "
              f"cfg fps={d['config'].get('frames_per_step')} streams={d.get('streams')}")
