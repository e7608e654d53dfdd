timeout 300 python tools/fused_check.py --var RVK_PAIR --a 1 --b 0 | grep -E "cfg4|mixed|cfg1"
for v in 1 0; do for T in 256 1024; do echo "== pair=$v T=$T"; RVK_PAIR=$v timeout 300 python bench.py --max-trials $T --no-cpu-baseline --e2e-steps 4 --latency-reps 10 2>/dev/null | tail -1 > /tmp/b.json; python tools/summarize_bench.py /tmp/b.json | cut -c1-230; done; done
