timeout 300 python tools/fused_check.py --var RVK_PREP_SCORE --a 1 --b 0 | grep -E "cfg4|cfg1|mixed"
for T in 256 1024; do echo "== T=$T"; RVK_PREP_SCORE=1 timeout 300 python bench.py --max-trials $T --no-cpu-baseline --e2e-steps 4 --latency-reps 20 2>/dev/null | tail -1 > /tmp/b.json; python tools/summarize_bench.py /tmp/b.json; done
