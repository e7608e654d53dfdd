#!/bin/bash
TAG=${1:-ct}; O=gpurun_out/$TAG; mkdir -p $O
for k in 3 2; do for st in 2 3; do
  RVK_SCORE_CTAS=$k timeout 300 python bench.py --config 2 --no-cpu-baseline --steps 100 --e2e-steps 5 --streams $st > $O/bench_k${k}_s$st.json 2>> $O/bench.err
done; done
RVK_SCORE_CTAS=2 timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/bench_c4_k2.json 2>> $O/bench.err
RVK_SCORE_CTAS=2 timeout 300 python bench.py --config 3 --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/bench_c3_k2.json 2>> $O/bench.err
