#!/bin/bash
TAG=${1:-sh}; O=gpurun_out/$TAG; mkdir -p $O
for cfg in "2 256 2048" "2 128 2048" "2 64 2048"; do
  set -- $cfg
  RVK_PREP_THREADS=$2 RVK_PREP_CAP=$3 timeout 300 python bench.py --config $1 --no-cpu-baseline --steps 100 --e2e-steps 5 > $O/bench_c$1_t$2_cap$3.json 2>> $O/bench.err
done
for t in 64 128 256; do
  RVK_SELECT_THREADS=$t timeout 300 python bench.py --config 2 --no-cpu-baseline --steps 100 --e2e-steps 5 > $O/bench_c2_sel$t.json 2>> $O/bench.err
done
