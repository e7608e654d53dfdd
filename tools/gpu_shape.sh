#!/bin/bash
TAG=${1:-sh}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for cfg in "4 32 512" "4 64 512" "4 128 512" "4 128 1024" "2 256 2048" "2 128 1024"; do
  set -- $cfg
  RVK_PREP_THREADS=$2 RVK_PREP_CAP=$3 timeout 300 python bench.py --config $1 --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/bench_c$1_t$2_cap$3.json 2>> $O/bench.err
done
