#!/bin/bash
TAG=${1:-sh}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for c in 2 4; do for t in 64 128 256; do
  RVK_PREP_THREADS=$t RVK_SELECT_THREADS=$t timeout 300 python bench.py --config $c --no-cpu-baseline --steps 50 --e2e-steps 5 > $O/bench_c${c}_t$t.json 2>> $O/bench.err
done; done
