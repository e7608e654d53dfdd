#!/bin/bash
# Quick iteration: selected gpu tests + bench (config given as $2, default 2).
TAG=${1:-it}; CFG=${2:-2}; TESTS=${3:-tests}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest $TESTS -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --config $CFG --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 120 python tools/e2e_trace.py > $O/e2e_trace.log 2>&1
