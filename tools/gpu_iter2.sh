#!/bin/bash
mkdir -p gpurun_out
for ni in 0 1 2; do
  RVK_SCORE_NI=$ni timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or c3 or radar or full_size or edge" > gpurun_out/pytest_ni$ni.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ni$ni.log
  RVK_SCORE_NI=$ni timeout 600 python bench.py --no-cpu-baseline --e2e-steps 10 > gpurun_out/bench_ni$ni.json 2> gpurun_out/bench_ni$ni.err
done
timeout 900 python tools/e2e_sweep.py > gpurun_out/e2e_sweep.json 2> gpurun_out/e2e_sweep.err
