#!/bin/bash
# Iteration call: GPU parity tests, bench, ncu of the pipeline kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"score_kernel|prep_hyp_kernel|select_kernel" -s 6 -c 3 \
    -o gpurun_out/prof_pipe python bench.py --steps 2 --warmup 2 --no-cpu-baseline \
    --streams 1 --e2e-steps 1 > gpurun_out/ncu_pipe.log 2>&1
