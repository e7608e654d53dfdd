#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 5 --frames-per-step 16 > gpurun_out/bench_f16.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 5 --streams 3 > gpurun_out/bench_s3.json 2>> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"prep_hyp_kernel|select_kernel" -s 4 -c 2 \
    -o gpurun_out/prof_pipe python bench.py --steps 2 --warmup 2 --no-cpu-baseline \
    --streams 1 --e2e-steps 1 > gpurun_out/ncu_pipe.log 2>&1
