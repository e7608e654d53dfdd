#!/bin/bash
# ncu captures of the four pipeline kernels (one launch each) + launch list.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
    -k regex:"score_kernel|prep_kernel|select_kernel|hyp_kernel" -s 8 -c 4 \
    -o gpurun_out/prof_pipe python bench.py --steps 2 --warmup 2 --no-cpu-baseline \
    --streams 1 --e2e-steps 1 > gpurun_out/ncu_pipe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 2 --no-cpu-baseline \
    --streams 1 --e2e-steps 2 > gpurun_out/ncu_launch_bench.log 2>&1
