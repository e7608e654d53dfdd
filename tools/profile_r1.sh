#!/bin/bash
# One-GPU ncu captures for the round-1 profiles (run under gpurun).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 2 --no-cpu-baseline \
    --frames-per-step 8 --e2e-steps 2 > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 3 -c 1 \
    -o gpurun_out/prof_score python bench.py --steps 2 --warmup 2 --no-cpu-baseline \
    --frames-per-step 8 --e2e-steps 1 > gpurun_out/ncu_score.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:prep_kernel -s 3 -c 1 \
    -o gpurun_out/prof_prep python bench.py --steps 2 --warmup 2 --no-cpu-baseline \
    --frames-per-step 8 --e2e-steps 1 > gpurun_out/ncu_prep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 3 -c 1 \
    -o gpurun_out/prof_select python bench.py --steps 2 --warmup 2 --no-cpu-baseline \
    --frames-per-step 8 --e2e-steps 1 > gpurun_out/ncu_select.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_mb -s 1 -c 1 \
    -o gpurun_out/prof_mb ./tools/score_mb > gpurun_out/ncu_mb.log 2>&1
