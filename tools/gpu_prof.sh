#!/bin/bash
# ncu --set full with source of the pipeline kernels on one config.
# Usage: bash tools/gpu_prof.sh TAG CONFIG [kernel-regex]
TAG=${1:-prof}; C=${2:-2}; K=${3:-"prep_hyp|prep_warp|select_kernel|score_kernel"}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"$K" -s 6 -c 4 \
    -o $O/prof_c$C python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline \
    --streams 1 --e2e-steps 1 --resident-frames 16 > $O/ncu_c$C.log 2>&1
echo done > $O/DONE
