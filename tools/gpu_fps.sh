#!/bin/bash
TAG=${1:-fps}; O=gpurun_out/$TAG; mkdir -p $O
for f in 4 8 16 32; do for s in 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --steps 60 --e2e-steps 10 --frames-per-step $f --streams $s --resident-frames 96 > $O/b_f${f}_s$s.json 2>> $O/err.log
done; done
