#!/bin/bash
# Functional check of the multi-rank bench path on one GPU (2 ranks share it, gloo for the
# timing reductions) + the default single-rank bench.
TAG=${1:-mr}; O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 10 > $O/bench1.json 2> $O/bench1.err
RVK_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --e2e-steps 6 --resident-frames 16 > $O/bench2.json 2> $O/bench2.err
echo rc=$? >> $O/bench2.err
