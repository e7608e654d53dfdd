#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (both arms, configs 2/3/4),
# ncu launch list and --set full captures of the pipeline kernels.
# Usage: bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
nproc > $O/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in 3 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline \
    --streams 1 --e2e-steps 2 > $O/ncu_launch_bench.log 2>&1
for c in 2 3 4; do
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"score_kernel|prep_hyp|prep_warp|select_kernel|select_warp" -s 6 -c 4 \
      -o $O/prof_c$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline \
      --streams 1 --e2e-steps 1 --resident-frames 16 > $O/ncu_c$c.log 2>&1
done
echo done > $O/DONE
