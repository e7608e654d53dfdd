# Round-2 capture (run on the GPU box from the repo root):
#   launch list of the default bench command + ncu --set full of one bench
#   step (16 frames) per configuration. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_gpu_parity.py -m gpu -x -q -k "cli or bench_harness or too_small or packed or multi" > gpurun_out/r2d_pytest.log 2>&1; tail -3 gpurun_out/r2d_pytest.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 2 --latency-reps 3 > gpurun_out/r2_launches_bench.log 2>&1
for spec in "4 256" "4 1024" "2 0" "3 0"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"prep_warp|prep_hyp|score_kernel|select_warp|select_kernel|fused_warp" -c 5 \
    -o gpurun_out/r2_c$1_t$2 python tools/one_call.py --config $1 --frames 16 --max-trials $2 --reps 1 \
    > gpurun_out/r2_c$1_t$2.log 2>&1
done
ls gpurun_out
