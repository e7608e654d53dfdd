#!/bin/bash
# warp-select A/B: .so variants in lib/ab on config 4, plus the CTA select
TAG=${1:-sw}; O=gpurun_out/$TAG; mkdir -p $O; L=paper_2012_12618_b200/lib
cp $L/librvk_gpu.so $L/ab/_orig.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "warp_select or cta_select" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for v in $L/ab/sw*.so; do
    n=$(basename $v .so); cp $v $L/librvk_gpu.so
    timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 60 --e2e-steps 3 > $O/${n}_c4_r$r.json 2>> $O/err.log
  done
  RVK_SELECT_WARP=0 timeout 300 python bench.py --config 4 --no-cpu-baseline --steps 60 --e2e-steps 3 > $O/cta_c4_r$r.json 2>> $O/err.log
done
cp $L/ab/_orig.so $L/librvk_gpu.so
