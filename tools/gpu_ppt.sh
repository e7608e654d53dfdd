#!/bin/bash
TAG=${1:-ppt}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or c3 or full_size or edge" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for c in 2 3 4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 60 --e2e-steps 5 > $O/b_c${c}.json 2>> $O/err.log
done
