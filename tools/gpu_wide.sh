#!/bin/bash
TAG=${1:-wide}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for w in 1024 999999; do for c in 2 3; do
  RVK_SCORE_WIDE=$w timeout 300 python bench.py --config $c --no-cpu-baseline --steps 60 --e2e-steps 5 > $O/b_c${c}_w$w.json 2>> $O/err.log
done; done
