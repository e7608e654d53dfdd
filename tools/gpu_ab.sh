#!/bin/bash
# A/B the .so variants in paper_2012_12618_b200/lib/ab/*.so on configs 2-4, interleaved, 2 rounds.
TAG=${1:-ab}; O=gpurun_out/$TAG; mkdir -p $O
cp paper_2012_12618_b200/lib/librvk_gpu.so paper_2012_12618_b200/lib/ab/_orig.so
for r in 1 2; do
  for v in paper_2012_12618_b200/lib/ab/*.so; do
    n=$(basename $v .so); [ "$n" = _orig ] && continue
    cp $v paper_2012_12618_b200/lib/librvk_gpu.so
    for c in 2 3 4; do
      timeout 300 python bench.py --config $c --no-cpu-baseline --steps 60 --e2e-steps 3 > $O/${n}_c${c}_r$r.json 2>> $O/err.log
    done
  done
done
cp paper_2012_12618_b200/lib/ab/_orig.so paper_2012_12618_b200/lib/librvk_gpu.so
if [ -n "$AB_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
fi
