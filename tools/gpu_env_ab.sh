#!/bin/bash
# A/B of runtime knobs: each argument after the tag is "name:ENV=V ENV2=V2";
# configs from $AB_CONFIGS (default "2"), 2 interleaved rounds.
TAG=$1; shift; O=gpurun_out/$TAG; mkdir -p $O
for r in 1 2; do
  for spec in "$@"; do
    n=${spec%%:*}; e=${spec#*:}
    for c in ${AB_CONFIGS:-2}; do
      env $e timeout 300 python bench.py --config $c --no-cpu-baseline --steps 60 --e2e-steps 3 \
          > $O/${n}_c${c}_r$r.json 2>> $O/err.log
    done
  done
done
