#!/bin/bash
TAG=${1:-san}; O=gpurun_out/$TAG; mkdir -p $O
for env in ${SAN_ENVS:-"" "RVK_SCORE=tc" "RVK_PREP_WARP=1" "RVK_PREP_WARP=0" "RVK_SCORE_STAGE=lanes"}; do
  for tool in memcheck racecheck synccheck; do
    name=$(echo "${tool}_${env:-default}" | tr '=' '_')
    env $env timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > $O/$name.log 2>&1
    echo "rc=$?" >> $O/$name.log
  done
done
