#!/bin/bash
mkdir -p gpurun_out
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" > gpurun_out/pcie.txt
for cs in 0 1; do
for cfg in "262144 4" "1048576 1" "131072 8"; do
  set -- $cfg
  echo "== copy_stream $cs chunk $1 max $2" >> gpurun_out/e2e_trace.log
  RVK_COPY_STREAM=$cs RVK_TRACE=1 RVK_PIPE_CHUNK=$1 RVK_PIPE_MAX=$2 timeout 300 python tools/e2e_trace.py >> gpurun_out/e2e_trace.log 2>&1
done; done
