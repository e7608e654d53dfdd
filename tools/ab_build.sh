# Variant builds of librvk_gpu.so for A/B timing (development helper):
#   tools/ab_build.sh NAME -DFLAG=V ...  ->  paper_2012_12618_b200/lib/ab_NAME.so
#   RVK_GPU_SO=paper_2012_12618_b200/lib/ab_NAME.so python bench.py ...
set -e
name=$1; shift
cd "$(dirname "$0")/.."
C=paper_2012_12618_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared \
  "$@" -I include -o paper_2012_12618_b200/lib/ab_$name.so $C/rvk_kernels.cu $C/rvk_dbscan.cu $C/rvk_capi.cu
echo paper_2012_12618_b200/lib/ab_$name.so
