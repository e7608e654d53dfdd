// Accuracy of sincos_az (rvk_device.cuh) against libdevice sincos over the
// azimuth range and beyond (development check, not shipped).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sincos_check tools/sincos_check.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../paper_2012_12618_b200/csrc/rvk_device.cuh"
using namespace rvk_dev;
__device__ unsigned long long ulps(double a, double b) {
  long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
  if (ia < 0) ia = 0x8000000000000000LL - ia;
  if (ib < 0) ib = 0x8000000000000000LL - ib;
  return ia > ib ? ia - ib : ib - ia;
}
__global__ void k(double lo, double hi, long long n, unsigned long long* worst, double* absw) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = lo + (hi - lo) * ((double)i / (double)(n - 1));
    double s, c, s2, c2;
    sincos_az(x, &s, &c);
    sincos(x, &s2, &c2);
    atomicMax(&worst[0], ulps(s, s2));
    atomicMax(&worst[1], ulps(c, c2));
    const double e = fmax(fabs(s - s2), fabs(c - c2));
    atomicMax(reinterpret_cast<unsigned long long*>(absw), __double_as_longlong(e));
  }
}
int main() {
  unsigned long long* w; double* a;
  cudaMallocManaged(&w, 16); cudaMallocManaged(&a, 8);
  const double ranges[][2] = {{-3.141592653589793, 3.141592653589793}, {-4.0, 4.0}, {-1e-3, 1e-3}};
  for (auto& r : ranges) {
    w[0] = w[1] = 0; *a = 0;
    k<<<1184, 256>>>(r[0], r[1], 400000000LL, w, a);
    cudaDeviceSynchronize();
    printf("{\"range\": [%g, %g], \"samples\": 4e8, \"max_ulp_sin\": %llu, \"max_ulp_cos\": %llu, \"max_abs\": %.3e}\n",
           r[0], r[1], w[0], w[1], *a);
  }
  return 0;
}
