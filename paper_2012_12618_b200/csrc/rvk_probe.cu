// FP32-pipe peak probe (measurement tool for bench.py's roofline; not on the
// product path). MEASURED_PEAKS.json has HBM and bf16-tensor peaks only; the
// scoring kernel is bound by the FP32 FMA pipe, so bench.py measures that
// peak in the same run with this kernel: every thread keeps 8 independent
// FFMA2 chains (16 FP32 FMAs per issue), enough ILP to saturate the pipe.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__global__ void __launch_bounds__(256) ffma2_probe(int iters, float seed, float* out) {
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(seed + i + threadIdx.x, seed - i);
  const float2 m = make_float2(0.9999f, 1.0001f);
  const float2 c = make_float2(1e-7f, -1e-7f);
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 1234.5f) out[threadIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) ffma_probe(int iters, float seed, float* out) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + i + threadIdx.x;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], 0.9999f, 1e-7f);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

}  // namespace

extern "C" {

// Launches the probe; FP32 FLOPs issued = blocks * 256 * iters * 32.
// kind 0 = FFMA2 (packed), 1 = scalar FFMA.
int rvk_probe_fp32(int32_t kind, int32_t blocks, int32_t iters, float* d_out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (kind == 0)
    ffma2_probe<<<blocks, 256, 0, s>>>(iters, 1.0f, d_out);
  else
    ffma_probe<<<blocks, 256, 0, s>>>(iters, 1.0f, d_out);
  return static_cast<int>(cudaGetLastError());
}

int64_t rvk_probe_flops(int32_t blocks, int32_t iters) {
  return static_cast<int64_t>(blocks) * 256 * iters * 32;
}

}  // extern "C"
