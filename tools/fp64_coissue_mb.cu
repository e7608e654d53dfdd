// Can the FP64 pipe score hypotheses alongside the FP32 (FFMA2) loop?
// (development microbenchmark, not shipped)
//
// Production loop per lane: 8 hypotheses (A, B, C, K) x a float4 of two
// points: 3 FFMA2 + 2 LEA.HI per hypothesis and point pair -> the FMA pipe
// caps it at 2/3 of the FP32 peak counted at 4 FLOP/eval. B200 has a
// separate FP64 pipe at half the FP32 rate; if it issues in parallel, KD
// extra hypotheses per lane in FP64 (3 DFMA + 1 LEA.HI per point) add evals
// on an otherwise idle pipe. Reports evals/s per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_coissue_mb tools/fp64_coissue_mb.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int kPairs = 512;  // 1024 points in shared memory

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ float u01(uint32_t x) { return (hsh(x) >> 8) * (1.0f / 16777216.0f); }

template <int KD>
__global__ void __launch_bounds__(256, 3) mb(int reps, uint32_t* out) {
  __shared__ float4 p32[kPairs];
  __shared__ double2 p64[2 * kPairs];
  for (int i = threadIdx.x; i < kPairs; i += blockDim.x) {
    const uint32_t s = blockIdx.x * 7919u + i * 4u;
    const float x0 = u01(s), x1 = u01(s + 1), y0 = u01(s + 2), y1 = u01(s + 3);
    p32[i] = make_float4(x0, x1, y0, y1);
    p64[2 * i] = make_double2(x0, y0);
    p64[2 * i + 1] = make_double2(x1, y1);
  }
  const uint32_t base = (blockIdx.x * 256 + threadIdx.x) * 64u;
  float A[8], B[8];
  float2 Cc[8], T2[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    A[q] = u01(base + 4 * q) - 0.5f;
    B[q] = 0.8f + 0.1f * u01(base + 4 * q + 1);
    const float c = -0.4f * u01(base + 4 * q + 2), t = 0.05f + 0.1f * u01(base + 4 * q + 3);
    Cc[q] = make_float2(c, c);
    T2[q] = make_float2(-t * t, -t * t);
  }
  double DA[KD > 0 ? KD : 1], DB[KD > 0 ? KD : 1], DC[KD > 0 ? KD : 1], DK[KD > 0 ? KD : 1];
#pragma unroll
  for (int q = 0; q < KD; ++q) {
    DA[q] = u01(base + 40 + 4 * q) - 0.5;
    DB[q] = 0.8 + 0.1 * u01(base + 41 + 4 * q);
    DC[q] = -0.4 * u01(base + 42 + 4 * q);
    const double t = 0.05 + 0.1 * u01(base + 43 + 4 * q);
    DK[q] = -t * t;
  }
  uint32_t cnt[8], dcnt[KD > 0 ? KD : 1];
#pragma unroll
  for (int q = 0; q < 8; ++q) cnt[q] = 0;
#pragma unroll
  for (int q = 0; q < KD; ++q) dcnt[q] = 0;
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int i = 0; i < kPairs; i += 2) {
      const float4 v0 = p32[i], v1 = p32[i + 1];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4 v = u ? v1 : v0;
        const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          float2 e = __ffma2_rn(X, make_float2(A[h], A[h]),
                                __ffma2_rn(Y, make_float2(B[h], B[h]), Cc[h]));
          e = __ffma2_rn(e, e, T2[h]);
          cnt[h] += (__float_as_uint(e.x) >> 31) + (__float_as_uint(e.y) >> 31);
        }
      }
      if (KD > 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 q = p64[2 * i + k];
#pragma unroll
          for (int h = 0; h < KD; ++h) {
            double e = fma(DA[h], q.x, fma(DB[h], q.y, DC[h]));
            e = fma(e, e, DK[h]);
            dcnt[h] += static_cast<uint32_t>(__double2hiint(e)) >> 31;
          }
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += cnt[q];
#pragma unroll
  for (int q = 0; q < KD; ++q) s += dcnt[q];
  if (s == 0x12345678u) out[0] = s;
}

template <int KD>
void run(int sms) {
  uint32_t* out;
  CK(cudaMalloc(&out, 4));
  const int blocks = sms * 3, reps = 200;
  mb<KD><<<blocks, 256>>>(2, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int t = 0; t < 3; ++t) {
    cudaEventRecord(a);
    mb<KD><<<blocks, 256>>>(reps, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  const double evals = double(blocks) * 256 * reps * (2.0 * kPairs) * (8 + KD);
  const double ev32 = double(blocks) * 256 * reps * (2.0 * kPairs) * 8;
  printf("{\"fp64_hyps_per_lane\": %d, \"ms\": %.3f, \"evals_per_s\": %.4e, \"fp32_evals_per_s\": %.4e, "
         "\"frac_of_74.4TF_at_4flop\": %.3f}\n",
         KD, best, evals / (best / 1e3), ev32 / (best / 1e3), evals / (best / 1e3) * 4 / 74.4e12);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms);
  run<1>(sms);
  run<2>(sms);
  run<3>(sms);
  run<4>(sms);
  return 0;
}
