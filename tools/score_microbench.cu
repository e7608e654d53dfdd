// Scoring inner-loop microbenchmark (development tool, not shipped).
//
// Measures, on one B200, how fast different instruction mixes evaluate the
// RANSAC inlier test  e = A x + B y + C ; inlier <=> e^2 < T2  and count it,
// with points broadcast from shared memory and NH hypotheses per thread.
// Reports evals/s and the fraction of the FP32 roofline (2 FMA per eval,
// peak measured in-run with an FFMA probe).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o score_mb tools/score_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int kThreads = 128;
constexpr int kPts = 2048;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352d;
  x ^= x >> 15;
  x *= 0x846ca68b;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ float u01(uint32_t x) { return (hsh(x) >> 8) * (1.0f / 16777216.0f); }

// V: 0 = FFMA2 affine + FFMA2 square-compare + LEA.HI
//    1 = FFMA2 affine + scalar FFMA square-compare + LEA.HI
//    2 = scalar FFMA affine + scalar FFMA compare + LEA.HI
//    3 = FFMA2 affine + integer compare on |e| bits (LEA) + LEA.HI
//    4 = FFMA2 affine + FSETP/compare-add (compiler's choice)
//    5 = FFMA2 affine; pair 0 FP compare, pair 1 integer compare (mixed)
//    6 = FFMA2 affine + FSET (|e| < t -> 0/-1) + IADD3 counting two at a time
//    7 = FFMA2 affine + FFMA2 compare, last pair integer compare (f = 1/NP)
//    8 = FFMA2 affine + FSET/IADD3, last pair integer compare
__device__ __forceinline__ uint32_t fset_lt(float a, float b) {
  uint32_t r;
  asm("set.lt.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

template <int V, int NH>
__global__ void __launch_bounds__(kThreads) score_mb(int n, int reps, uint32_t* out) {
  __shared__ float4 pts[kPts / 2];
  for (int i = threadIdx.x; i < kPts / 2; i += blockDim.x) {
    const uint32_t s = blockIdx.x * 7919u + i * 4u;
    pts[i] = make_float4(u01(s), u01(s + 1), u01(s + 2), u01(s + 3));
  }
  constexpr int NP = NH / 2;
  float2 A[NP], B[NP], Cc[NP], T2[NP];
  float Tl[NP];
  uint32_t K[NH];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const uint32_t s = (blockIdx.x * kThreads + threadIdx.x) * 64u + q * 8u;
    A[q] = make_float2(u01(s) - 0.5f, u01(s + 1) - 0.5f);
    B[q] = make_float2(0.8f + 0.1f * u01(s + 2), 0.8f + 0.1f * u01(s + 3));
    Cc[q] = make_float2(-0.4f * u01(s + 4), -0.4f * u01(s + 5));
    const float t = 0.05f + 0.1f * u01(s + 6);
    T2[q] = make_float2(-t * t, -t * t);
    Tl[q] = t;
    K[2 * q] = (__float_as_uint(t) << 1) + 1u;
    K[2 * q + 1] = K[2 * q];
  }
  uint32_t cnt[NH];
#pragma unroll
  for (int q = 0; q < NH; ++q) cnt[q] = 0;
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int i = 0; i < n / 2; ++i) {
      const float4 v = pts[i];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float x = h ? v.z : v.x;
        const float y = h ? v.w : v.y;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (V == 2) {
            const float e0 = __fmaf_rn(A[q].x, x, __fmaf_rn(B[q].x, y, Cc[q].x));
            const float e1 = __fmaf_rn(A[q].y, x, __fmaf_rn(B[q].y, y, Cc[q].y));
            cnt[2 * q] += __float_as_uint(__fmaf_rn(e0, e0, T2[q].x)) >> 31;
            cnt[2 * q + 1] += __float_as_uint(__fmaf_rn(e1, e1, T2[q].y)) >> 31;
          } else {
            const float2 e = __ffma2_rn(A[q], make_float2(x, x),
                                        __ffma2_rn(B[q], make_float2(y, y), Cc[q]));
            const bool fp = (V == 0 || V == 1 || (V == 5 && (q & 1) == 0));
            const bool last = (q == NP - 1);
            if (V == 6 || (V == 8 && !last)) {
              cnt[2 * q] -= fset_lt(fabsf(e.x), Tl[q]) + fset_lt(fabsf(e.y), Tl[q]);
            } else if (V == 7 && !last) {
              const float2 g = __ffma2_rn(e, e, T2[q]);
              cnt[2 * q] += __float_as_uint(g.x) >> 31;
              cnt[2 * q + 1] += __float_as_uint(g.y) >> 31;
            } else if ((V == 7 || V == 8) && last) {
              cnt[2 * q] += ((__float_as_uint(e.x) << 1) - K[2 * q]) >> 31;
              cnt[2 * q + 1] += ((__float_as_uint(e.y) << 1) - K[2 * q + 1]) >> 31;
            } else if (V == 0 || (V == 5 && fp)) {
              const float2 g = __ffma2_rn(e, e, T2[q]);
              cnt[2 * q] += __float_as_uint(g.x) >> 31;
              cnt[2 * q + 1] += __float_as_uint(g.y) >> 31;
            } else if (V == 1) {
              cnt[2 * q] += __float_as_uint(__fmaf_rn(e.x, e.x, T2[q].x)) >> 31;
              cnt[2 * q + 1] += __float_as_uint(__fmaf_rn(e.y, e.y, T2[q].y)) >> 31;
            } else if (V == 3 || V == 5) {
              cnt[2 * q] += ((__float_as_uint(e.x) << 1) - K[2 * q]) >> 31;
              cnt[2 * q + 1] += ((__float_as_uint(e.y) << 1) - K[2 * q + 1]) >> 31;
            } else if (V == 4) {
              cnt[2 * q] += (e.x * e.x < -T2[q].x);
              cnt[2 * q + 1] += (e.y * e.y < -T2[q].y);
            }
          }
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < NH; ++q) s += cnt[q] * (q + 1);
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma_peak(int iters, float* out) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1.0f + i + threadIdx.x;
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], 0.9999f, 1e-7f);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}

// 3-register FFMA (no immediates): coefficients live in registers.
__global__ void __launch_bounds__(256) ffma3_peak(int iters, float m, float c, float* out) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1.0f + i + threadIdx.x;
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], m, c);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345f) out[0] = s;
}

// ALU throughput: LEA.HI-style sign accumulate chains.
__global__ void __launch_bounds__(256) alu_peak(int iters, uint32_t x0, uint32_t* out) {
  uint32_t a[16], c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = x0 * (i + 1) + threadIdx.x;
    c[i] = 0;
  }
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] += (a[i] ^ (k + i)) >> 31;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  out[threadIdx.x] = s;
}

template <class F>
float time_ms(F f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < 3; ++i) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float t;
    CK(cudaEventElapsedTime(&t, a, b));
    best = t < best ? t : best;
  }
  return best;
}

template <int V, int NH>
void run(const char* name, int blocks, double peak_flops, uint32_t* d_out) {
  const int n = kPts, reps = 8;
  const float ms = time_ms([&] { score_mb<V, NH><<<blocks, kThreads>>>(n, reps, d_out); });
  CK(cudaGetLastError());
  const double evals = double(blocks) * kThreads * NH * n * reps;
  const double rate = evals / (ms * 1e-3);
  printf("{\"variant\": \"%s\", \"V\": %d, \"NH\": %d, \"blocks\": %d, \"ms\": %.3f, "
         "\"evals_per_s\": %.4e, \"tflops_4_per_eval\": %.2f, \"frac_of_peak\": %.3f}\n",
         name, V, NH, blocks, ms, rate, rate * 4 / 1e12, rate * 4 / peak_flops);
}

// Correct per-hypothesis counting with a mix of the two compare forms over a
// point pair (v.xy, v.zw): pairs q < NF use the squared FFMA2 compare +
// LEA.HI sign accumulate; pairs q >= NF use FSET(|e| <= t) on both points and
// one IADD3 per hypothesis (cnt - s0 - s1).
template <int NF>
__global__ void __launch_bounds__(256) score_mix(int n, int reps, uint32_t* out) {
  __shared__ float4 pts[kPts / 2];
  for (int i = threadIdx.x; i < kPts / 2; i += blockDim.x) {
    const uint32_t s = blockIdx.x * 7919u + i * 4u;
    pts[i] = make_float4(u01(s), u01(s + 1), u01(s + 2), u01(s + 3));
  }
  constexpr int NP = 4;
  float2 A[NP], B[NP], Cc[NP], K[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const uint32_t s = (blockIdx.x * 256 + threadIdx.x) * 64u + q * 8u;
    A[q] = make_float2(u01(s) - 0.5f, u01(s + 1) - 0.5f);
    B[q] = make_float2(0.8f + 0.1f * u01(s + 2), 0.8f + 0.1f * u01(s + 3));
    Cc[q] = make_float2(-0.4f * u01(s + 4), -0.4f * u01(s + 5));
    const float t = 0.05f + 0.1f * u01(s + 6);
    K[q] = q < NF ? make_float2(-t * t, -t * t) : make_float2(t, t);
  }
  uint32_t cnt[2 * NP];
#pragma unroll
  for (int q = 0; q < 2 * NP; ++q) cnt[q] = 0;
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int i = 0; i < n / 2; ++i) {
      const float4 v = pts[i];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const float2 e0 = __ffma2_rn(A[q], make_float2(v.x, v.x),
                                     __ffma2_rn(B[q], make_float2(v.y, v.y), Cc[q]));
        const float2 e1 = __ffma2_rn(A[q], make_float2(v.z, v.z),
                                     __ffma2_rn(B[q], make_float2(v.w, v.w), Cc[q]));
        if (q < NF) {
          const float2 g0 = __ffma2_rn(e0, e0, K[q]);
          const float2 g1 = __ffma2_rn(e1, e1, K[q]);
          cnt[2 * q] += (__float_as_uint(g0.x) >> 31) + (__float_as_uint(g1.x) >> 31);
          cnt[2 * q + 1] += (__float_as_uint(g0.y) >> 31) + (__float_as_uint(g1.y) >> 31);
        } else {
          uint32_t a0, a1, b0, b1;
          asm("set.le.u32.f32 %0, %1, %2;" : "=r"(a0) : "f"(fabsf(e0.x)), "f"(K[q].x));
          asm("set.le.u32.f32 %0, %1, %2;" : "=r"(a1) : "f"(fabsf(e1.x)), "f"(K[q].x));
          asm("set.le.u32.f32 %0, %1, %2;" : "=r"(b0) : "f"(fabsf(e0.y)), "f"(K[q].y));
          asm("set.le.u32.f32 %0, %1, %2;" : "=r"(b1) : "f"(fabsf(e1.y)), "f"(K[q].y));
          cnt[2 * q] = cnt[2 * q] - a0 - a1;
          cnt[2 * q + 1] = cnt[2 * q + 1] - b0 - b1;
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < 2 * NP; ++q) s += cnt[q] * (q + 1);
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int NF>
void run_mix(const char* name, int blocks, double peak_flops, uint32_t* d_out) {
  const int n = kPts, reps = 8;
  const float ms = time_ms([&] { score_mix<NF><<<blocks, 256>>>(n, reps, d_out); });
  CK(cudaGetLastError());
  const double evals = double(blocks) * 256 * 8 * n * reps;
  const double rate = evals / (ms * 1e-3);
  printf("{\"variant\": \"%s\", \"NF\": %d, \"blocks\": %d, \"ms\": %.3f, "
         "\"evals_per_s\": %.4e, \"tflops_4_per_eval\": %.2f, \"frac_of_peak\": %.3f}\n",
         name, NF, blocks, ms, rate, rate * 4 / 1e12, rate * 4 / peak_flops);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* d_f;
  uint32_t* d_u;
  CK(cudaMalloc(&d_f, 1024));
  CK(cudaMalloc(&d_u, sizeof(uint32_t) * 148 * 64 * kThreads));
  const int pb = sms * 8, iters = 20000;
  const float ms_p = time_ms([&] { ffma_peak<<<pb, 256>>>(iters, d_f); });
  const double peak = double(pb) * 256 * iters * 16 * 2 / (ms_p * 1e-3);
  const float ms_p3 = time_ms([&] { ffma3_peak<<<pb, 256>>>(iters, 0.9999f, 1e-7f, d_f); });
  const double peak3 = double(pb) * 256 * iters * 16 * 2 / (ms_p3 * 1e-3);
  const float ms_a = time_ms([&] { alu_peak<<<pb, 256>>>(iters, 12345u, d_u); });
  const double alu = double(pb) * 256 * iters * 16 / (ms_a * 1e-3);
  printf("{\"sms\": %d, \"ffma_imm_tflops\": %.2f, \"ffma_3reg_tflops\": %.2f, "
         "\"alu_xor_shr_add_gops\": %.1f}\n", sms, peak / 1e12, peak3 / 1e12, alu / 1e9);
  for (int waves : {3, 6}) {
    const int blocks = sms * waves;
    run_mix<4>("mix_sq4_fset0", blocks, peak, d_u);
    run_mix<3>("mix_sq3_fset1", blocks, peak, d_u);
    run_mix<2>("mix_sq2_fset2", blocks, peak, d_u);
    run_mix<1>("mix_sq1_fset3", blocks, peak, d_u);
    run_mix<0>("mix_sq0_fset4", blocks, peak, d_u);
  }
  for (int waves : {6}) {
    const int blocks = sms * waves;
    run<0, 8>("ffma2_all", blocks, peak, d_u);
    run<0, 16>("ffma2_all", blocks, peak, d_u);
    run<6, 8>("ffma2_aff_fset_iadd3", blocks, peak, d_u);
    run<6, 16>("ffma2_aff_fset_iadd3", blocks, peak, d_u);
    run<7, 8>("ffma2_cmp_last_int", blocks, peak, d_u);
    run<7, 16>("ffma2_cmp_last_int", blocks, peak, d_u);
    run<8, 8>("fset_last_int", blocks, peak, d_u);
    run<8, 16>("fset_last_int", blocks, peak, d_u);
  }
  for (int waves : {4}) {
    const int blocks = sms * waves;
    run<0, 4>("ffma2_all", blocks, peak, d_u);
    run<0, 8>("ffma2_all", blocks, peak, d_u);
    run<1, 4>("ffma2_aff_ffma_cmp", blocks, peak, d_u);
    run<1, 8>("ffma2_aff_ffma_cmp", blocks, peak, d_u);
    run<2, 4>("ffma_all", blocks, peak, d_u);
    run<2, 8>("ffma_all", blocks, peak, d_u);
    run<3, 4>("ffma2_aff_int_cmp", blocks, peak, d_u);
    run<3, 8>("ffma2_aff_int_cmp", blocks, peak, d_u);
    run<4, 4>("ffma2_aff_setp", blocks, peak, d_u);
    run<4, 8>("ffma2_aff_setp", blocks, peak, d_u);
    run<5, 4>("ffma2_mixed_cmp", blocks, peak, d_u);
    run<5, 8>("ffma2_mixed_cmp", blocks, peak, d_u);
  }
  return 0;
}
