// Scoring inner-loop shapes (development microbenchmark, not shipped).
// Each variant: 8 hypotheses per thread, points broadcast from shared
// memory, squared corridor compare, sign-bit counting; only the code shape
// (operand layout / instruction order) differs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/score_loop_mb tools/score_loop_mb.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int kPts = 2048;
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ float u01(uint32_t x) { return (hsh(x) >> 8) * (1.0f / 16777216.0f); }

__device__ __forceinline__ uint32_t le_mask(float e, float t) {
  uint32_t m;
  asm("set.le.u32.f32 %0, %1, %2;" : "=r"(m) : "f"(fabsf(e)), "f"(t));
  return m;
}

struct Hy { float2 A[4], B[4], C[4], T[4]; };
__device__ __forceinline__ void init_h(Hy& h, uint32_t base) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t s = base + q * 8u;
    h.A[q] = make_float2(u01(s) - 0.5f, u01(s + 1) - 0.5f);
    h.B[q] = make_float2(0.8f + 0.1f * u01(s + 2), 0.8f + 0.1f * u01(s + 3));
    h.C[q] = make_float2(-0.4f * u01(s + 4), -0.4f * u01(s + 5));
    const float t = 0.05f + 0.1f * u01(s + 6);
    h.T[q] = make_float2(-t * t, -t * t);
  }
}

// V=0: per point, per pair: B-step, A-step, square (production shape)
// V=1: per point pair: all B-steps, then all A-steps, then squares
// V=2: point-pair packing: smem float4 (x1,x2,y1,y2); hypothesis scalars
// V=6..8: V=2 with some FFMA2 steps as scalar FFMA (measured slower, mb4)
__device__ float4 g_pts[64][kPts / 2];  // V=4: points in global memory (L1-cached broadcast)

template <int V, int TH, int MINB, int UNR>
__global__ void __launch_bounds__(TH, MINB) loop_mb(int reps, uint32_t* out) {
  __shared__ float4 pts_s[V == 4 ? 1 : kPts / 2];
  float4* pts = V == 4 ? g_pts[blockIdx.x & 63] : pts_s;
  if (V != 4)
    for (int i = threadIdx.x; i < kPts / 2; i += blockDim.x) {
      const uint32_t s = blockIdx.x * 7919u + i * 4u;
      pts[i] = make_float4(u01(s), u01(s + 1), u01(s + 2), u01(s + 3));
    }
  Hy h;
  init_h(h, (blockIdx.x * TH + threadIdx.x) * 64u);
  uint32_t cnt[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) cnt[q] = 0;
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
#pragma unroll UNR
    for (int i = 0; i < kPts / 2; ++i) {
      const float4 v = V == 4 ? __ldg(&pts[i]) : pts[i];
      if (V == 0 || V == 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 e = __ffma2_rn(h.A[q], make_float2(v.x, v.x), __ffma2_rn(h.B[q], make_float2(v.y, v.y), h.C[q]));
          float2 g = __ffma2_rn(e, e, h.T[q]);
          cnt[2 * q] += __float_as_uint(g.x) >> 31; cnt[2 * q + 1] += __float_as_uint(g.y) >> 31;
          e = __ffma2_rn(h.A[q], make_float2(v.z, v.z), __ffma2_rn(h.B[q], make_float2(v.w, v.w), h.C[q]));
          g = __ffma2_rn(e, e, h.T[q]);
          cnt[2 * q] += __float_as_uint(g.x) >> 31; cnt[2 * q + 1] += __float_as_uint(g.y) >> 31;
        }
      } else if (V == 1) {
        float2 t0[4], t1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) t0[q] = __ffma2_rn(h.B[q], make_float2(v.y, v.y), h.C[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) t1[q] = __ffma2_rn(h.B[q], make_float2(v.w, v.w), h.C[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) t0[q] = __ffma2_rn(h.A[q], make_float2(v.x, v.x), t0[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) t1[q] = __ffma2_rn(h.A[q], make_float2(v.z, v.z), t1[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 g0 = __ffma2_rn(t0[q], t0[q], h.T[q]);
          const float2 g1 = __ffma2_rn(t1[q], t1[q], h.T[q]);
          cnt[2 * q] += (__float_as_uint(g0.x) >> 31) + (__float_as_uint(g1.x) >> 31);
          cnt[2 * q + 1] += (__float_as_uint(g0.y) >> 31) + (__float_as_uint(g1.y) >> 31);
        }
      } else if (V == 3) {
        // hypothesis-pair outer, 4 points inner: the coefficient pairs sit in
        // the same operand slot of consecutive FFMA2s (operand-reuse cache)
        const float4 w = pts[(i + 1) & (kPts / 2 - 1)];
        const float xs[4] = {v.x, v.z, w.x, w.z}, ys[4] = {v.y, v.w, w.y, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 t[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) t[p] = __ffma2_rn(h.B[q], make_float2(ys[p], ys[p]), h.C[q]);
#pragma unroll
          for (int p = 0; p < 4; ++p) t[p] = __ffma2_rn(h.A[q], make_float2(xs[p], xs[p]), t[p]);
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const float2 g = __ffma2_rn(t[p], t[p], h.T[q]);
            cnt[2 * q] += __float_as_uint(g.x) >> 31; cnt[2 * q + 1] += __float_as_uint(g.y) >> 31;
          }
        }
        ++i;
      } else if (V == 5) {
        // diagonal pairing, no broadcast operand: v = (x1, x2, y1, y2);
        // FFMA2 lanes = (hyp 2k, point 1) + (hyp 2k+1, point 2), then swapped
        const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
        const float2 Xs = make_float2(v.y, v.x), Ys = make_float2(v.w, v.z);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 ea = __ffma2_rn(h.A[q], X, __ffma2_rn(h.B[q], Y, h.C[q]));
          float2 eb = __ffma2_rn(h.A[q], Xs, __ffma2_rn(h.B[q], Ys, h.C[q]));
          ea = __ffma2_rn(ea, ea, h.T[q]);
          eb = __ffma2_rn(eb, eb, h.T[q]);
          cnt[2 * q] += __float_as_uint(ea.x) >> 31;
          cnt[2 * q + 1] += __float_as_uint(ea.y) >> 31;
          cnt[2 * q] += __float_as_uint(eb.x) >> 31;
          cnt[2 * q + 1] += __float_as_uint(eb.y) >> 31;
        }
      } else if (V >= 6 && V <= 8) {
        // V=6: as V=2 but the square step as two scalar FFMA
        // V=7: as V=2 but the B step as two scalar FFMA
        // V=8: all scalar FFMA (3 per eval)
        const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float a = hh ? h.A[q].y : h.A[q].x, b = hh ? h.B[q].y : h.B[q].x;
            const float c = hh ? h.C[q].y : h.C[q].x, t = hh ? h.T[q].y : h.T[q].x;
            float2 e, g;
            if (V == 8) {
              e.x = __fmaf_rn(X.x, a, __fmaf_rn(Y.x, b, c));
              e.y = __fmaf_rn(X.y, a, __fmaf_rn(Y.y, b, c));
            } else if (V == 7) {
              const float2 u = make_float2(__fmaf_rn(Y.x, b, c), __fmaf_rn(Y.y, b, c));
              e = __ffma2_rn(X, make_float2(a, a), u);
            } else {
              e = __ffma2_rn(X, make_float2(a, a), __ffma2_rn(Y, make_float2(b, b), make_float2(c, c)));
            }
            if (V == 7) {
              g = __ffma2_rn(e, e, make_float2(t, t));
            } else {
              g.x = __fmaf_rn(e.x, e.x, t);
              g.y = __fmaf_rn(e.y, e.y, t);
            }
            cnt[2 * q + hh] += (__float_as_uint(g.x) >> 31) + (__float_as_uint(g.y) >> 31);
          }
        }
      } else if (V == 9 || V == 10) {
        // V=9: V=2 with the hypothesis scaled so that t = 1: the square step
        // as two scalar FFMA with the immediate -1 (FFMA imm-form)
        // V=10: the same as FFMA2 with a constant (-1, -1)
        const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float a = hh ? h.A[q].y : h.A[q].x, b = hh ? h.B[q].y : h.B[q].x;
            const float c = hh ? h.C[q].y : h.C[q].x;
            const float2 e = __ffma2_rn(X, make_float2(a, a), __ffma2_rn(Y, make_float2(b, b), make_float2(c, c)));
            float2 g;
            if (V == 9) {
              g.x = __fmaf_rn(e.x, e.x, -1.0f);
              g.y = __fmaf_rn(e.y, e.y, -1.0f);
            } else {
              g = __ffma2_rn(e, e, make_float2(-1.0f, -1.0f));
            }
            cnt[2 * q + hh] += (__float_as_uint(g.x) >> 31) + (__float_as_uint(g.y) >> 31);
          }
        }
      } else if (V >= 11 && V <= 14) {
        // V=11..14: V=2 with the last NL hypotheses of the 8 scored by the
        // linear compare |e| <= thi on the ALU pipe (FSET -> 0 / -1 masks,
        // one IADD3 per two masks) instead of the square step (FFMA2) and the
        // sign count: NL = 4, 3, 2, 8 -- balances the FMA and ALU pipes
        constexpr int NL = V == 11 ? 4 : V == 12 ? 3 : V == 13 ? 2 : 8;
        const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float a = hh ? h.A[q].y : h.A[q].x, b = hh ? h.B[q].y : h.B[q].x;
            const float c = hh ? h.C[q].y : h.C[q].x, t = hh ? h.T[q].y : h.T[q].x;
            const float2 e = __ffma2_rn(X, make_float2(a, a), __ffma2_rn(Y, make_float2(b, b), make_float2(c, c)));
            if (2 * q + hh >= 8 - NL) {
              const float tl = sqrtf(-t);  // (hoisted: loop-invariant)
              cnt[2 * q + hh] -= le_mask(e.x, tl) + le_mask(e.y, tl);
            } else {
              const float2 g = __ffma2_rn(e, e, make_float2(t, t));
              cnt[2 * q + hh] += (__float_as_uint(g.x) >> 31) + (__float_as_uint(g.y) >> 31);
            }
          }
        }
      } else {
        // v = (x1, x2, y1, y2)
        const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float a = hh ? h.A[q].y : h.A[q].x, b = hh ? h.B[q].y : h.B[q].x;
            const float c = hh ? h.C[q].y : h.C[q].x, t = hh ? h.T[q].y : h.T[q].x;
            const float2 e = __ffma2_rn(X, make_float2(a, a), __ffma2_rn(Y, make_float2(b, b), make_float2(c, c)));
            const float2 g = __ffma2_rn(e, e, make_float2(t, t));
            cnt[2 * q + hh] += (__float_as_uint(g.x) >> 31) + (__float_as_uint(g.y) >> 31);
          }
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += cnt[q] * (q + 1);
  out[blockIdx.x * TH + threadIdx.x] = s;
}

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

template <class F> float time_ms(F f) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < 3; ++i) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float t; CK(cudaEventElapsedTime(&t, a, b)); best = t < best ? t : best;
  }
  return best;
}

template <int V, int TH, int MINB, int UNR>
void run(int sms, double peak, uint32_t* d) {
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, loop_mb<V, TH, MINB, UNR>, TH, 0));
  const int blocks = sms * per * 4, reps = 4;
  const float ms = time_ms([&] { loop_mb<V, TH, MINB, UNR><<<blocks, TH>>>(reps, d); });
  CK(cudaGetLastError());
  const double ev = double(blocks) * TH * 8 * kPts * reps;
  const double rate = ev / (ms * 1e-3);
  cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, loop_mb<V, TH, MINB, UNR>));
  printf("{\"V\": %d, \"threads\": %d, \"minb\": %d, \"unroll\": %d, \"regs\": %d, \"ctas_per_sm\": %d, "
         "\"evals_per_s\": %.4e, \"frac_of_ffma_peak\": %.3f}\n",
         V, TH, MINB, UNR, fa.numRegs, per, rate, rate * 4 / peak);
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* df; uint32_t* du;
  CK(cudaMalloc(&df, 1024)); CK(cudaMalloc(&du, sizeof(uint32_t) * sms * 64 * 1024));
  const int pb = sms * 8, iters = 20000;
  const float mp = time_ms([&] { ffma3_peak<<<pb, 256>>>(iters, 0.9999f, 1e-7f, df); });
  const double peak = double(pb) * 256 * iters * 16 * 2 / (mp * 1e-3);
  printf("{\"ffma_peak_tflops\": %.2f}\n", peak / 1e12);
  {
    std::vector<float4> h(64 * (kPts / 2));
    for (size_t i = 0; i < h.size(); ++i) h[i] = make_float4(0.1f * (i % 7), 0.2f, 0.3f * (i % 3), 0.4f);
    CK(cudaMemcpyToSymbol(g_pts, h.data(), h.size() * sizeof(float4)));
  }
  run<2, 256, 2, 2>(sms, peak, du);
  run<2, 128, 4, 2>(sms, peak, du);
  run<11, 256, 2, 2>(sms, peak, du);
  run<11, 128, 4, 2>(sms, peak, du);
  run<12, 256, 2, 2>(sms, peak, du);
  run<12, 128, 4, 2>(sms, peak, du);
  run<13, 256, 2, 2>(sms, peak, du);
  run<14, 256, 2, 2>(sms, peak, du);
  run<9, 256, 2, 2>(sms, peak, du);
  run<9, 128, 4, 2>(sms, peak, du);
  run<10, 256, 2, 2>(sms, peak, du);
  run<10, 128, 4, 2>(sms, peak, du);
  run<6, 256, 2, 2>(sms, peak, du);
  run<6, 128, 4, 2>(sms, peak, du);
  run<7, 256, 2, 2>(sms, peak, du);
  run<7, 128, 4, 2>(sms, peak, du);
  run<8, 256, 2, 2>(sms, peak, du);
  run<8, 128, 4, 2>(sms, peak, du);
  return 0;
}
