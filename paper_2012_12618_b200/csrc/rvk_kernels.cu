// sm_100a kernels of the per-cluster velocity-profile estimator.
//
//   prep_warp_kernel / prep_hyp_kernel
//                  normalize_cluster + median + mad_threshold
//                  (src/ransac.cpp:69-94, include/rvk/ransac.hpp:53-84), every
//                  trial's seed pair (src/ransac.cpp:111-123) and the FP32
//                  coefficients of its line, scoring-unit registration; one
//                  warp per small cluster or one CTA per cluster
//   score_kernel   the hot loop: every (cluster, trial) line hypothesis
//                  against every point of its cluster (run_trial,
//                  src/ransac.cpp:32-65), FP32 packed FFMA2 with a guard band
//                  -> UPPER-BOUND counts; persistent, TMA-staged units
//   select_kernel / select_warp_kernel
//                  exact argmax (max count, lowest trial; :181-189): the best
//                  upper bound is verified exactly, then every trial whose
//                  upper bound reaches that exact count; winner mask rebuilt
//                  exactly; then the least-squares refit + heading of
//                  estimate_cluster_velocity (src/velocity.cpp:26-90)
//   fused_warp_kernel
//                  all of the above for one small cluster per warp with the
//                  intermediates in shared memory (single-frame calls)
//   refit_kernel   estimate_all on caller-provided masks (velocity.cpp:92-121)
//   pack_mask_kernel, mad_exact_kernel, exact_counts_kernel, seed_pairs_kernel
//                  packed mask output and the exact-threshold / per-trial-count
//                  / seed-pair entry points
//
// Why the argmax stays exact: upper[t] >= exact[t] for every trial (the FP32
// band only ever admits extra points). If E0 is the exact count of the
// lowest-index trial with the largest upper bound, any trial t with
// upper[t] < E0 has exact[t] < E0 and cannot win or tie, so verifying the
// trials with upper[t] >= E0 decides the reference's winner exactly.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include <math_constants.h>

#include "rvk_device.cuh"
#include "rvk_kernels.cuh"

namespace rvk_gpu {

using namespace rvk_dev;

namespace {

constexpr int kPrepThreads = 256;
constexpr int kSelectThreads = 256;
constexpr int kNH = 8;            // hypotheses per scoring thread (four FFMA2 pairs)

// Sign counting in the scoring loops. g = e^2 - t2hi comes out of FFMA2 as a
// pair (point 2q in .x, point 2q+1 in .y); a point is a possible inlier when
// its g is negative. RVK_SIGN_PRMT=0: one LEA.HI per point (cnt += bits >> 31).
// RVK_SIGN_PRMT=1: one PRMT per pair packs both signs, sign-replicated, into
// the bytes (sx, sx, sy, sy) = 65535 sx - 65536 sy (mod 2^32), and one IADD3
// adds two such words to the accumulator: 1.5 ALU instructions per pair
// instead of 2. After A even-point and B odd-point hits the accumulator holds
// V = 65535 A - 65536 B (mod 2^32): A = -V mod 2^16 (A < 2^16), and
// A - B = (V + A) / 2^16 as a signed value, so the count A + B is exact.
// Measured (B200, profiles/r2_sign_prmt.md): score_kernel 0.924 -> 0.915 ms on
// config 3, 0.249 -> 0.248 ms on config 2 (kept); the fused prep + score
// kernel 0.900 -> 0.909 ms at T = 256, 2.681 -> 2.672 ms at T = 1024 (off).
#ifndef RVK_SIGN_PRMT  // A/B builds (RVK_NVCC_FLAGS): score_kernel
#define RVK_SIGN_PRMT 1
#endif
#ifndef RVK_FUSED_SIGN_PRMT  // A/B builds: fused_score_block
#define RVK_FUSED_SIGN_PRMT 0
#endif
__device__ __forceinline__ uint32_t sign_pair(float2 g) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0xFFBB;"
      : "=r"(r)
      : "r"(__float_as_uint(g.x)), "r"(__float_as_uint(g.y)));
  return r;
}
__device__ __forceinline__ uint32_t sign_pair_count(uint32_t v) {
  const uint32_t a = (0u - v) & 0xFFFFu;
  const int32_t a_minus_b = static_cast<int32_t>(v + a) >> 16;
  return 2u * a - static_cast<uint32_t>(a_minus_b);
}
static_assert(kScorePPT < 32768, "sign_pair_count: A < 2^16 and |A - B| < 2^15 per unit");
constexpr float kPadY = 1e30f;    // padding point: e^2 overflows any corridor

// ---------------------------------------------------------------- helpers

template <class T, class Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide reduction; every thread gets the result. `red` holds >= 32 T.
template <class T, class Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_reduce(v, op);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = red[0];
  if (nw <= 4) {  // few partials: every thread combines them (no extra barrier)
    for (int w = 1; w < nw; ++w) r = op(r, red[w]);
    return r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one thread combines the warp partials, same order
    for (int w = 1; w < nw; ++w) r = op(r, red[w]);
    red[0] = r;
  }
  __syncthreads();
  return red[0];
}

struct SumI {
  __device__ int operator()(int a, int b) const { return a + b; }
};
struct SumD {
  __device__ double operator()(double a, double b) const { return a + b; }
};
struct MaxU64 {
  __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
    return a > b ? a : b;
  }
};
struct MinI {
  __device__ int operator()(int a, int b) const { return b < a ? b : a; }
};

// k-th smallest (0-based) normalized doppler of the block's cluster, exact:
// MSD radix select over the IEEE bit patterns (non-negative doubles order
// like their bit patterns). hist: 256 counters in shared memory.
// xy is written earlier in the same kernel: no __restrict__ (no .nc loads).
__device__ double block_select_y(const double2* xy, int n, int k,
                                 unsigned int* hist, unsigned long long* sh_prefix,
                                 int* sh_k) {
  unsigned long long prefix = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned long long hi_mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long key =
          static_cast<unsigned long long>(__double_as_longlong(xy[i].y)) & ~(1ull << 63);
      if (((key ^ prefix) & hi_mask) == 0) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: find the bucket holding rank k
      const int lane = threadIdx.x;
      unsigned int local[8];
      unsigned int sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        local[q] = hist[lane * 8 + q];
        sum += local[q];
      }
      unsigned int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned int excl = incl - sum;
      const unsigned int kk = static_cast<unsigned int>(k);
      const bool mine = kk >= excl && kk < incl;
      if (mine) {
        unsigned int cum = excl;
        int digit = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (kk >= cum && kk < cum + local[q]) {
            digit = lane * 8 + q;
            *sh_k = static_cast<int>(kk - cum);
          }
          cum += local[q];
        }
        *sh_prefix = prefix | (static_cast<unsigned long long>(digit) << shift);
      }
    }
    __syncthreads();
    prefix = *sh_prefix;
    k = *sh_k;
    __syncthreads();
  }
  return __longlong_as_double(static_cast<long long>(prefix));
}

// ------------------------------------------------------------- prep kernel

// k-th smallest (0-based) of n non-negative doubles given as bit patterns in
// shared memory: MSD radix select with `bits`-bit digits (11: 6 passes over
// 2048 counters, 8: 8 passes over 256), exact. hist: 2^bits counters; sh: 2
// ints of scratch. Fallback of block_select_pair.
__device__ unsigned long long block_radix_select(const unsigned long long* keys, int n, int k,
                                                 unsigned int* hist, int* sh, int bits) {
  unsigned long long prefix = 0, mask = 0;
  const int nt = blockDim.x;
#pragma unroll 1
  for (int top = 64; top > 0; top -= bits) {
    const int shift = top > bits ? top - bits : 0;
    const unsigned int nb = 1u << (top - shift);
    for (int i = threadIdx.x; i < (int)nb; i += nt) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += nt) {
      const unsigned long long key = keys[i];
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & (nb - 1)], 1u);
    }
    __syncthreads();
    // Block-wide search for the bucket holding rank k: thread j owns bins
    // [j*per, (j+1)*per).
    const int per = (nb + nt - 1) / nt;
    unsigned int local = 0;
    for (int q = 0; q < per; ++q) {
      const int bin = threadIdx.x * per + q;
      if (bin < (int)nb) local += hist[bin];
    }
    // exclusive scan of `local` across the block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    __shared__ unsigned int wsum[32];
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned int base = 0;
    for (int w = 0; w < warp; ++w) base += wsum[w];
    const unsigned int excl = base + incl - local;
    const unsigned int kk = static_cast<unsigned int>(k);
    if (kk >= excl && kk < excl + local) {
      unsigned int cum = excl;
      for (int q = 0; q < per; ++q) {
        const int bin = threadIdx.x * per + q;
        const unsigned int h = bin < (int)nb ? hist[bin] : 0u;
        if (kk < cum + h) {
          sh[0] = bin;
          sh[1] = static_cast<int>(kk - cum);
          break;
        }
        cum += h;
      }
    }
    __syncthreads();
    prefix |= static_cast<unsigned long long>(sh[0]) << shift;
    mask |= static_cast<unsigned long long>(nb - 1) << shift;
    k = sh[1];
    __syncthreads();
  }
  return prefix;
}

constexpr int kMedBins = 2048;  // value buckets of [0, 1] for the median (maximum)
constexpr int kCandCap = 512;   // candidates ranked directly (maximum)

// nb: a power of two <= kMedBins, so y * nb is exact and the map monotone
__device__ __forceinline__ int med_bin(unsigned long long key, int nb) {
  const double y = __longlong_as_double(static_cast<long long>(key));
  const int b = static_cast<int>(y * nb);  // exact scaling; y in [0, 1]
  return b < nb - 1 ? b : nb - 1;
}

// Dynamic shared memory of the prep kernels, sized per launch from the
// sort capacity (prep_dyn_bytes): [keys: cap][cand: candcap][hist: histcap]
// [xs: cap].
// Addressed from the extern symbol (not through stored pointers) so every
// access compiles to LDS/STS rather than generic loads.
extern __shared__ __align__(16) unsigned char prep_dyn[];

struct PrepShared {
  // [cap] normalized dopplers (bit patterns, sign cleared)
  __device__ unsigned long long* keys() const {
    return reinterpret_cast<unsigned long long*>(prep_dyn);
  }
  // [candcap] candidates of the median bucket
  __device__ unsigned long long* cand() const { return keys() + cap; }
  // [histcap] bucket / radix counters (>= 256)
  __device__ unsigned int* hist() const {
    return reinterpret_cast<unsigned int*>(keys() + cap + candcap);
  }
  // [cap] normalized azimuths (the hypotheses' seed points come from here and
  // from keys(), not from global memory)
  __device__ double* xs() const { return reinterpret_cast<double*>(hist() + histcap); }
  int cap;                   // clusters up to this size are kept in shared memory
  int candcap;
  int histcap;               // 2048: 11-bit radix digits, else 8-bit
  double red[32];
  double4 red4[32];
  unsigned long long sel[2];
  int sh[4];
  unsigned int wsum[32];
  double4 stat;
};

__host__ __device__ inline int prep_histcap(int cap) {
  if (cap >= 1024) return kMedBins;
  int h = 256;
  while (h < cap) h <<= 1;
  return h;
}
__host__ __device__ inline int prep_candcap(int cap) { return cap < kCandCap ? cap : kCandCap; }
__host__ __device__ inline size_t prep_dyn_bytes(int cap) {
  return static_cast<size_t>(cap) * 8 + static_cast<size_t>(prep_candcap(cap)) * 8 +
         static_cast<size_t>(prep_histcap(cap)) * 4 + static_cast<size_t>(cap) * 8;
}
__device__ void prep_smem_setup(PrepShared& sm, int cap) {
  if (threadIdx.x == 0) {
    sm.cap = cap;
    sm.candcap = prep_candcap(cap);
    sm.histcap = prep_histcap(cap);
  }
  __syncthreads();
}

// Median buckets of a cluster of n points: about one per point (small
// clusters scan few empty buckets), at least one per thread; a power of two.
__device__ __forceinline__ int med_buckets(int n, int histcap) {
  int nb = blockDim.x;
  while (nb < n && nb < histcap) nb <<= 1;
  return nb;
}

// The k-th and (k+1)-th smallest keys (k+1 only if `pair`), exact. Keys are
// bucketed by value (a monotone map), the bucket holding rank k is collected
// and ranked directly; a crowded bucket falls back to the radix select.
// On entry sm.hist()[0, nb) holds the bucket histogram of the n keys
// (built by prep_cluster's normalize pass) and sm.sh[2] == 0.
__device__ void block_select_pair(PrepShared& sm, int n, int k, bool pair, int nb,
                                  unsigned long long& v0, unsigned long long& v1) {
  const int nt = blockDim.x, tid = threadIdx.x;
  // bin holding rank k: thread j owns bins [j*per, (j+1)*per)
  const int per = nb >> (31 - __clz(nt));  // both powers of two, nb >= nt
  unsigned int local = 0;
  if (per >= 4) {
    const uint4* h4 = reinterpret_cast<const uint4*>(sm.hist() + tid * per);
    for (int q = 0; q < (per >> 2); ++q) {
      const uint4 u = h4[q];
      local += u.x + u.y + u.z + u.w;
    }
  } else {
    for (int q = 0; q < per; ++q) local += sm.hist()[tid * per + q];
  }
  const int lane = tid & 31, warp = tid >> 5;
  unsigned int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) sm.wsum[warp] = incl;
  __syncthreads();
  unsigned int base = 0;
  for (int w = 0; w < warp; ++w) base += sm.wsum[w];
  const unsigned int excl = base + incl - local;
  const unsigned int kk = static_cast<unsigned int>(k);
  if (kk >= excl && kk < excl + local) {
    unsigned int cum = excl;
    for (int q = 0; q < per; ++q) {
      const unsigned int h = sm.hist()[tid * per + q];
      if (kk < cum + h) {
        sm.sh[0] = tid * per + q;          // bin
        sm.sh[1] = static_cast<int>(cum);  // keys below the bin
        break;
      }
      cum += h;
    }
  }
  __syncthreads();
  const int bin = sm.sh[0];
  const int below = sm.sh[1];
  const int in_bin = static_cast<int>(sm.hist()[bin]);
  if (in_bin > sm.candcap) {  // crowded bucket: exact radix select
    const int bits = sm.histcap >= 2048 ? 11 : 8;
    v0 = block_radix_select(sm.keys(), n, k, sm.hist(), sm.sh, bits);
    if (pair) v1 = block_radix_select(sm.keys(), n, k + 1, sm.hist(), sm.sh, bits);
    return;
  }
  for (int i = tid; i < n; i += nt) {
    const unsigned long long key = sm.keys()[i];
    if (med_bin(key, nb) == bin) sm.cand()[atomicAdd(reinterpret_cast<unsigned int*>(&sm.sh[2]), 1u)] = key;
  }
  const bool second_in_bin = pair && k + 1 < below + in_bin;
  __syncthreads();
  const int r0 = k - below;
  for (int i = tid; i < in_bin; i += nt) {
    const unsigned long long ci = sm.cand()[i];
    int less = 0, eq = 0;
    for (int j = 0; j < in_bin; ++j) {
      const unsigned long long cj = sm.cand()[j];
      less += cj < ci;
      eq += cj == ci;
    }
    if (r0 >= less && r0 < less + eq) sm.sel[0] = ci;
    if (second_in_bin && r0 + 1 >= less && r0 + 1 < less + eq) sm.sel[1] = ci;
  }
  if (pair && !second_in_bin) {
    // the (k+1)-th is the smallest key above the bin
    unsigned long long m = ~0ull;
    for (int i = tid; i < n; i += nt) {
      const unsigned long long key = sm.keys()[i];
      if (med_bin(key, nb) > bin && key < m) m = key;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long u = __shfl_xor_sync(0xffffffffu, m, o);
      m = u < m ? u : m;
    }
    __syncthreads();
    if (lane == 0) sm.cand()[warp] = m;  // cand[] reads are done
    __syncthreads();
    if (tid == 0) {
      unsigned long long r = sm.cand()[0];
      for (int w = 1; w < (nt >> 5); ++w) r = sm.cand()[w] < r ? sm.cand()[w] : r;
      sm.sel[1] = r;
    }
  }
  __syncthreads();
  v0 = sm.sel[0];
  if (pair) v1 = sm.sel[1];
}

__device__ double first_zero(double v, const double* __restrict__ a, int n, double* red) {
  if (v != 0.0) return v;
  int first = INT_MAX;
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    if (a[k] == 0.0) first = k < first ? k : first;
  first = block_reduce(first, MinI(), reinterpret_cast<int*>(red));
  return a[first];
}

// Size bucket of a partial tile of `rem` points (1 <= rem < ppt): larger
// tiles get lower buckets, bucket 0 holds the full tiles.
__device__ __forceinline__ int tile_bucket(int rem, const ScoreGeom& g) {
  return 1 + (((g.ppt - 1 - rem) * (kTileBuckets - 1)) >> g.ppt_shift);
}
// The same for full-size (kScorePPT) units, as the warp-per-cluster prep
// registers them whatever the call's ppt (its clusters are small and many;
// tile_capacity() at any ppt <= kScorePPT bounds that count).
__device__ __forceinline__ int tile_bucket_full(int rem) {
  return 1 + (kScorePPT - 1 - rem) / (kScorePPT / (kTileBuckets - 1));
}

__device__ __forceinline__ int64_t xy32_base(const int64_t* offsets, int c) {
  return ((offsets[c] + 1) & ~int64_t{1}) + 2 * static_cast<int64_t>(c);
}

// xy32 holds each cluster's points two at a time as (x_2q, x_2q+1, y_2q,
// y_2q+1): one float4 = two points with x and y already paired for the
// scoring loop's FFMA2 (two points x one hypothesis per instruction).
__device__ __forceinline__ void xy32_put(float2* base, int k, float x, float y) {
  float* f = reinterpret_cast<float*>(base) + (k >> 1) * 4 + (k & 1);
  f[0] = x;
  f[2] = y;
}
__device__ __forceinline__ float2 xy32_get(const float2* base, int k) {
  const float* f = reinterpret_cast<const float*>(base) + (k >> 1) * 4 + (k & 1);
  return make_float2(f[0], f[2]);
}

// Per cluster (one CTA): normalize_cluster (src/ransac.cpp:69-87), the median
// of the normalized dopplers (ransac.hpp:53-70, exact selection), and the MAD
// corridor as a guaranteed interval. Leaves stat in sm.stat for the caller.
//
// The reference sums |y_i - med| left to right (ransac.hpp:78-83), n
// dependent FP64 adds; that order cannot be parallelized bit-exactly. Here
// the deviations (identical doubles) are summed in a tree; for non-negative
// terms any summation order is within gamma_{n-1} * S of the exact sum S, so
// the reference's sum lies within 2 gamma_{n-1} S_tree of ours, and after the
// division by n and the scale multiply (a few more roundings) the reference's
// threshold lies in thr_mid * (1 -/+ (4n + 16) 2^-53). Every consumer decides
// with that interval and takes the exact sequential sum only when a distance
// lands inside it (exact_threshold(); practically never).
//
// stat[c] = (thr_lo, thr_hi, median, thr_exact or NaN).
__device__ void prep_cluster(PrepShared& sm, int c, const int64_t* __restrict__ offsets,
                             const double* __restrict__ az, const double* __restrict__ dop,
                             double scale, double2* xy64, float2* __restrict__ xy32,
                             double4* __restrict__ stat, double* __restrict__ norm) {
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);

  const bool in_smem = n <= sm.cap;
  const int nb = med_buckets(n, sm.histcap);
  double lo0 = DBL_MAX, hi0 = -DBL_MAX, lo1 = DBL_MAX, hi1 = -DBL_MAX;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double a = az[b + k], d = dop[b + k];
    lo0 = a < lo0 ? a : lo0;
    hi0 = a > hi0 ? a : hi0;
    lo1 = d < lo1 ? d : lo1;
    hi1 = d > hi1 ? d : hi1;
  }
  {  // (min az, max az, min dop, max dop): per-thread partials go to the
     // keys area (free until the normalize pass below; cap >= 512 keeps it
     // >= 32 B per thread), warp 0 combines them. No partial is NaN (the
     // loop above never takes one), so plain compares are exact.
    double4* part = reinterpret_cast<double4*>(prep_dyn);
    part[threadIdx.x] = make_double4(lo0, hi0, lo1, hi1);
    if (in_smem) {  // median buckets, filled by the normalize pass
      uint4* h4 = reinterpret_cast<uint4*>(sm.hist());
      for (int i = threadIdx.x; i < (nb >> 2); i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
      if (threadIdx.x == 0) sm.sh[2] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      double4 v = part[threadIdx.x];
      for (int i = threadIdx.x + 32; i < (int)blockDim.x; i += 32) {
        const double4 u = part[i];
        v.x = u.x < v.x ? u.x : v.x;
        v.y = u.y > v.y ? u.y : v.y;
        v.z = u.z < v.z ? u.z : v.z;
        v.w = u.w > v.w ? u.w : v.w;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ux = __shfl_xor_sync(0xffffffffu, v.x, o);
        const double uy = __shfl_xor_sync(0xffffffffu, v.y, o);
        const double uz = __shfl_xor_sync(0xffffffffu, v.z, o);
        const double uw = __shfl_xor_sync(0xffffffffu, v.w, o);
        v.x = ux < v.x ? ux : v.x;
        v.y = uy > v.y ? uy : v.y;
        v.z = uz < v.z ? uz : v.z;
        v.w = uw > v.w ? uw : v.w;
      }
      if (threadIdx.x == 0) sm.red4[0] = v;
    }
    __syncthreads();
    const double4 v = sm.red4[0];
    lo0 = v.x;
    hi0 = v.y;
    lo1 = v.z;
    hi1 = v.w;
  }
  // Eigen's minCoeff/maxCoeff keep the FIRST extreme in index order; values
  // that compare equal differ in bits only for +-0, so an extreme equal to
  // zero takes the bits of its first occurrence (block-uniform branch).
  lo0 = first_zero(lo0, az + b, n, sm.red);
  hi0 = first_zero(hi0, az + b, n, sm.red);
  lo1 = first_zero(lo1, dop + b, n, sm.red);
  hi1 = first_zero(hi1, dop + b, n, sm.red);
  const double s0 = __dsub_rn(hi0, lo0);
  const double s1 = __dsub_rn(hi1, lo1);
  float2* p32 = xy32 + xy32_base(offsets, c);
  // (div_rn_shared, as in prep_warp_kernel, measured slower here: spills)
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double x = s0 == 0.0 ? 0.5 : __ddiv_rn(__dsub_rn(az[b + k], lo0), s0);
    const double y = s1 == 0.0 ? 0.5 : __ddiv_rn(__dsub_rn(dop[b + k], lo1), s1);
    xy64[b + k] = make_double2(x, y);
    xy32_put(p32, k, __double2float_rn(x), __double2float_rn(y));
    if (in_smem) {
      // key: bit pattern with the sign cleared (-0.0 sorts with +0.0, as
      // std::sort's operator< treats them; every other value is >= +0),
      // counted into its median bucket right away
      const unsigned long long key =
          static_cast<unsigned long long>(__double_as_longlong(y)) & ~(1ull << 63);
      sm.keys()[k] = key;
      sm.xs()[k] = x;
      atomicAdd(&sm.hist()[med_bin(key, nb)], 1u);
    }
  }
  if (threadIdx.x == 0 && (n & 1)) xy32_put(p32, n, 0.f, kPadY);  // pad to even
  if (threadIdx.x == 0 && norm != nullptr) {
    norm[4 * c + 0] = lo0;
    norm[4 * c + 1] = lo1;
    norm[4 * c + 2] = s0;
    norm[4 * c + 3] = s1;
  }
  __syncthreads();

  double med;
  if (in_smem) {
    // k-th order statistics (median of the sorted copy, ransac.hpp:60-69).
    const int k0 = (n & 1) ? n / 2 : n / 2 - 1;
    unsigned long long v0 = 0, v1 = 0;
    block_select_pair(sm, n, k0, (n & 1) == 0, nb, v0, v1);
    const double d0 = __longlong_as_double(static_cast<long long>(v0));
    med = (n & 1) ? d0
                  : __ddiv_rn(__dadd_rn(d0, __longlong_as_double(static_cast<long long>(v1))), 2.0);
  } else {
    const double2* cxy = xy64 + b;
    if (n & 1) {
      med = block_select_y(cxy, n, n / 2, sm.hist(), &sm.sel[0], &sm.sh[0]);
    } else {
      const double lo = block_select_y(cxy, n, n / 2 - 1, sm.hist(), &sm.sel[0], &sm.sh[0]);
      const double hi = block_select_y(cxy, n, n / 2, sm.hist(), &sm.sel[0], &sm.sh[0]);
      med = __ddiv_rn(__dadd_rn(lo, hi), 2.0);
    }
  }

  double part = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double y = in_smem ? __longlong_as_double(static_cast<long long>(sm.keys()[k]))
                             : xy64[b + k].y;
    part += fabs(__dsub_rn(y, med));
  }
  const double S = block_reduce(part, SumD(), sm.red);
  if (threadIdx.x == 0) {
    const double mid = scale * (S / n);
    const double delta = (4.0 * n + 16.0) * 0x1p-53;
    const double4 st = make_double4(mid * (1.0 - delta), mid * (1.0 + delta), med, CUDART_NAN);
    stat[c] = st;
    sm.stat = st;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPrepThreads)
prep_kernel(int32_t n_clusters, const int64_t* __restrict__ offsets,
            const double* __restrict__ az, const double* __restrict__ dop, double scale,
            double2* xy64, float2* __restrict__ xy32, double4* __restrict__ stat,
            double* __restrict__ norm, int cap) {
  __shared__ PrepShared sm;
  prep_smem_setup(sm, cap);
  prep_cluster(sm, blockIdx.x, offsets, az, dop, scale, xy64, xy32, stat, norm);
}

// prep + hypothesis setup + tile registration, one CTA per cluster.
//
// Hypotheses (src/ransac.cpp:35-46 for every trial of draw_seed_pair
// :111-123): exact FP64 slope/intercept from the KeyedRng seed pair, FP32
// coefficients and corridor bound, stored per group of 8 trials as
// A[8] B[8] C[8] K[8] (K = -t2hi for the squared compare). Trials beyond T
// in the last group are inert. The cluster's upper-bound counters are zeroed
// and its scoring tiles (g.ppt <= kScorePPT points x TS groups each) are appended to
// the size bucket they belong to, so the scoring kernel takes them
// largest-first.
__device__ void prep_hyp_body(PrepShared& sm, int* tile_pos, int c,
                              const int64_t* __restrict__ offsets, const double* __restrict__ az,
                              const double* __restrict__ dop, double scale,
                              const int32_t* __restrict__ keys, const ScoreGeom& g,
                              uint64_t seed, double2* xy64, float2* __restrict__ xy32,
                              double4* __restrict__ stat, float* __restrict__ hyp,
                              int32_t* __restrict__ upper, int4* __restrict__ tiles,
                              int32_t* __restrict__ tile_count, int64_t tile_cap) {
  if (offsets[c + 1] - offsets[c] < 3) return;  // select writes the too-small sentinel
  prep_cluster(sm, c, offsets, az, dop, scale, xy64, xy32, stat, nullptr);
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  const uint32_t key = keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c);
  const uint64_t k1 = seed_key(key);
  const double thr_lo = sm.stat.x, thr_hi = sm.stat.y;
  const double2* p64 = xy64 + b;  // written by this CTA before the barrier
  int32_t* uc = upper + static_cast<int64_t>(c) * g.Tg * 8;
  float* hc = hyp + static_cast<int64_t>(c) * g.Tg * 32;
  const bool seeds_in_smem = n <= sm.cap;
  for (int t = threadIdx.x; t < g.Tg * 8; t += blockDim.x) {
    FastHyp f = inert_fast();
    if (t < g.T) {
      int i, j;
      seed_pair_k(seed, k1, static_cast<uint32_t>(t), static_cast<uint32_t>(n), i, j);
      if (seeds_in_smem) {  // |y| (keys): a -0.0 seed is +0.0 here, same FP32 line
        const double* xs = sm.xs();
        const unsigned long long* ks = sm.keys();
        f = make_fast_from_seeds(xs[i], __longlong_as_double(static_cast<long long>(ks[i])),
                                 xs[j], __longlong_as_double(static_cast<long long>(ks[j])),
                                 thr_lo, thr_hi);
      } else {
        const double2 p = p64[i], q = p64[j];  // written by this CTA before the barrier
        f = make_fast_from_seeds(p.x, p.y, q.x, q.y, thr_lo, thr_hi);
      }
    }
    float* h = hc + (t >> 3) * 32 + (t & 7);
    h[0] = f.A;
    h[8] = f.B;
    h[16] = f.C;
    h[24] = -f.t2hi;  // K: the squared compare's bound
    uc[t] = 0;
  }
  // scoring tiles of this cluster
  const int full = n >> g.ppt_shift, rem = n & (g.ppt - 1);
  if (threadIdx.x == 0) {
    tile_pos[0] = full ? atomicAdd(&tile_count[0], full * g.nhb) : 0;
    tile_pos[1] = rem ? atomicAdd(&tile_count[tile_bucket(rem, g)], g.nhb) : 0;
  }
  __syncthreads();
  const int64_t base32 = xy32_base(offsets, c);
  for (int i = threadIdx.x; i < full * g.nhb; i += blockDim.x) {
    const int pb = i / g.nhb, hb = i - pb * g.nhb;
    tiles[tile_pos[0] + i] =
        make_int4(c, static_cast<int>(base32 + pb * g.ppt), g.ppt, hb * g.TS);
  }
  if (rem) {
    const int bk = tile_bucket(rem, g);
    for (int hb = threadIdx.x; hb < g.nhb; hb += blockDim.x)
      tiles[bk * tile_cap + tile_pos[1] + hb] =
          make_int4(c, static_cast<int>(base32 + full * g.ppt), rem, hb * g.TS);
  }
}

// One CTA per cluster (big_list == nullptr), or persistent CTAs working
// through the list of clusters the warp kernel left for them
// (big_ctl[0] = count, big_ctl[1] = claim counter). 256-thread CTAs for
// throughput, 512 for calls with few clusters (latency: the largest
// cluster's chain is the call's critical path).
template <int kMaxThreads, int kMinBlocks>
__global__ void __launch_bounds__(kMaxThreads, kMinBlocks)
prep_hyp_kernel(int32_t n_clusters, const int64_t* __restrict__ offsets,
                const double* __restrict__ az, const double* __restrict__ dop, double scale,
                const int32_t* __restrict__ keys, ScoreGeom g, uint64_t seed, double2* xy64,
                float2* __restrict__ xy32, double4* __restrict__ stat, float* __restrict__ hyp,
                int32_t* __restrict__ upper, int4* __restrict__ tiles,
                int32_t* __restrict__ tile_count, int64_t tile_cap, int cap,
                const int32_t* __restrict__ big_list, int32_t* big_ctl) {
  __shared__ PrepShared sm;
  prep_smem_setup(sm, cap);
  __shared__ int tile_pos[2];
  __shared__ int s_idx;
  if (big_list == nullptr) {
    prep_hyp_body(sm, tile_pos, blockIdx.x, offsets, az, dop, scale, keys, g, seed, xy64, xy32,
                  stat, hyp, upper, tiles, tile_count, tile_cap);
    return;
  }
  if (*reinterpret_cast<volatile int32_t*>(&big_ctl[0]) == 0) return;  // nothing listed
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(&big_ctl[1], 1);
    __syncthreads();
    const int i = s_idx;
    if (i >= *reinterpret_cast<volatile int32_t*>(&big_ctl[0])) break;
    prep_hyp_body(sm, tile_pos, big_list[i], offsets, az, dop, scale, keys, g, seed, xy64, xy32,
                  stat, hyp, upper, tiles, tile_count, tile_cap);
    __syncthreads();
  }
}

// ------------------------------------------------ warp-per-cluster prep
//
// Clusters of up to kWarpCap points (the common case of imaging-radar
// frames: thousands of clusters of ~50-350 points) are prepared by ONE warp
// each, with warp shuffles and __syncwarp instead of block barriers: the
// same normalize_cluster / median / MAD interval / hypothesis setup / unit
// registration as prep_hyp_body, bit for bit. Larger clusters are appended
// to a list for the CTA kernel.
constexpr int kWarpCap = 512;
constexpr int kWarpCand = 128;
constexpr int kPrepWarps = 4;  // 4 x 10 KB of static shared memory per CTA

// One warp's cluster in shared memory: the raw azimuth/doppler are staged
// here by the min/max pass (one global read per point), normalized in place,
// and the hypotheses' seed points come from here (no global round trip).
struct WarpPrep {
  unsigned long long keys[kWarpCap];  // raw doppler bits, then |normalized doppler| bits
  double xs[kWarpCap];                // raw azimuth, then normalized x
  union {
    unsigned int hist[kWarpCap];          // median buckets / radix counters
    unsigned long long cand[kWarpCand];   // the median bucket's keys (after hist is read)
  };
};

// Warp-wide (min, max, min, max) of non-NaN partials: plain compares (no
// fmin NaN handling), the four butterflies interleaved.
__device__ __forceinline__ void warp_minmax2(double& lo0, double& hi0, double& lo1, double& hi1) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double a = __shfl_xor_sync(0xffffffffu, lo0, o);
    const double b = __shfl_xor_sync(0xffffffffu, hi0, o);
    const double c = __shfl_xor_sync(0xffffffffu, lo1, o);
    const double d = __shfl_xor_sync(0xffffffffu, hi1, o);
    lo0 = a < lo0 ? a : lo0;
    hi0 = b > hi0 ? b : hi0;
    lo1 = c < lo1 ? c : lo1;
    hi1 = d > hi1 ? d : hi1;
  }
}
__device__ __forceinline__ int warp_imin(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_umin64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}
// inclusive prefix sum over the warp
__device__ __forceinline__ unsigned int warp_scan(unsigned int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}
// The bits of the first element equal to zero (Eigen's first-occurrence
// minCoeff/maxCoeff for +-0), as first_zero().
__device__ __forceinline__ double warp_first_zero(double v, const double* __restrict__ a, int n,
                                                  int lane) {
  if (v != 0.0) return v;
  int first = INT_MAX;
  for (int k = lane; k < n; k += 32)
    if (a[k] == 0.0) first = k < first ? k : first;
  return a[warp_imin(first)];
}
// Rank `k` among `bins` counters split into per-lane runs of `per`:
// returns (bin, count below the bin) on every lane.
__device__ __forceinline__ void warp_find_rank(const unsigned int* hist, int per, int k, int lane,
                                               int& bin, int& below) {
  unsigned int local = 0;
  for (int q = 0; q < per; ++q) local += hist[lane * per + q];
  const unsigned int incl = warp_scan(local, lane);
  const unsigned int excl = incl - local;
  const unsigned int kk = static_cast<unsigned int>(k);
  const bool mine = kk >= excl && kk < incl;
  int b = 0, c = 0;
  if (mine) {
    unsigned int cum = excl;
    for (int q = 0; q < per; ++q) {
      const unsigned int h = hist[lane * per + q];
      if (kk < cum + h) {
        b = lane * per + q;
        c = static_cast<int>(cum);
        break;
      }
      cum += h;
    }
  }
  const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
  bin = __shfl_sync(0xffffffffu, b, src);
  below = __shfl_sync(0xffffffffu, c, src);
}
// k-th smallest key, MSD radix select with 8-bit digits (fallback for a
// crowded median bucket).
__device__ unsigned long long warp_radix_select(WarpPrep& w, int n, int k, int lane) {
  unsigned long long prefix = 0, mask = 0;
#pragma unroll 1
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) w.hist[i] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const unsigned long long key = w.keys[i];
      if ((key & mask) == prefix) atomicAdd(&w.hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    int digit, below;
    warp_find_rank(w.hist, 8, k, lane, digit, below);
    prefix |= static_cast<unsigned long long>(digit) << shift;
    mask |= 0xFFull << shift;
    k -= below;
    __syncwarp();
  }
  return prefix;
}
// k-th and (k+1)-th smallest keys, exact (warp version of block_select_pair).
// On entry w.hist[0, nb) holds the bucket histogram of the n keys.
__device__ void warp_select_pair(WarpPrep& w, int n, int k, bool pair, int nb, int lane,
                                 unsigned long long& v0, unsigned long long& v1) {
  int bin, below;
  warp_find_rank(w.hist, nb >> 5, k, lane, bin, below);
  const int in_bin = static_cast<int>(w.hist[bin]);
  __syncwarp();  // every lane's hist reads before cand (aliasing hist) is written
  if (in_bin > kWarpCand) {
    v0 = warp_radix_select(w, n, k, lane);
    if (pair) v1 = warp_radix_select(w, n, k + 1, lane);
    return;
  }
  int cnt = 0;  // compact the bucket's keys (order irrelevant)
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const unsigned long long key = i < n ? w.keys[i] : 0ull;
    const bool hit = i < n && med_bin(key, nb) == bin;
    const unsigned int m = __ballot_sync(0xffffffffu, hit);
    if (hit) w.cand[cnt + __popc(m & ((1u << lane) - 1u))] = key;
    cnt += __popc(m);
  }
  __syncwarp();
  const int r0 = k - below;
  const bool second_in_bin = pair && k + 1 < below + in_bin;
  unsigned long long s0 = 0, s1 = 0;
  bool f0 = false, f1 = false;
  for (int i = lane; i < in_bin; i += 32) {
    const unsigned long long ci = w.cand[i];
    int less = 0, eq = 0;
    for (int j = 0; j < in_bin; ++j) {
      const unsigned long long cj = w.cand[j];
      less += cj < ci;
      eq += cj == ci;
    }
    if (r0 >= less && r0 < less + eq) {
      s0 = ci;
      f0 = true;
    }
    if (second_in_bin && r0 + 1 >= less && r0 + 1 < less + eq) {
      s1 = ci;
      f1 = true;
    }
  }
  v0 = __shfl_sync(0xffffffffu, s0, __ffs(__ballot_sync(0xffffffffu, f0)) - 1);
  if (pair) {
    if (second_in_bin) {
      v1 = __shfl_sync(0xffffffffu, s1, __ffs(__ballot_sync(0xffffffffu, f1)) - 1);
    } else {  // the smallest key above the bucket
      unsigned long long m = ~0ull;
      for (int i = lane; i < n; i += 32) {
        const unsigned long long key = w.keys[i];
        if (med_bin(key, nb) > bin && key < m) m = key;
      }
      v1 = warp_umin64(m);
    }
  }
  __syncwarp();
}

// <= 72 registers: at 76 (the allocation rounds to 80) the overlapped
// config 4 step measured 2.3 % slower although the kernel alone was faster.
__global__ void __maxnreg__(72)
prep_warp_kernel(int32_t n_clusters, const int64_t* __restrict__ offsets,
                 const double* __restrict__ az, const double* __restrict__ dop, double scale,
                 const int32_t* __restrict__ keys, ScoreGeom g, uint64_t seed, double2* xy64,
                 float2* __restrict__ xy32, double4* __restrict__ stat, float* __restrict__ hyp,
                 int32_t* __restrict__ upper, int4* __restrict__ tiles,
                 int32_t* __restrict__ tile_count, int64_t tile_cap, int32_t* __restrict__ big_list,
                 int32_t* big_ctl) {
  __shared__ WarpPrep wp[kPrepWarps];
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kPrepWarps + (threadIdx.x >> 5);
  if (c >= n_clusters) return;
  WarpPrep& w = wp[threadIdx.x >> 5];
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  if (n < 3) return;  // select writes the too-small sentinel
  if (n > kWarpCap) {
    if (lane == 0) big_list[atomicAdd(&big_ctl[0], 1)] = c;
    return;
  }
  // median buckets (<= kWarpCap, about one per point), zeroed here and
  // filled by the normalize pass
  int nb = 32;
  while (nb < n) nb <<= 1;
  for (int i = lane; i < nb; i += 32) w.hist[i] = 0;
  // normalize_cluster (src/ransac.cpp:69-87)
  double lo0 = DBL_MAX, hi0 = -DBL_MAX, lo1 = DBL_MAX, hi1 = -DBL_MAX;
  for (int k = lane; k < n; k += 32) {
    const double a = az[b + k], d = dop[b + k];
    w.xs[k] = a;  // staged raw; the same lane normalizes it in place below
    w.keys[k] = static_cast<unsigned long long>(__double_as_longlong(d));
    lo0 = a < lo0 ? a : lo0;
    hi0 = a > hi0 ? a : hi0;
    lo1 = d < lo1 ? d : lo1;
    hi1 = d > hi1 ? d : hi1;
  }
  warp_minmax2(lo0, hi0, lo1, hi1);  // the loop above never takes a NaN
  __syncwarp();  // the zeroed buckets before any lane's atomics
  if (lo0 == 0.0 || hi0 == 0.0 || lo1 == 0.0 || hi1 == 0.0) {  // (rare) first +-0
    lo0 = warp_first_zero(lo0, az + b, n, lane);
    hi0 = warp_first_zero(hi0, az + b, n, lane);
    lo1 = warp_first_zero(lo1, dop + b, n, lane);
    hi1 = warp_first_zero(hi1, dop + b, n, lane);
  }
  const double s0 = __dsub_rn(hi0, lo0);
  const double s1 = __dsub_rn(hi1, lo1);
  float2* p32 = xy32 + xy32_base(offsets, c);
  // the spans are shared by the cluster: one reciprocal each, verified
  // correctly rounded quotients (div_rn_shared == __ddiv_rn, bit for bit)
  const bool f0 = div_span_ok(s0), f1 = div_span_ok(s1);
  const double r0 = f0 ? fast_rcp(s0) : 0.0, r1 = f1 ? fast_rcp(s1) : 0.0;
  auto norm_div = [](double a, double s, bool fast, double r) {
    return fast ? div_rn_shared(a, s, r) : __ddiv_rn(a, s);
  };
  for (int k0 = lane; k0 < n; k0 += 64) {  // two points per lane and step
    const int k1 = k0 + 32;
    const double a0 = w.xs[k0], d0 = __longlong_as_double(static_cast<long long>(w.keys[k0]));
    const double a1 = k1 < n ? w.xs[k1] : 0.0;
    const double d1 = k1 < n ? __longlong_as_double(static_cast<long long>(w.keys[k1])) : 0.0;
    const double x0 = s0 == 0.0 ? 0.5 : norm_div(__dsub_rn(a0, lo0), s0, f0, r0);
    const double y0 = s1 == 0.0 ? 0.5 : norm_div(__dsub_rn(d0, lo1), s1, f1, r1);
    const double x1 = s0 == 0.0 ? 0.5 : norm_div(__dsub_rn(a1, lo0), s0, f0, r0);
    const double y1 = s1 == 0.0 ? 0.5 : norm_div(__dsub_rn(d1, lo1), s1, f1, r1);
    xy64[b + k0] = make_double2(x0, y0);
    xy32_put(p32, k0, __double2float_rn(x0), __double2float_rn(y0));
    const unsigned long long key0 =
        static_cast<unsigned long long>(__double_as_longlong(y0)) & ~(1ull << 63);
    w.keys[k0] = key0;
    w.xs[k0] = x0;
    atomicAdd(&w.hist[med_bin(key0, nb)], 1u);
    if (k1 < n) {
      xy64[b + k1] = make_double2(x1, y1);
      xy32_put(p32, k1, __double2float_rn(x1), __double2float_rn(y1));
      const unsigned long long key1 =
          static_cast<unsigned long long>(__double_as_longlong(y1)) & ~(1ull << 63);
      w.keys[k1] = key1;
      w.xs[k1] = x1;
      atomicAdd(&w.hist[med_bin(key1, nb)], 1u);
    }
  }
  if (lane == 0 && (n & 1)) xy32_put(p32, n, 0.f, kPadY);
  __syncwarp();
  // median (ransac.hpp:53-70) and the MAD interval (see prep_cluster)
  const int k0 = (n & 1) ? n / 2 : n / 2 - 1;
  unsigned long long v0 = 0, v1 = 0;
  warp_select_pair(w, n, k0, (n & 1) == 0, nb, lane, v0, v1);
  const double d0 = __longlong_as_double(static_cast<long long>(v0));
  const double med = (n & 1) ? d0
                             : __ddiv_rn(__dadd_rn(d0, __longlong_as_double(static_cast<long long>(v1))), 2.0);
  double part = 0.0;
  for (int k = lane; k < n; k += 32)
    part += fabs(__dsub_rn(__longlong_as_double(static_cast<long long>(w.keys[k])), med));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  const double mid = scale * (part / n);
  const double delta = (4.0 * n + 16.0) * 0x1p-53;
  const double thr_lo = mid * (1.0 - delta), thr_hi = mid * (1.0 + delta);
  if (lane == 0) stat[c] = make_double4(thr_lo, thr_hi, med, CUDART_NAN);
  // hypotheses (as prep_hyp_body, FFMA2 layout) and zeroed counters
  const uint32_t key = keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c);
  const uint64_t k1 = seed_key(key);
  float* hc = hyp + static_cast<int64_t>(c) * g.Tg * 32;
  int32_t* uc = upper + static_cast<int64_t>(c) * g.Tg * 8;
  // two trials per lane and step: both seed pairs' loads are in flight
  // before the first FP64 line is built
  for (int t0 = lane; t0 < g.Tg * 8; t0 += 64) {
    const int t1 = t0 + 32;
    const bool a0 = t0 < g.T, a1 = t1 < g.T;
    int i0 = 0, j0 = 0, i1 = 0, j1 = 0;
    if (a0) seed_pair_k(seed, k1, static_cast<uint32_t>(t0), static_cast<uint32_t>(n), i0, j0);
    if (a1) seed_pair_k(seed, k1, static_cast<uint32_t>(t1), static_cast<uint32_t>(n), i1, j1);
    // seeds from the slot: x, and |y| (a -0.0 seed is +0.0 here: the same FP32 line)
    auto ky = [&](int i) { return __longlong_as_double(static_cast<long long>(w.keys[i])); };
    const FastHyp f0 = a0 ? make_fast_from_seeds(w.xs[i0], ky(i0), w.xs[j0], ky(j0), thr_lo,
                                                 thr_hi)
                          : inert_fast();
    const FastHyp f1 = a1 ? make_fast_from_seeds(w.xs[i1], ky(i1), w.xs[j1], ky(j1), thr_lo,
                                                 thr_hi)
                          : inert_fast();
    float* h = hc + (t0 >> 3) * 32 + (t0 & 7);
    h[0] = f0.A;
    h[8] = f0.B;
    h[16] = f0.C;
    h[24] = -f0.t2hi;
    uc[t0] = 0;
    if (t1 < g.Tg * 8) {
      h = hc + (t1 >> 3) * 32 + (t1 & 7);
      h[0] = f1.A;
      h[8] = f1.B;
      h[16] = f1.C;
      h[24] = -f1.t2hi;
      uc[t1] = 0;
    }
  }
  // scoring units of this cluster
  const int full = n / kScorePPT, rem = n % kScorePPT;
  int pos0 = 0, pos1 = 0;
  if (lane == 0) {
    pos0 = full ? atomicAdd(&tile_count[0], full * g.nhb) : 0;
    pos1 = rem ? atomicAdd(&tile_count[tile_bucket_full(rem)], g.nhb) : 0;
  }
  pos0 = __shfl_sync(0xffffffffu, pos0, 0);
  pos1 = __shfl_sync(0xffffffffu, pos1, 0);
  const int64_t base32 = xy32_base(offsets, c);
  for (int i = lane; i < full * g.nhb; i += 32) {
    const int pb = i / g.nhb, hb = i - pb * g.nhb;
    tiles[pos0 + i] = make_int4(c, static_cast<int>(base32 + pb * kScorePPT), kScorePPT, hb * g.TS);
  }
  if (rem) {
    const int bk = tile_bucket_full(rem);
    for (int hb = lane; hb < g.nhb; hb += 32)
      tiles[bk * tile_cap + pos1 + hb] =
          make_int4(c, static_cast<int>(base32 + full * kScorePPT), rem, hb * g.TS);
  }
}

// The exact reference threshold (left-to-right MAD sum), one warp per
// cluster: used where the threshold itself is an output
// (rvk_cluster_thresholds) and by the all-trials exact counter.
__global__ void mad_exact_kernel(int32_t n_clusters, const int64_t* __restrict__ offsets,
                                 const double2* __restrict__ xy64, double scale,
                                 double4* __restrict__ stat) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n_clusters || (threadIdx.x & 31) != 0) return;
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  double4 st = stat[c];
  const double t = exact_threshold(xy64 + b, n, st.z, scale);
  st.x = t;
  st.y = t;
  st.w = t;
  stat[c] = st;
}

// ------------------------------------------------------------ score kernel

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Waits for the phase with the given parity. A wait that never completes is
// a pipeline bug: trap (the launch fails with an error) instead of hanging.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t spins = 0; !mbar_try_wait(bar, parity);)
    if (++spins == (1u << 26)) __trap();
}
// 1-D bulk copy global -> shared (TMA engine), completion on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The hot loop, persistent and warp-granular. Every warp claims scoring
// units from the LPT-ordered unit list with an atomic counter (largest
// first, so the tail is short); a unit = (cluster, 32 groups of 8
// hypotheses, up to kScorePPT points). Lane j holds group j's 8 hypotheses
// (A, B, C, K = -t2hi; four FFMA2 pairs) in registers and streams the
// unit's points (staged in the warp's shared-memory slot) as float4
// broadcast loads (two points each): per point and pair 3 FFMA2 (e = A x + (B y + C); g = e^2 - t2hi) and the sign
// bit of g added to the count (LEA.HI). No shared memory and no CTA
// barrier in the loop: the per-unit latency of one warp (claim, descriptor,
// hypothesis loads) is covered by the other warps of the SM sub-partition.
// Counts are upper bounds (guard band, see make_fast) and accumulate over
// units with integer atomics (order-free, deterministic).
// per warp two slots of (kScorePPT / 2 + 2) float4
constexpr size_t kScoreSmemBytes =
    static_cast<size_t>(kScoreThreads / 32) * 2 * (kScorePPT / 2 + 2) * sizeof(float4);

// Unit index (LPT order) -> descriptor: binary search of the bucket starts.
__device__ __forceinline__ int4 unit_desc(const int* bstart, const int4* __restrict__ tiles,
                                          int64_t tile_cap, int u) {
  int lo = 0, hi = kTileBuckets;  // bstart[lo] <= u < bstart[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (bstart[mid] <= u) lo = mid;
    else hi = mid;
  }
  return tiles[lo * tile_cap + (u - bstart[lo])];
}

// Stages a unit's points (an even-aligned run of float2 = (n + 1) / 2 float4)
// into a warp's shared-memory slot through the TMA engine: one 1-D bulk copy
// issued by lane 0, completion (bytes) tracked on the slot's mbarrier.
__device__ __forceinline__ void stage_points_bulk(float4* slot, uint64_t* bar,
                                                  const float2* __restrict__ xy32, int4 d,
                                                  int lane) {
  if (lane == 0) {
    const uint32_t bytes = static_cast<uint32_t>((d.z + 1) >> 1) * 16u;
    mbar_expect_tx(bar, bytes);
    bulk_g2s(slot, xy32 + d.y, bytes, bar);
  }
}

__global__ void __launch_bounds__(kScoreThreads, 3)
score_kernel(const int32_t* __restrict__ tile_count, const int4* __restrict__ tiles,
             int64_t tile_cap, const float2* __restrict__ xy32, const float* __restrict__ hyp,
             ScoreGeom g, int32_t* __restrict__ upper, const int32_t* __restrict__ list_n) {
  // CTA path behind the fused kernels (list_n = big_ctl: its units come only
  // from the listed clusters): nothing listed, nothing to score -- the host
  // cannot know that for device-resident offsets, so the launch stays and
  // every CTA leaves before the prologue
  if (list_n != nullptr && *list_n == 0) return;
  constexpr int kSlot = kScorePPT / 2 + 2;  // float4 per slot (+2: read-ahead slack)
  __shared__ int bstart[kTileBuckets + 1];
  // two point slots per warp: the current unit's and the next unit's (prefetch)
  extern __shared__ __align__(16) float4 pts_dyn[];
  auto pts_s = reinterpret_cast<float4(*)[2][kSlot]>(pts_dyn);
  __shared__ __align__(8) uint64_t slot_bar[kScoreThreads / 32][2];  // per slot
  const int tid = threadIdx.x, lane = tid & 31;
  if (lane == 0) {
    mbar_init(&slot_bar[tid >> 5][0], 1);
    mbar_init(&slot_bar[tid >> 5][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t phase = 0;  // parity bit per slot (bit b = slot b)
  if (tid < 32) {  // exclusive prefix of the bucket sizes
    int carry = 0;
    for (int b0 = 0; b0 < kTileBuckets; b0 += 32) {
      const int v = b0 + tid < kTileBuckets ? tile_count[b0 + tid] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += u;
      }
      if (b0 + tid < kTileBuckets) bstart[b0 + tid] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) bstart[kTileBuckets] = carry;
  }
  __syncthreads();
  const int total = bstart[kTileBuckets];
  int* next = const_cast<int*>(tile_count) + kTileBuckets;
  int u = 0, un = 0;
  if (lane == 0) {
    u = atomicAdd(next, 1);
    un = atomicAdd(next, 1);
  }
  u = __shfl_sync(0xffffffffu, u, 0);
  int4 d = make_int4(0, 0, 0, 0);
  int buf = 0;
  if (u < total) {
    d = unit_desc(bstart, tiles, tile_cap, u);
    stage_points_bulk(pts_s[tid >> 5][0], &slot_bar[tid >> 5][0], xy32, d, lane);
  }
#pragma unroll 1
  while (u < total) {
    // 1. this unit's hypotheses: lane j holds group d.w + j (A, B, C, K x 8)
    const int gi = d.w + lane;
    const bool active = gi < g.Tg;
    float A[kNH], B[kNH];
    float2 Cc[kNH], T2[kNH];
    {
      const float4* hp = reinterpret_cast<const float4*>(
          hyp + (static_cast<int64_t>(d.x) * g.Tg + (active ? gi : d.w)) * 32);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 a = __ldg(hp + h), bb = __ldg(hp + 2 + h), cc = __ldg(hp + 4 + h),
                     kk = __ldg(hp + 6 + h);
        A[4 * h] = a.x, A[4 * h + 1] = a.y, A[4 * h + 2] = a.z, A[4 * h + 3] = a.w;
        B[4 * h] = bb.x, B[4 * h + 1] = bb.y, B[4 * h + 2] = bb.z, B[4 * h + 3] = bb.w;
        Cc[4 * h] = make_float2(cc.x, cc.x);
        Cc[4 * h + 1] = make_float2(cc.y, cc.y);
        Cc[4 * h + 2] = make_float2(cc.z, cc.z);
        Cc[4 * h + 3] = make_float2(cc.w, cc.w);
        T2[4 * h] = make_float2(kk.x, kk.x);
        T2[4 * h + 1] = make_float2(kk.y, kk.y);
        T2[4 * h + 2] = make_float2(kk.z, kk.z);
        T2[4 * h + 3] = make_float2(kk.w, kk.w);
      }
    }
    // 2. the next unit (claimed one unit ago): descriptor + point prefetch,
    //    and the claim after it
    const int u_next = __shfl_sync(0xffffffffu, un, 0);
    int4 dn = make_int4(0, 0, 0, 0);
    if (u_next < total) {
      dn = unit_desc(bstart, tiles, tile_cap, u_next);
      // the slot was last read one unit ago (the warp is converged)
      stage_points_bulk(pts_s[tid >> 5][buf ^ 1], &slot_bar[tid >> 5][buf ^ 1], xy32, dn, lane);
    }
    if (lane == 0) un = atomicAdd(next, 1);
    // 3. this unit's points have landed
    mbar_wait(&slot_bar[tid >> 5][buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    __syncwarp();

    uint32_t cnt[kNH];
#pragma unroll
    for (int q = 0; q < kNH; ++q) cnt[q] = 0;
    // v = (x_2q, x_2q+1, y_2q, y_2q+1): per hypothesis 3 FFMA2 over the two
    // points (e = A x + (B y + C); g = e^2 - t2hi) and two sign bits
    auto g_of = [&](const float4& v, int h) {
      const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
      const float2 e = __ffma2_rn(X, make_float2(A[h], A[h]),
                                  __ffma2_rn(Y, make_float2(B[h], B[h]), Cc[h]));
      return __ffma2_rn(e, e, T2[h]);
    };
    auto score_pair = [&](const float4& v) {
#pragma unroll
      for (int h = 0; h < kNH; ++h) {
        const float2 g = g_of(v, h);
        if (RVK_SIGN_PRMT) cnt[h] += sign_pair(g);
        else cnt[h] += (__float_as_uint(g.x) >> 31) + (__float_as_uint(g.y) >> 31);
      }
    };
    // 4. broadcast LDS.128 (two points each), four float4 per iteration
    //    (the other warps of the sub-partition cover the LDS latency)
    const float4* cp = pts_s[tid >> 5][buf];
    const int m2 = (d.z + 1) >> 1;
    int q2 = 0;
#pragma unroll 1
    for (; q2 + 4 <= m2; q2 += 4) {
      const float4 v0 = cp[q2], v1 = cp[q2 + 1], v2 = cp[q2 + 2], v3 = cp[q2 + 3];
      if (RVK_SIGN_PRMT) {
#pragma unroll
        for (int h = 0; h < kNH; ++h) {
          cnt[h] += sign_pair(g_of(v0, h)) + sign_pair(g_of(v1, h));
          cnt[h] += sign_pair(g_of(v2, h)) + sign_pair(g_of(v3, h));
        }
      } else {
        score_pair(v0);
        score_pair(v1);
        score_pair(v2);
        score_pair(v3);
      }
    }
#pragma unroll 1
    for (; q2 < m2; ++q2) score_pair(cp[q2]);
    if (RVK_SIGN_PRMT) {
#pragma unroll
      for (int q = 0; q < kNH; ++q) cnt[q] = sign_pair_count(cnt[q]);
    }
    if (active) {
      int32_t* up = upper + (static_cast<int64_t>(d.x) * g.Tg + gi) * 8;
#pragma unroll
      for (int q = 0; q < kNH; ++q)
        if (cnt[q]) atomicAdd(&up[q], static_cast<int32_t>(cnt[q]));
    }
    __syncwarp();  // this slot is refilled two units from now
    u = u_next;
    d = dn;
    buf ^= 1;
  }
}

// ----------------------------------------------------------- select kernel

// Exact count of one hypothesis by one warp; sets *undecided when some
// point's FP64 distance fell inside the threshold interval.
__device__ int warp_exact_count(const ExactHyp& H, int n, const float2* __restrict__ p32,
                                const double2* __restrict__ p64, double thr_lo, double thr_hi,
                                bool* undecided) {
  if (H.L.degenerate) return 0;
  int cnt = 0;
  bool und = false;
  for (int k = threadIdx.x & 31; k < n; k += 32) {
    const int d = classify(H, k, xy32_get(p32, k), p64, thr_lo, thr_hi);
    cnt += d == kIn;
    und |= d == kUndecided;
  }
  *undecided = __any_sync(0xffffffffu, und);
  return warp_reduce(cnt, SumI());
}

// LSQ refit + heading of one cluster (estimate_cluster_velocity,
// src/velocity.cpp:26-90; solve_velocity / min_norm_fallback,
// include/rvk/velocity.hpp:46-105; heading_angle velocity.cpp:19-24).
// Each thread accumulates the normal-equation sums of its inliers
// (RefitAcc::add); one fused block reduction with a fixed tree follows, so
// results are deterministic; they differ from Eigen's reduction order only
// in the last bits (tolerance-checked).
// Canonical order (every kernel, every launch shape): lane l of ONE warp
// sums the inliers k == l (mod 32) in increasing k with the explicit FMAs of
// add_cs, then warp_reduce_refit's butterfly combines the 32 lanes -- so the
// velocities are bit-identical whatever CTA shape or batch a cluster is in.
struct RefitAcc {
  double g00 = 0, g01 = 0, g11 = 0, b0 = 0, b1 = 0, ds = 0;
  int nin = 0, first = INT_MAX;
  __device__ __forceinline__ void add_cs(int k, double c, double s, double d) {
    g00 = fma(c, c, g00);
    g01 = fma(c, s, g01);
    g11 = fma(s, s, g11);
    b0 = fma(c, d, b0);
    b1 = fma(s, d, b1);
    ds = __dadd_rn(ds, d);
    ++nin;
    first = k < first ? k : first;
  }
  __device__ __forceinline__ void add(int k, double a, double d) {
    double s, c;
    sincos_az(a, &s, &c);
    add_cs(k, c, s, d);
  }
  // add_cs for a staged point whose (c, s, d) are zeros unless it is an
  // inlier: the sums never hold -0.0, so x + 0 == x and the result equals
  // add_cs on the inliers alone -- branch-free, so the loop can pipeline
  __device__ __forceinline__ void add_staged(int k, double c, double s, double d, bool in) {
    g00 = fma(c, c, g00);
    g01 = fma(c, s, g01);
    g11 = fma(s, s, g11);
    b0 = fma(c, d, b0);
    b1 = fma(s, d, b1);
    ds = __dadd_rn(ds, d);
    nin += in;
    first = in && k < first ? k : first;
  }
};

__device__ __forceinline__ RefitAcc warp_reduce_refit(RefitAcc a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.g00 = __dadd_rn(a.g00, __shfl_xor_sync(0xffffffffu, a.g00, o));
    a.g01 = __dadd_rn(a.g01, __shfl_xor_sync(0xffffffffu, a.g01, o));
    a.g11 = __dadd_rn(a.g11, __shfl_xor_sync(0xffffffffu, a.g11, o));
    a.b0 = __dadd_rn(a.b0, __shfl_xor_sync(0xffffffffu, a.b0, o));
    a.b1 = __dadd_rn(a.b1, __shfl_xor_sync(0xffffffffu, a.b1, o));
    a.ds = __dadd_rn(a.ds, __shfl_xor_sync(0xffffffffu, a.ds, o));
    a.nin += __shfl_xor_sync(0xffffffffu, a.nin, o);
    a.first = min(a.first, __shfl_xor_sync(0xffffffffu, a.first, o));
  }
  return a;
}

// Staging for the canonical order in CTA kernels: all threads compute the
// (cos, sin, doppler) of the inliers of a chunk, warp 0 accumulates it.
constexpr int kRefitChunk = 1024;
struct RefitStage {
  double c[kRefitChunk], s[kRefitChunk], d[kRefitChunk];
  uint8_t in[kRefitChunk];
};

// Thread 0: the 2x2 solve, fallback and heading from the reduced sums.
__device__ __noinline__ void finish_refit(const RefitAcc& a, const double* __restrict__ az,
                             const double* __restrict__ dop, int64_t frame_id, int cluster_id,
                             rvk_estimate* __restrict__ out) {
  const double g00 = a.g00, g01 = a.g01, g11 = a.g11, b0 = a.b0, b1 = a.b1;
  const int nin = a.nin, first = a.first;
  rvk_estimate e;
  e.frame_id = frame_id;
  e.cluster_id = cluster_id;
  e.inlier_count = nin;
  e.heading = 0.0;
  e.has_heading = 0;
  if (nin == 0) {  // velocity.cpp:56-62
    e.v_x = 0.0;
    e.v_y = 0.0;
    e.condition_ok = 0;
    *out = e;
    return;
  }
  if (nin == 1) {  // velocity.cpp:63-67
    double s, c;
    sincos_az(az[first], &s, &c);
    e.v_x = dop[first] * c;
    e.v_y = dop[first] * s;
    e.condition_ok = 0;
  } else {
    const double det = g00 * g11 - g01 * g01;
    const double half_trace = (g00 + g11) / 2.0;
    if (det >= kRankEpsilon * half_trace * half_trace) {  // velocity.hpp:64
      e.v_x = (g11 * b0 - g01 * b1) / det;
      e.v_y = (g00 * b1 - g01 * b0) / det;
      e.condition_ok = 1;
    } else {  // min_norm_fallback, velocity.hpp:79-105
      const double half_sum = (g00 + g11) / 2.0;
      const double half_diff = (g00 - g11) / 2.0;
      const double lambda = half_sum + sqrt(half_diff * half_diff + g01 * g01);
      double u0, u1;
      if (g01 != 0.0) {
        u0 = g01;
        u1 = lambda - g00;
      } else if (g00 >= g11) {
        u0 = 1.0;
        u1 = 0.0;
      } else {
        u0 = 0.0;
        u1 = 1.0;
      }
      const double nr = sqrt(u0 * u0 + u1 * u1);
      if (nr > 0.0) {
        u0 /= nr;
        u1 /= nr;
      }
      double s0, c0;
      sincos_az(az[first], &s0, &c0);
      if (u0 * c0 + u1 * s0 < 0.0) {
        u0 = -u0;
        u1 = -u1;
      }
      const double mean = a.ds / nin;
      e.v_x = mean * u0;
      e.v_y = mean * u1;
      e.condition_ok = 0;
    }
  }
  if (!(fabs(e.v_x) < kZeroVelocityEpsilon && fabs(e.v_y) < kZeroVelocityEpsilon)) {
    const double h = atan2(e.v_y, e.v_x);
    e.heading = h == -kPi ? kPi : h;  // to_half_open_angle, types.hpp:74-77
    e.has_heading = 1;
  }
  *out = e;
}

// estimate_cluster_velocity on a mask in memory, in the canonical order
// (RefitAcc): all threads stage the inliers' (cos, sin, doppler) chunk by
// chunk, warp 0 accumulates, lane 0 solves.
__device__ void block_refit(int n, const double* __restrict__ az, const double* __restrict__ dop,
                            const uint8_t* mask, int64_t frame_id, int cluster_id,
                            rvk_estimate* __restrict__ out, RefitStage& st) {
  RefitAcc acc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int kb = 0; kb < n; kb += kRefitChunk) {
    const int kn = min(kRefitChunk, n - kb);
    for (int i = threadIdx.x; i < kn; i += blockDim.x) {
      const int k = kb + i;
      const bool in = mask[k] != 0;
      st.in[i] = in;
      double sn = 0.0, cs = 0.0, dd = 0.0;
      if (in) {
        sincos_az(az[k], &sn, &cs);
        dd = dop[k];
      }
      st.c[i] = cs;
      st.s[i] = sn;
      st.d[i] = dd;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll 4
      for (int i = lane; i < kn; i += 32)
        acc.add_staged(kb + i, st.c[i], st.s[i], st.d[i], st.in[i] != 0);
    }
    __syncthreads();
  }
  if (warp == 0) {
    const RefitAcc t = warp_reduce_refit(acc);
    if (lane == 0) finish_refit(t, az, dop, frame_id, cluster_id, out);
  }
}

// The device API does no host-side size check (its offsets live in HBM), so a
// cluster below the reference's minimum (kMinClusterSize = 3,
// include/rvk/types.hpp:20; the host API throws ClusterTooSmall first,
// src/ransac.cpp:147-156) is never read: prep skips it and the select /
// fused kernels write a sentinel -- inlier_count = winning_trial = -1, an
// all-zero mask, a zero estimate with condition_ok = 0 and no heading.
constexpr int kMinClusterPoints = 3;
__device__ void write_too_small(int c, int n, int64_t frame_id, int cluster_id,
                                int32_t* out_count, int32_t* out_trial, uint8_t* cmask,
                                rvk_estimate* est, int tid, int nthreads) {
  for (int k = tid; k < n; k += nthreads) cmask[k] = 0;
  if (tid == 0) {
    if (out_count) out_count[c] = -1;
    if (out_trial) out_trial[c] = -1;
    if (est) {
      rvk_estimate e;
      e.frame_id = frame_id;
      e.cluster_id = cluster_id;
      e.inlier_count = 0;
      e.v_x = e.v_y = e.heading = 0.0;
      e.has_heading = 0;
      e.condition_ok = 0;
      est[c] = e;
    }
  }
}

// Exact winner per cluster (one CTA). With U = the fast pass's upper bounds
// (exact[t] <= U[t]), t0 = the lowest trial with the largest U and
// E0 = exact[t0], a trial t can only beat or tie-win against t0 if
// U[t] > E0, or U[t] == E0 and t < t0 (ties go to the lowest trial,
// src/ransac.cpp:181-189). Only those are verified; when U[t0] == E0 there
// are none. One pass over the points classifies them for t0 exactly, writes
// the mask (evaluate_trial, :129-136) and accumulates the LSQ refit sums of
// its inliers; only if another trial wins (or a distance fell inside the
// threshold interval) is the pass repeated.
__device__ __forceinline__ void select_cluster(
    int c, const int64_t* __restrict__ offsets, const double* __restrict__ az,
    const double* __restrict__ dop, const int32_t* __restrict__ keys,
    const int32_t* __restrict__ cluster_ids, int64_t frame_id, const double2* __restrict__ xy64,
    const float2* __restrict__ xy32, const double4* __restrict__ stat, double scale,
    const int32_t* __restrict__ upper, int T, uint64_t seed, int32_t* __restrict__ out_count,
    int32_t* __restrict__ out_trial, uint8_t* __restrict__ mask, rvk_estimate* __restrict__ est) {
  __shared__ unsigned long long redu[32];
  __shared__ RefitStage rst;
  __shared__ unsigned long long best;
  __shared__ double sh_thr;
  __shared__ int sh_need_exact;
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  if (n < kMinClusterPoints) {
    write_too_small(c, n, frame_id, cluster_ids ? cluster_ids[c] : c, out_count, out_trial,
                    mask + b, est, threadIdx.x, blockDim.x);
    return;
  }
  const uint32_t key = keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c);
  const double4 st = stat[c];
  double thr_lo = st.x, thr_hi = st.y;
  const float2* p32 = xy32 + xy32_base(offsets, c);
  const double2* p64 = xy64 + b;
  const double* caz = az + b;
  const double* cdop = dop + b;
  uint8_t* cmask = mask + b;
  const int32_t* U = upper + static_cast<int64_t>(c) * ((T + 7) / 8) * 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool refit = est != nullptr;

  // Switches the whole block to the exact sequential threshold (rare).
  auto go_exact = [&]() {
    if (threadIdx.x == 0) sh_thr = exact_threshold(p64, n, st.z, scale);
    __syncthreads();
    thr_lo = thr_hi = sh_thr;
  };
  // One pass for trial t: mask + exact count + refit sums. Returns false if
  // some distance was undecided (then nothing is valid and the caller
  // switches to the exact threshold).
  auto pass = [&](int t, int& count, RefitAcc& total) -> bool {
    const ExactHyp H = make_exact(p64, seed, key, static_cast<uint32_t>(t), n, thr_lo, thr_hi);
    RefitAcc acc;  // warp 0 (canonical order, see RefitAcc)
    bool und = false;
    int cnt = 0;
    const int nt = blockDim.x;
    for (int kb = 0; kb < n; kb += kRefitChunk) {
      const int ke = min(n, kb + kRefitChunk);
      // two points per thread and step, every load issued before the first
      // use (the loop is latency-bound: few points per thread, one CTA per
      // cluster; four deep costs more in spills than it hides, measured)
      for (int k0 = kb + threadIdx.x; k0 < ke; k0 += 2 * nt) {
        float2 pp[2];
        double pa[2], pd[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = k0 + u * nt;
          if (k < ke) {
            pp[u] = xy32_get(p32, k);
            if (refit) {
              pa[u] = caz[k];
              pd[u] = cdop[k];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = k0 + u * nt;
          if (k >= ke) break;
          const int d = H.L.degenerate ? kOut : classify(H, k, pp[u], p64, thr_lo, thr_hi);
          und |= d == kUndecided;
          const bool in = d == kIn;
          cmask[k] = in ? 1 : 0;
          cnt += in;
          if (refit) {
            rst.in[k - kb] = in;
            double sn = 0.0, cs = 0.0;
            if (in) sincos_az(pa[u], &sn, &cs);
            rst.c[k - kb] = cs;
            rst.s[k - kb] = sn;
            rst.d[k - kb] = in ? pd[u] : 0.0;
          }
        }
      }
      if (refit) {
        __syncthreads();
        if (warp == 0) {
#pragma unroll 4
          for (int i = lane; i < ke - kb; i += 32)
            acc.add_staged(kb + i, rst.c[i], rst.s[i], rst.d[i], rst.in[i] != 0);
        }
        __syncthreads();
      }
    }
    if (__syncthreads_or(und)) return false;
    count = block_reduce(cnt, SumI(), reinterpret_cast<int*>(redu));
    if (refit && warp == 0) total = warp_reduce_refit(acc);  // thread 0 solves
    return true;
  };

  // 1. trial with the largest upper bound (lowest index on ties).
  unsigned long long v = 0;
  {
    // U rows are padded to a multiple of 8 trials (16 B aligned): int4 loads
    const int4* U4 = reinterpret_cast<const int4*>(U);
    for (int q = threadIdx.x; 4 * q < T; q += blockDim.x) {
      const int4 w = U4[q];
      const int t = 4 * q;
      v = MaxU64()(v, pack_best(w.x, t));
      if (t + 1 < T) v = MaxU64()(v, pack_best(w.y, t + 1));
      if (t + 2 < T) v = MaxU64()(v, pack_best(w.z, t + 2));
      if (t + 3 < T) v = MaxU64()(v, pack_best(w.w, t + 3));
    }
  }
  v = block_reduce(v, MaxU64(), redu);
  const int t0 = unpack_trial(v);
  const int u0 = unpack_count(v);

  // 2. its exact count, mask and refit sums in one pass.
  int e0 = 0;
  RefitAcc tot;
  if (!pass(t0, e0, tot)) {
    go_exact();
    pass(t0, e0, tot);
  }
  if (threadIdx.x == 0) {
    best = pack_best(e0, t0);
    sh_need_exact = 0;
  }
  __syncthreads();

  // 3. verify the trials that could still win (none when u0 == e0).
  if (u0 > e0) {
    for (int round = 0; round < 2; ++round) {
      for (int t = warp; t < T; t += nw) {
        const int u = U[t];
        if (t == t0 || u < e0 || (u == e0 && t > t0)) continue;
        const ExactHyp H = make_exact(p64, seed, key, static_cast<uint32_t>(t), n, thr_lo, thr_hi);
        bool und;
        const int e = warp_exact_count(H, n, p32, p64, thr_lo, thr_hi, &und);
        if (und) {
          if (lane == 0) sh_need_exact = 1;
        } else if (lane == 0) {
          atomicMax(&best, pack_best(e, t));
        }
      }
      if (__syncthreads_or(sh_need_exact) && round == 0) {
        go_exact();  // redo every candidate (and t0) with the exact threshold
        if (threadIdx.x == 0) sh_need_exact = 0;
        __syncthreads();
        pass(t0, e0, tot);
        if (threadIdx.x == 0) best = pack_best(e0, t0);
        __syncthreads();
        continue;
      }
      break;
    }
  }
  __syncthreads();
  const int win = unpack_trial(best);
  const int win_count = unpack_count(best);

  // 4. another trial won: its mask and refit sums.
  if (win != t0) {
    int cnt;
    if (!pass(win, cnt, tot)) {
      go_exact();
      pass(win, cnt, tot);
    }
  }
  if (threadIdx.x == 0) {
    if (out_count) out_count[c] = win_count;
    if (out_trial) out_trial[c] = win;
    if (refit)
      finish_refit(tot, caz, cdop, frame_id, cluster_ids ? cluster_ids[c] : c, est + c);
  }
}

// One CTA per cluster (list == nullptr), or persistent CTAs over the list of
// clusters the fused warp kernel left for the CTA path (list_n[0] entries).
__global__ void __launch_bounds__(kSelectThreads, 3)
select_kernel(const int64_t* __restrict__ offsets, const double* __restrict__ az,
              const double* __restrict__ dop, const int32_t* __restrict__ keys,
              const int32_t* __restrict__ cluster_ids, int64_t frame_id,
              const double2* __restrict__ xy64, const float2* __restrict__ xy32,
              const double4* __restrict__ stat, double scale, const int32_t* __restrict__ upper,
              int T, uint64_t seed, int32_t* __restrict__ out_count,
              int32_t* __restrict__ out_trial, uint8_t* __restrict__ mask,
              rvk_estimate* __restrict__ est, const int32_t* __restrict__ list,
              const int32_t* list_n) {
  if (list == nullptr) {
    select_cluster(blockIdx.x, offsets, az, dop, keys, cluster_ids, frame_id, xy64, xy32, stat,
                   scale, upper, T, seed, out_count, out_trial, mask, est);
    return;
  }
  const int m = *list_n;
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    select_cluster(list[i], offsets, az, dop, keys, cluster_ids, frame_id, xy64, xy32, stat,
                   scale, upper, T, seed, out_count, out_trial, mask, est);
    __syncthreads();
  }
}

// ------------------------------------------------ warp-per-cluster select
//
// The same exact winner / mask / refit as select_kernel with ONE warp per
// cluster and no block barriers (imaging-radar frames: thousands of clusters
// of a few hundred points, where select_kernel's CTAs spend their time in
// barrier and latency chains). Candidates are found 32 trials at a time
// with a ballot over the upper bounds.
// One-warp CTAs, 20 per SM (<= 102 registers: 94, no spills): a finished
// warp frees its slot at once (config 4 select 0.239 -> 0.234 ms against
// 4-warp CTAs; 2-warp CTAs 0.240, 24 warps at 80 registers 0.236). Round 2
// before: 5 CTAs of 4 warps took 0.305 -> 0.260 ms against the unbounded
// 123-register build.
#ifndef RVK_SELECT_WARPS  // A/B builds (RVK_NVCC_FLAGS)
#define RVK_SELECT_WARPS 1
#endif
constexpr int kSelectWarps = RVK_SELECT_WARPS;

// Asynchronous global -> shared copies (LDGSTS) and their completion.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// (t0, u0) -- the trial with the largest upper bound and that bound -- in
// stat.w: the bits (u0 << 32 | t0) are a zero or subnormal double (u0 < 2^20),
// never the NaN the prep kernels leave there.
__device__ __forceinline__ double pack_t0(int t0, int u0) {
  return __longlong_as_double((static_cast<long long>(u0) << 32) | static_cast<uint32_t>(t0));
}
__device__ __forceinline__ int unpack_t0_trial(double w) {
  return static_cast<int>(static_cast<uint32_t>(__double_as_longlong(w)));
}
__device__ __forceinline__ int unpack_t0_count(double w) {
  return static_cast<int>(__double_as_longlong(w) >> 32);
}

// A warp's shared slot: the cluster's FP32 pairs and raw az / dop.
constexpr int kSelStage = 384;
struct SelSlot {
  float4 p32[kSelStage / 2];
  double az[kSelStage];
  double dop[kSelStage];
};
constexpr size_t kSelSmem = sizeof(SelSlot) * kSelectWarps;
extern __shared__ __align__(16) unsigned char sel_dyn[];

#ifndef RVK_SELECT_WARP_MINB  // A/B builds (RVK_NVCC_FLAGS)
#define RVK_SELECT_WARP_MINB (20 / kSelectWarps)
#endif
__global__ void __launch_bounds__(kSelectWarps * 32, RVK_SELECT_WARP_MINB)
select_warp_kernel(int32_t n_clusters, const int64_t* __restrict__ offsets,
                   const double* __restrict__ az, const double* __restrict__ dop,
                   const int32_t* __restrict__ keys, const int32_t* __restrict__ cluster_ids,
                   int64_t frame_id, const double2* __restrict__ xy64,
                   const float2* __restrict__ xy32, const double4* __restrict__ stat,
                   double scale, const int32_t* __restrict__ upper, int T, uint64_t seed,
                   int32_t* __restrict__ out_count, int32_t* __restrict__ out_trial,
                   uint8_t* __restrict__ mask, rvk_estimate* __restrict__ est) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kSelectWarps + (threadIdx.x >> 5);
  if (c >= n_clusters) return;
  // stat and the key do not depend on the offsets: their loads go out first,
  // so the two global latencies overlap (stat is in-bounds for every cluster)
  const uint32_t key = keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c);
  const double4 st = stat[c];
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  if (n < kMinClusterPoints) {
    write_too_small(c, n, frame_id, cluster_ids ? cluster_ids[c] : c, out_count, out_trial,
                    mask + b, est, lane, 32);
    return;
  }
  double thr_lo = st.x, thr_hi = st.y;
  const float2* p32 = xy32 + xy32_base(offsets, c);
  const double2* p64 = xy64 + b;
  const double* caz = az + b;
  const double* cdop = dop + b;
  uint8_t* cmask = mask + b;
  const int32_t* U = upper + static_cast<int64_t>(c) * ((T + 7) / 8) * 8;
  const bool refit = est != nullptr;
  // the passes read every point: a cluster of <= kSelStage points is copied
  // into the warp's shared slot (cp.async) while the upper bounds are scanned
  // and t0's line is built, instead of one global round trip per 64 points
  const bool staged = n <= kSelStage;
  if (staged) {
    SelSlot& sl = reinterpret_cast<SelSlot*>(sel_dyn)[threadIdx.x >> 5];
    const float4* g4 = reinterpret_cast<const float4*>(p32);
    for (int q = lane; 2 * q < n; q += 32) cp_async16(sl.p32 + q, g4 + q);
    if (refit)
      for (int k = lane; k < n; k += 32) {
        cp_async8(sl.az + k, caz + k);
        cp_async8(sl.dop + k, cdop + k);
      }
    cp_async_commit();
  }

  auto go_exact = [&]() {  // the exact sequential threshold (rare)
    double t = 0.0;
    if (lane == 0) t = exact_threshold(p64, n, st.z, scale);
    thr_lo = thr_hi = __shfl_sync(0xffffffffu, t, 0);
  };
  // one pass for trial t: mask + exact count + refit sums (false: undecided)
  auto pass = [&](int t, int& count, RefitAcc& total) -> bool {
    const ExactHyp H = make_exact(p64, seed, key, static_cast<uint32_t>(t), n, thr_lo, thr_hi);
    RefitAcc acc;
    bool und = false;
    for (int k0 = lane; k0 < n; k0 += 64) {
      float2 pp[2];
      double pa[2], pd[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + 32 * u;
        if (k < n) {
          pp[u] = xy32_get(p32, k);
          if (refit) {
            pa[u] = caz[k];
            pd[u] = cdop[k];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + 32 * u;
        if (k >= n) break;
        const int d = H.L.degenerate ? kOut : classify(H, k, pp[u], p64, thr_lo, thr_hi);
        und |= d == kUndecided;
        cmask[k] = d == kIn ? 1 : 0;
        if (d == kIn) {
          if (refit) acc.add(k, pa[u], pd[u]);
          else ++acc.nin;
        }
      }
    }
    if (__any_sync(0xffffffffu, und)) return false;
    total = warp_reduce_refit(acc);
    count = total.nin;
    return true;
  };

  // 1. trial with the largest upper bound (lowest index on ties): handed over
  //    in stat.w by the fused prep + score kernel, else a scan of the bounds
  unsigned long long v = 0;
  if (!isnan(st.w)) {
    v = pack_best(unpack_t0_count(st.w), unpack_t0_trial(st.w));
  } else {
    const int4* U4 = reinterpret_cast<const int4*>(U);
    for (int q = lane; 4 * q < T; q += 32) {
      const int4 w = U4[q];
      const int t = 4 * q;
      v = MaxU64()(v, pack_best(w.x, t));
      if (t + 1 < T) v = MaxU64()(v, pack_best(w.y, t + 1));
      if (t + 2 < T) v = MaxU64()(v, pack_best(w.z, t + 2));
      if (t + 3 < T) v = MaxU64()(v, pack_best(w.w, t + 3));
    }
    v = warp_reduce(v, MaxU64());
  }
  const int t0 = unpack_trial(v);
  const int u0 = unpack_count(v);

  // 2. its exact count, mask and refit sums in one pass
  if (staged) {
    SelSlot& sl = reinterpret_cast<SelSlot*>(sel_dyn)[threadIdx.x >> 5];
    cp_async_wait_all();
    __syncwarp();
    p32 = reinterpret_cast<const float2*>(sl.p32);
    caz = sl.az;
    cdop = sl.dop;
  }
  int e0 = 0;
  RefitAcc tot;
  if (!pass(t0, e0, tot)) {
    go_exact();
    pass(t0, e0, tot);
  }
  unsigned long long best = pack_best(e0, t0);

  // 3. verify the trials that could still win (none when u0 == e0); the
  //    candidates of 32 trials at a time by ballot
  if (u0 > e0) {
    for (int round = 0; round < 2; ++round) {
      bool need_exact = false;
      for (int tb = 0; tb < T; tb += 32) {
        const int tl = tb + lane;
        const int u = tl < T ? U[tl] : -1;
        unsigned cand = __ballot_sync(
            0xffffffffu, tl < T && tl != t0 && !(u < e0 || (u == e0 && tl > t0)));
        while (cand) {
          const int t = tb + __ffs(cand) - 1;
          cand &= cand - 1;
          const ExactHyp H =
              make_exact(p64, seed, key, static_cast<uint32_t>(t), n, thr_lo, thr_hi);
          bool und;
          const int e = warp_exact_count(H, n, p32, p64, thr_lo, thr_hi, &und);
          if (und) need_exact = true;
          else best = MaxU64()(best, pack_best(e, t));
        }
      }
      if (need_exact && round == 0) {
        go_exact();  // redo every candidate (and t0) with the exact threshold
        pass(t0, e0, tot);
        best = pack_best(e0, t0);
        continue;
      }
      break;
    }
  }
  const int win = unpack_trial(best);
  const int win_count = unpack_count(best);

  // 4. another trial won: its mask and refit sums
  if (win != t0) {
    int cnt;
    if (!pass(win, cnt, tot)) {
      go_exact();
      pass(win, cnt, tot);
    }
  }
  if (lane == 0) {
    if (out_count) out_count[c] = win_count;
    if (out_trial) out_trial[c] = win;
    if (refit) finish_refit(tot, caz, cdop, frame_id, cluster_ids ? cluster_ids[c] : c, est + c);
  }
}

// --------------------------------------------- fused warp-per-cluster path
//
// One warp owns one cluster from the raw FP64 input onwards; every
// intermediate lives in the warp's shared-memory slot or in registers:
//   1. load az/dop once (coalesced) into the slot, min/max (first-occurrence
//      +-0 semantics), exact normalisation in place (normalize_cluster,
//      src/ransac.cpp:69-87) + FP32 point pairs for the scoring loop;
//   2. exact median of the normalized dopplers and the MAD interval
//      (include/rvk/ransac.hpp:53-84, src/ransac.cpp:89-94), as
//      prep_warp_kernel;
//   3. per block of 256 trials: lane j builds trials 8j..8j+7 (seed pairs,
//      src/ransac.cpp:111-123; FP32 coefficients of the line, :35-46) in
//      registers and scores them against the staged points (the FFMA2 loop
//      of score_kernel): upper-bound counts;
//   4. (kSelect) the exact argmax / verification / winner mask / LSQ refit
//      of select_warp_kernel (src/ransac.cpp:158-199, src/velocity.cpp:26-90).
// Two instantiations:
//   * whole path (kSelect, 508-point slots): HBM sees only the input
//     (16 B/pt), the mask and the per-cluster outputs; one launch -- the
//     default for a call of at most one small-cluster frame;
//   * prep + score (!kSelect, 384-point slots): steps 1-3, then xy64, the
//     xy32 pairs, stat and the upper bounds go to HBM for select_warp_kernel
//     -- the default for batches of small clusters. Without the select code
//     the hot instructions fit the instruction caches, which the whole-path
//     kernel does not on full batches.
// Persistent: warps claim clusters from a counter, so the latency-bound
// phases of some warps overlap the FMA-bound scoring of the others.
// Clusters larger than the slot (or whole-path calls with T > 1024) go to the
// list for the CTA path (prep_hyp_kernel -> score_kernel -> select list).
constexpr int kFusedWarps = 4;

// One warp's shared-memory slot for clusters of up to kCap points. The pair
// region holds the median's candidates until the pairs are written (after
// the median); the bucket region holds the u16 upper bounds after it.
// kHistInPairs (prep + score: no u16 upper bounds in the slot): the buckets
// live in the pair region too, after the candidates -- both are dead once
// the pairs are written -- so the slot is 18 % smaller.
template <int kCap, bool kHistInPairs = false>
struct FusedGeom {
  static constexpr int cap = kCap;
  static constexpr int hist = kCap <= 256 ? 256 : 512;  // median buckets (power of two >= cap)
  static constexpr int max_t = 2 * hist;                // u16 upper bounds in the bucket region
  static constexpr int pairs = kCap / 2 + 3;            // float4 (two points), + read-ahead
  static constexpr size_t x = 0;                        // double x[cap]  (normalized)
  static constexpr size_t y = x + 8 * kCap;             // double y[cap]  (normalized)
  static constexpr size_t p = y + 8 * kCap;             // float4 pairs | u64 cand (| u32 hist)
  static constexpr size_t h = kHistInPairs ? p + 8 * kWarpCand  // u32 hist | u16 upper
                                           : p + 16 * pairs;
  static constexpr size_t slot = kHistInPairs ? p + 16 * pairs : h + 4 * hist;
  static constexpr size_t smem = slot * kFusedWarps;
  static_assert(8 * kWarpCand <= 16 * pairs, "median candidates live in the pair region");
  static_assert(!kHistInPairs || 8 * kWarpCand + 4 * hist <= 16 * pairs, "buckets in pairs");
  static_assert(kCap <= 512, "bucket region");
};
#ifndef RVK_FUSED_PS_HIP  // A/B builds (RVK_NVCC_FLAGS): prep + score buckets in the pair region
#define RVK_FUSED_PS_HIP 1
#endif
#ifndef RVK_FUSED_PS_MINB  // A/B builds: prep + score CTAs per SM (register budget)
#define RVK_FUSED_PS_MINB 5
#endif
// the whole path, one warp per cluster: 508 points, four 4-warp CTAs per SM
using FusedFull = FusedGeom<508>;
// prep + score only (select_warp_kernel follows): 384 points (every config-4
// cluster), five 4-warp CTAs per SM at <= 102 registers
using FusedPrepScore = FusedGeom<384, RVK_FUSED_PS_HIP != 0>;
constexpr int kFusedCap = FusedFull::cap;
constexpr int kFusedMaxT = FusedFull::max_t;

extern __shared__ __align__(16) unsigned char fused_dyn[];

// median key of point i: the normalized doppler's bits with the sign cleared
// (-0.0 sorts with +0.0, as std::sort's operator< treats them)
__device__ __forceinline__ unsigned long long fused_key(const double* y, int i) {
  return static_cast<unsigned long long>(__double_as_longlong(y[i])) & ~(1ull << 63);
}

// k-th smallest key, MSD radix select with 8-bit digits (crowded bucket).
__device__ __noinline__ unsigned long long fused_radix_select(const double* y, unsigned int* hist,
                                                              int n, int k, int lane) {
  unsigned long long prefix = 0, mask = 0;
#pragma unroll 1
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const unsigned long long key = fused_key(y, i);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    int digit, below;
    warp_find_rank(hist, 8, k, lane, digit, below);
    prefix |= static_cast<unsigned long long>(digit) << shift;
    mask |= 0xFFull << shift;
    k -= below;
    __syncwarp();
  }
  return prefix;
}

// k-th and (k+1)-th smallest keys (warp_select_pair on the slot's arrays).
// On entry hist[0, nb) holds the bucket histogram of the n keys.
__device__ __forceinline__ void fused_select_pair(const double* y, unsigned int* hist,
                                                  unsigned long long* cand, int n, int k,
                                                  bool pair, int nb, int lane,
                                                  unsigned long long& v0,
                                                  unsigned long long& v1) {
  int bin, below;
  warp_find_rank(hist, nb >> 5, k, lane, bin, below);
  const int in_bin = static_cast<int>(hist[bin]);
  if (in_bin > kWarpCand) {
    __syncwarp();
    v0 = fused_radix_select(y, hist, n, k, lane);
    if (pair) v1 = fused_radix_select(y, hist, n, k + 1, lane);
    return;
  }
  int cnt = 0;  // compact the bucket's keys (order irrelevant)
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const unsigned long long key = i < n ? fused_key(y, i) : 0ull;
    const bool hit = i < n && med_bin(key, nb) == bin;
    const unsigned int m = __ballot_sync(0xffffffffu, hit);
    if (hit) cand[cnt + __popc(m & ((1u << lane) - 1u))] = key;
    cnt += __popc(m);
  }
  __syncwarp();
  const int r0 = k - below;
  const bool second_in_bin = pair && k + 1 < below + in_bin;
  unsigned long long s0 = 0, s1 = 0;
  bool f0 = false, f1 = false;
  for (int i = lane; i < in_bin; i += 32) {
    const unsigned long long ci = cand[i];
    int less = 0, eq = 0;
    for (int j = 0; j < in_bin; ++j) {
      const unsigned long long cj = cand[j];
      less += cj < ci;
      eq += cj == ci;
    }
    if (r0 >= less && r0 < less + eq) {
      s0 = ci;
      f0 = true;
    }
    if (second_in_bin && r0 + 1 >= less && r0 + 1 < less + eq) {
      s1 = ci;
      f1 = true;
    }
  }
  v0 = __shfl_sync(0xffffffffu, s0, __ffs(__ballot_sync(0xffffffffu, f0)) - 1);
  if (pair) {
    if (second_in_bin) {
      v1 = __shfl_sync(0xffffffffu, s1, __ffs(__ballot_sync(0xffffffffu, f1)) - 1);
    } else {  // the smallest key above the bucket
      unsigned long long m = ~0ull;
      for (int i = lane; i < n; i += 32) {
        const unsigned long long key = fused_key(y, i);
        if (med_bin(key, nb) > bin && key < m) m = key;
      }
      v1 = warp_umin64(m);
    }
  }
  __syncwarp();
}

// exact_threshold on the slot's normalized dopplers (the reference's
// left-to-right MAD sum, ransac.hpp:74-84 + ransac.cpp:89-94), one lane.
__device__ __noinline__ double fused_exact_threshold(const double* y, int n, double med,
                                                     double scale) {
  double acc = 0.0;
  for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, fabs(__dsub_rn(y[k], med)));
  return __dmul_rn(scale, __ddiv_rn(acc, static_cast<double>(n)));
}

// One cluster's slot as the select phase sees it.
struct FusedCluster {
  const double* xs;
  const double* ys;
  const float2* p32;
  const double* caz;
  const double* cdop;
  uint8_t* cmask;
  int n;
  uint32_t key;
  uint64_t seed;
  bool refit;
};

__device__ __forceinline__ ExactHyp fused_make_exact(const FusedCluster& fc, int t, double thr_lo,
                                                     double thr_hi) {
  ExactHyp H;
  seed_pair(fc.seed, fc.key, static_cast<uint32_t>(t), static_cast<uint32_t>(fc.n), H.a, H.b);
  H.L = make_line(fc.xs[H.a], fc.ys[H.a], fc.xs[H.b], fc.ys[H.b]);
  H.f = make_fast(H.L, thr_lo, thr_hi);
  return H;
}

// classify() on the slot: the FP32 test with its certain-in / certain-out
// bounds, the FP64 reference distance inside the band.
__device__ __forceinline__ int fused_classify(const FusedCluster& fc, const ExactHyp& H, int k,
                                              double thr_lo, double thr_hi) {
  if (k == H.a || k == H.b) return kIn;
  const float2 p = xy32_get(fc.p32, k);
  const float e = __fmaf_rn(H.f.A, p.x, __fmaf_rn(H.f.B, p.y, H.f.C));
  if (__fmaf_rn(e, e, -H.f.t2lo) < 0.f) return kIn;
  if (!(__fmaf_rn(e, e, -H.f.t2hi) < 0.f)) return kOut;
  const double r = __dsub_rn(__dadd_rn(__dmul_rn(-H.L.m, fc.xs[k]), fc.ys[k]), H.L.c);
  const double d = __ddiv_rn(fabs(r), H.L.den);
  if (d <= thr_lo) return kIn;
  if (d > thr_hi) return kOut;
  return kUndecided;
}

// One pass for trial t: mask + exact count + refit sums in the canonical
// order (lane l, points k == l mod 32 ascending). false: some distance was
// undecided (nothing valid; the caller switches to the exact threshold).
__device__ __noinline__ bool fused_pass(const FusedCluster fc, int t, double thr_lo,
                                        double thr_hi, int& count, RefitAcc& total) {
  const ExactHyp H = fused_make_exact(fc, t, thr_lo, thr_hi);
  RefitAcc acc;
  bool und = false;
  for (int k = threadIdx.x & 31; k < fc.n; k += 32) {
    const int d = H.L.degenerate ? kOut : fused_classify(fc, H, k, thr_lo, thr_hi);
    und |= d == kUndecided;
    fc.cmask[k] = d == kIn ? 1 : 0;
    if (d == kIn) {
      if (fc.refit) acc.add(k, fc.caz[k], fc.cdop[k]);
      else ++acc.nin;
    }
  }
  if (__any_sync(0xffffffffu, und)) return false;
  total = warp_reduce_refit(acc);
  count = total.nin;
  return true;
}

// Exact count of trial t by the warp (und: some distance undecided).
__device__ __noinline__ int fused_exact_count(const FusedCluster fc, int t, double thr_lo,
                                              double thr_hi, bool& und_out) {
  const ExactHyp H = fused_make_exact(fc, t, thr_lo, thr_hi);
  if (H.L.degenerate) {
    und_out = false;
    return 0;
  }
  int cnt = 0;
  bool und = false;
  for (int k = threadIdx.x & 31; k < fc.n; k += 32) {
    const int d = fused_classify(fc, H, k, thr_lo, thr_hi);
    cnt += d == kIn;
    und |= d == kUndecided;
  }
  und_out = __any_sync(0xffffffffu, und);
  return warp_reduce(cnt, SumI());
}

// kSelect == false: the prep + score half only (prep_score mode): the warp
// writes what select_warp_kernel reads -- xy64, the xy32 pairs, stat and the
// upper-bound counts -- and moves on; the hypotheses never leave registers.
struct PrepScoreOut {
  double2* xy64;
  float2* xy32;
  double4* stat;
  int32_t* upper;  // [C][Tg * 8]
  int Tg;
};

// Steps 1-2 of a fused warp and the slot's FP32 pairs: normalize, median,
// MAD interval (kWrite: xy64, stat and the xy32 pairs to HBM as well, for
// select_warp_kernel). The raw points are read once.
template <bool kWrite>
__device__ __forceinline__ void fused_prep_cluster(
    const double* __restrict__ caz, const double* __restrict__ cdop, int n, int64_t b, int c,
    double scale, const int64_t* __restrict__ offsets, double* xs, double* ys, float4* pairs,
    unsigned int* hist, unsigned long long* cand, int lane, const PrepScoreOut& ps,
    double& thr_lo, double& thr_hi, double& med) {
  constexpr bool kSelect = !kWrite;
  // ---- 1. load, min/max, normalize (src/ransac.cpp:69-87)
  int nb = 32;  // median buckets: about one per point, a power of two
  while (nb < n) nb <<= 1;
  for (int i = lane; i < nb; i += 32) hist[i] = 0;
  double lo0 = DBL_MAX, hi0 = -DBL_MAX, lo1 = DBL_MAX, hi1 = -DBL_MAX;
#pragma unroll 2
  for (int k = lane; k < n; k += 32) {
    const double a = __ldcs(caz + k), d = __ldcs(cdop + k);  // read once: streaming
    xs[k] = a;  // raw values, normalized in place below (same lane)
    ys[k] = d;
    lo0 = a < lo0 ? a : lo0;
    hi0 = a > hi0 ? a : hi0;
    lo1 = d < lo1 ? d : lo1;
    hi1 = d > hi1 ? d : hi1;
  }
  warp_minmax2(lo0, hi0, lo1, hi1);  // the loop above never takes a NaN
  __syncwarp();  // the zeroed buckets and the raw slot before any other lane uses them
  if (lo0 == 0.0 || hi0 == 0.0 || lo1 == 0.0 || hi1 == 0.0) {
    lo0 = warp_first_zero(lo0, xs, n, lane);
    hi0 = warp_first_zero(hi0, xs, n, lane);
    lo1 = warp_first_zero(lo1, ys, n, lane);
    hi1 = warp_first_zero(hi1, ys, n, lane);
  }
  const double s0 = __dsub_rn(hi0, lo0);
  const double s1 = __dsub_rn(hi1, lo1);
  {
    const bool f0 = div_span_ok(s0), f1 = div_span_ok(s1);
    const double r0 = f0 ? fast_rcp(s0) : 0.0, r1 = f1 ? fast_rcp(s1) : 0.0;
    for (int k = lane; k < n; k += 32) {
      const double x = s0 == 0.0 ? 0.5
                       : (f0 ? div_rn_shared(__dsub_rn(xs[k], lo0), s0, r0)
                             : __ddiv_rn(__dsub_rn(xs[k], lo0), s0));
      const double y = s1 == 0.0 ? 0.5
                       : (f1 ? div_rn_shared(__dsub_rn(ys[k], lo1), s1, r1)
                             : __ddiv_rn(__dsub_rn(ys[k], lo1), s1));
      xs[k] = x;
      ys[k] = y;
      if (!kSelect) ps.xy64[b + k] = make_double2(x, y);
      atomicAdd(&hist[med_bin(fused_key(ys, k), nb)], 1u);
    }
  }
  __syncwarp();

  // ---- 2. median (ransac.hpp:53-70) and the MAD interval (prep_cluster)
  {
    const int k0 = (n & 1) ? n / 2 : n / 2 - 1;
    unsigned long long v0 = 0, v1 = 0;
    fused_select_pair(ys, hist, cand, n, k0, (n & 1) == 0, nb, lane, v0, v1);
    const double d0 = __longlong_as_double(static_cast<long long>(v0));
    med = (n & 1) ? d0
                  : __ddiv_rn(__dadd_rn(d0, __longlong_as_double(static_cast<long long>(v1))),
                              2.0);
    double part = 0.0;
    for (int k = lane; k < n; k += 32)
      part += fabs(__dsub_rn(__longlong_as_double(static_cast<long long>(fused_key(ys, k))), med));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double mid = scale * (part / n);
    const double delta = (4.0 * n + 16.0) * 0x1p-53;
    thr_lo = mid * (1.0 - delta);
    thr_hi = mid * (1.0 + delta);
    if (!kSelect && lane == 0) ps.stat[c] = make_double4(thr_lo, thr_hi, med, CUDART_NAN);
  }
  __syncwarp();  // cand and hist are free: the pairs and the upper bounds reuse them
  // FP32 point pairs (x_2q, x_2q+1, y_2q, y_2q+1) for the scoring loop;
  // odd n padded with an inert point, plus the loop's read-ahead slack
  {
    const int m2 = (n + 1) >> 1;
    for (int q = lane; q < m2 + 3; q += 32) {
      float4 v = make_float4(0.f, 0.f, kPadY, kPadY);
      const int k0 = 2 * q, k1 = 2 * q + 1;
      if (k0 < n) {
        v.x = __double2float_rn(xs[k0]);
        v.z = __double2float_rn(ys[k0]);
      }
      if (k1 < n) {
        v.y = __double2float_rn(xs[k1]);
        v.w = __double2float_rn(ys[k1]);
      }
      pairs[q] = v;
      if (!kSelect && q < m2)  // the same pair layout as xy32_put's
        reinterpret_cast<float4*>(ps.xy32 + xy32_base(offsets, c))[q] = v;
    }
  }
  __syncwarp();

}

// Step 3 for one block of 256 trials: lane j builds trials tb + 8j .. +7 in
// registers and scores them against the slot's point pairs -> cnt[q].
__device__ __forceinline__ void fused_score_block(int tb, int T, uint64_t seed, uint64_t k1,
                                              int n, const double* xs, const double* ys,
                                              const float4* pairs, double thr_lo,
                                              double thr_hi, int lane,
                                              uint32_t (&cnt)[kNH]) {
  const int m2 = (n + 1) >> 1;
  float A[kNH], B[kNH];
  float2 Cc[kNH], T2[kNH];
  // kHU trials per step (independent chains), the code of one step once:
  // the step's trials enter at slots kNH-kHU.. and the registers rotate
  // down by kHU, so slot q holds trial 8 lane + q at the end (static
  // register indices; rotating one trial at a time cost 336 moves per
  // lane and block, measured)
#ifndef RVK_FUSED_HU  // A/B builds (RVK_NVCC_FLAGS)
#define RVK_FUSED_HU 4
#endif
  constexpr int kHU = RVK_FUSED_HU;
#pragma unroll 1
  for (int q0 = 0; q0 < kNH; q0 += kHU) {
    FastHyp f[kHU];
#pragma unroll
    for (int u = 0; u < kHU; ++u) {
      const int t = tb + 8 * lane + q0 + u;
      f[u] = inert_fast();
      if (t < T) {
        int i, j;
        seed_pair_k(seed, k1, static_cast<uint32_t>(t), static_cast<uint32_t>(n), i, j);
        f[u] = make_fast_from_seeds(xs[i], ys[i], xs[j], ys[j], thr_lo, thr_hi);
      }
    }
#pragma unroll
    for (int r = 0; r + kHU < kNH; ++r) {
      A[r] = A[r + kHU];
      B[r] = B[r + kHU];
      Cc[r] = Cc[r + kHU];
      T2[r] = T2[r + kHU];
    }
#pragma unroll
    for (int u = 0; u < kHU; ++u) {
      A[kNH - kHU + u] = f[u].A;
      B[kNH - kHU + u] = f[u].B;
      Cc[kNH - kHU + u] = make_float2(f[u].C, f[u].C);
      T2[kNH - kHU + u] = make_float2(-f[u].t2hi, -f[u].t2hi);
    }
  }
#pragma unroll
  for (int q = 0; q < kNH; ++q) cnt[q] = 0;
  auto g_of = [&](const float4& v, int h) {
    const float2 X = make_float2(v.x, v.y), Y = make_float2(v.z, v.w);
    const float2 e = __ffma2_rn(X, make_float2(A[h], A[h]),
                                __ffma2_rn(Y, make_float2(B[h], B[h]), Cc[h]));
    return __ffma2_rn(e, e, T2[h]);
  };
  // four pairs per iteration; the padded slack is inert (e^2 overflows)
#pragma unroll 1
  for (int q2 = 0; q2 < m2; q2 += 4) {
    const float4 v0 = pairs[q2], v1 = pairs[q2 + 1], v2 = pairs[q2 + 2], v3 = pairs[q2 + 3];
    if (RVK_FUSED_SIGN_PRMT) {
#pragma unroll
      for (int h = 0; h < kNH; ++h) {
        cnt[h] += sign_pair(g_of(v0, h)) + sign_pair(g_of(v1, h));
        cnt[h] += sign_pair(g_of(v2, h)) + sign_pair(g_of(v3, h));
      }
    } else {
      auto score_pair = [&](const float4& v) {
#pragma unroll
        for (int h = 0; h < kNH; ++h) {
          const float2 g = g_of(v, h);
          cnt[h] += (__float_as_uint(g.x) >> 31) + (__float_as_uint(g.y) >> 31);
        }
      };
      score_pair(v0);
      score_pair(v1);
      score_pair(v2);
      score_pair(v3);
    }
  }
  if (RVK_FUSED_SIGN_PRMT) {
#pragma unroll
    for (int q = 0; q < kNH; ++q) cnt[q] = sign_pair_count(cnt[q]);
  }
}

template <bool kSelect, class G, int kMinBlocks>
__global__ void __launch_bounds__(kFusedWarps * 32, kMinBlocks)
fused_warp_kernel(int32_t n_clusters, const int64_t* __restrict__ offsets,
                  const double* __restrict__ az, const double* __restrict__ dop, double scale,
                  const int32_t* __restrict__ keys, const int32_t* __restrict__ cluster_ids,
                  int64_t frame_id, int T, uint64_t seed, int32_t* __restrict__ out_count,
                  int32_t* __restrict__ out_trial, uint8_t* __restrict__ mask,
                  rvk_estimate* __restrict__ est, int32_t* __restrict__ big_list,
                  int32_t* big_ctl, PrepScoreOut ps) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* slot = fused_dyn + G::slot * wib;
  double* xs = reinterpret_cast<double*>(slot + G::x);
  double* ys = reinterpret_cast<double*>(slot + G::y);
  float4* pairs = reinterpret_cast<float4*>(slot + G::p);
  float2* p32 = reinterpret_cast<float2*>(slot + G::p);  // xy32_put / xy32_get layout
  unsigned int* hist = reinterpret_cast<unsigned int*>(slot + G::h);
  uint16_t* upper = reinterpret_cast<uint16_t*>(slot + G::h);
  unsigned long long* cand = reinterpret_cast<unsigned long long*>(slot + G::p);
  const bool refit = est != nullptr;
  const int fused_T = !kSelect || T <= G::max_t;

#pragma unroll 1
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&big_ctl[2], 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= n_clusters) break;
    const int64_t b = offsets[c];
    const int n = static_cast<int>(offsets[c + 1] - b);
    if (n < kMinClusterPoints) {
      if (kSelect)  // (prep_score mode: select_warp_kernel writes the sentinel)
        write_too_small(c, n, frame_id, cluster_ids ? cluster_ids[c] : c, out_count, out_trial,
                        mask + b, est, lane, 32);
      continue;
    }
    if (n > G::cap || !fused_T) {  // the CTA path takes it
      if (lane == 0) big_list[atomicAdd(&big_ctl[0], 1)] = c;
      continue;
    }
    const double* caz = az + b;
    const double* cdop = dop + b;

    double thr_lo, thr_hi, med;
    fused_prep_cluster<!kSelect>(caz, cdop, n, b, c, scale, offsets, xs, ys, pairs, hist, cand,
                                 lane, ps, thr_lo, thr_hi, med);

    // ---- 3. hypotheses + FP32 upper-bound scoring, 256 trials per block
    const uint32_t key = keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c);
    const uint64_t k1 = seed_key(key);
    unsigned long long vbest = 0;
#pragma unroll 1
    for (int tb = 0; tb < T; tb += 8 * 32) {
      uint32_t cnt[kNH];
      fused_score_block(tb, T, seed, k1, n, xs, ys, pairs, thr_lo, thr_hi, lane, cnt);
      if (!kSelect) {  // this warp saw every point: plain stores, trials padded to 8
        int32_t* gu = ps.upper + static_cast<int64_t>(c) * ps.Tg * 8;
        if (8 * (tb / 8 + lane) < ps.Tg * 8) {
          int4* g4 = reinterpret_cast<int4*>(gu + tb + 8 * lane);
          g4[0] = make_int4(cnt[0], cnt[1], cnt[2], cnt[3]);
          g4[1] = make_int4(cnt[4], cnt[5], cnt[6], cnt[7]);
        }
#pragma unroll
        for (int q = 0; q < kNH; ++q)
          if (tb + 8 * lane + q < T)
            vbest = MaxU64()(vbest, pack_best(static_cast<int>(cnt[q]), tb + 8 * lane + q));
        continue;
      }
#pragma unroll
      for (int q = 0; q < kNH; ++q) {
        const int t = tb + 8 * lane + q;
        if (t < T) {
          upper[t] = static_cast<uint16_t>(cnt[q]);
          vbest = MaxU64()(vbest, pack_best(static_cast<int>(cnt[q]), t));
        }
      }
    }
    if (!kSelect) {  // select_warp_kernel takes it from here, t0 and u0 in stat.w
      vbest = warp_reduce(vbest, MaxU64());
      if (lane == 0) ps.stat[c].w = pack_t0(unpack_trial(vbest), unpack_count(vbest));
      __syncwarp();
      continue;
    }
    vbest = warp_reduce(vbest, MaxU64());
    __syncwarp();  // upper[] visible to the whole warp
    const int t0 = unpack_trial(vbest);
    const int u0 = unpack_count(vbest);

    // ---- 4. exact winner, mask, refit (select_warp_kernel on the slot)
    const FusedCluster fc{xs, ys, p32, caz, cdop, mask + b, n, key, seed, refit};
    auto pass = [&](int t, int& count, RefitAcc& total) -> bool {
      return fused_pass(fc, t, thr_lo, thr_hi, count, total);
    };
    auto exact_count = [&](int t, bool& und) -> int {
      return fused_exact_count(fc, t, thr_lo, thr_hi, und);
    };
    auto go_exact = [&]() {  // the exact sequential threshold (rare)
      double t = 0.0;
      if (lane == 0) t = fused_exact_threshold(ys, n, med, scale);
      thr_lo = thr_hi = __shfl_sync(0xffffffffu, t, 0);
    };
    int e0 = 0;
    RefitAcc tot;
    if (!pass(t0, e0, tot)) {
      go_exact();
      pass(t0, e0, tot);
    }
    unsigned long long best = pack_best(e0, t0);
    if (u0 > e0) {  // verify the trials that could still win
      for (int round = 0; round < 2; ++round) {
        bool need_exact = false;
        for (int tb = 0; tb < T; tb += 32) {
          const int tl = tb + lane;
          const int u = tl < T ? static_cast<int>(upper[tl]) : -1;
          unsigned cand_m = __ballot_sync(
              0xffffffffu, tl < T && tl != t0 && !(u < e0 || (u == e0 && tl > t0)));
          while (cand_m) {
            const int t = tb + __ffs(cand_m) - 1;
            cand_m &= cand_m - 1;
            bool und;
            const int e = exact_count(t, und);
            if (und) need_exact = true;
            else best = MaxU64()(best, pack_best(e, t));
          }
        }
        if (need_exact && round == 0) {
          go_exact();  // redo every candidate (and t0) with the exact threshold
          pass(t0, e0, tot);
          best = pack_best(e0, t0);
          continue;
        }
        break;
      }
    }
    const int win = unpack_trial(best);
    const int win_count = unpack_count(best);
    if (win != t0) {  // another trial won: its mask and refit sums
      int cnt;
      if (!pass(win, cnt, tot)) {
        go_exact();
        pass(win, cnt, tot);
      }
    }
    if (lane == 0) {
      if (out_count) out_count[c] = win_count;
      if (out_trial) out_trial[c] = win;
      if (refit) finish_refit(tot, caz, cdop, frame_id, cluster_ids ? cluster_ids[c] : c, est + c);
    }
    __syncwarp();  // the slot is rewritten by the next cluster
  }
}

__global__ void __launch_bounds__(kSelectThreads)
refit_kernel(const int64_t* __restrict__ offsets, const double* __restrict__ az,
             const double* __restrict__ dop, const int32_t* __restrict__ cluster_ids,
             int64_t frame_id, const uint8_t* __restrict__ mask, rvk_estimate* __restrict__ est) {
  __shared__ RefitStage rst;
  const int c = blockIdx.x;
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  block_refit(n, az + b, dop + b, mask + b, frame_id, cluster_ids ? cluster_ids[c] : c, est + c,
              rst);
}

// Exact count of every (cluster, trial) (warp per trial). Requires the exact
// threshold in stat (mad_exact_kernel ran), so nothing is ever undecided.
__global__ void __launch_bounds__(kSelectThreads)
exact_counts_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ keys,
                    const double2* __restrict__ xy64, const float2* __restrict__ xy32,
                    const double4* __restrict__ stat, int T, uint64_t seed,
                    int32_t* __restrict__ counts) {
  const int c = blockIdx.x;
  const int64_t b = offsets[c];
  const int n = static_cast<int>(offsets[c + 1] - b);
  const uint32_t key = keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c);
  const double th = stat[c].w;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = warp; t < T; t += nw) {
    const ExactHyp H = make_exact(xy64 + b, seed, key, static_cast<uint32_t>(t), n, th, th);
    bool und;
    const int e = warp_exact_count(H, n, xy32 + xy32_base(offsets, c), xy64 + b, th, th, &und);
    if ((threadIdx.x & 31) == 0) counts[static_cast<int64_t>(c) * T + t] = e;
  }
}

// One output byte per thread: 8 mask bytes (one 8-byte load when the run
// is complete) -> 8 bits, LSB = the lowest point index.
__global__ void __launch_bounds__(256)
pack_mask_kernel(const uint8_t* __restrict__ mask, int64_t n_points, uint8_t* __restrict__ bits) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t k0 = i * 8;
  if (k0 >= n_points) return;
  uint32_t b = 0;
  if (k0 + 8 <= n_points && (reinterpret_cast<uintptr_t>(mask + k0) & 7) == 0) {
    const uint64_t v = *reinterpret_cast<const uint64_t*>(mask + k0);
#pragma unroll
    for (int q = 0; q < 8; ++q) b |= ((v >> (8 * q)) & 1u) << q;
  } else {
    for (int q = 0; q < 8 && k0 + q < n_points; ++q) b |= (mask[k0 + q] & 1u) << q;
  }
  bits[i] = static_cast<uint8_t>(b);
}

__global__ void seed_pairs_kernel(const int64_t* __restrict__ offsets,
                                  const int32_t* __restrict__ keys, int32_t n_clusters, int T,
                                  uint64_t seed, int32_t* __restrict__ pairs) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(n_clusters) * T) return;
  const int c = static_cast<int>(idx / T), t = static_cast<int>(idx % T);
  const int n = static_cast<int>(offsets[c + 1] - offsets[c]);
  int i, j;
  seed_pair(seed, keys ? static_cast<uint32_t>(keys[c]) : static_cast<uint32_t>(c),
            static_cast<uint32_t>(t), static_cast<uint32_t>(n), i, j);
  pairs[2 * idx] = i;
  pairs[2 * idx + 1] = j;
}

}  // namespace

// ---------------------------------------------------------------- launchers

// Per-cluster CTA shape: many small clusters run best with small CTAs (more
// clusters in flight per SM, fewer threads idling at every block barrier);
// large ones with 256 threads. Chosen from the mean cluster size; the
// kernels are correct for any cluster size at any shape (clusters larger
// than the shared-memory cap take the global-memory selection path).
struct CtaShape {
  int threads;
  int cap;  // shared-memory sort capacity (points)
};
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
// Measured on B200 (profiles/r1d_summary.md, r1e): prep wants 128 threads for
// clusters of ~200 points and 256 above ~400; select 64 for ~200 points, 128
// for ~600.
CtaShape cluster_cta_shape(int64_t n_points, int32_t n_clusters, const char* env, bool select) {
  const int64_t avg = n_clusters ? n_points / n_clusters : 0;
  int t = select ? (avg < 384 ? 64 : (avg < 1024 ? 128 : 256)) : (avg < 384 ? 128 : 256);
  // a call with few clusters (one frame): twice the threads per cluster,
  // the largest cluster's chain is the latency (measured, tools/frame_latency.py)
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  if (avg >= 384 && n_clusters <= 2 * sms) t = select ? 256 : 512;
  t = env_int(env, t);
  const int tmax = select ? 256 : 512;
  t = t <= 32 ? 32 : (t <= 64 ? 64 : (t <= 128 ? 128 : (t <= 256 ? 256 : tmax)));
  int cap = std::max(512, t * 8);
  if (!select) cap = env_int("RVK_PREP_CAP", cap);
  // >= 512: prep_cluster's reduction scratch; multiple of 32: 16-byte
  // aligned histogram
  cap = std::min(2048, std::max(512, cap)) & ~31;
  return {t, cap};
}

void launch_prep(const FrameDev& f, double scale, const Scratch& s, cudaStream_t st) {
  if (f.n_clusters == 0) return;
  const CtaShape sh = cluster_cta_shape(f.n_points, f.n_clusters, "RVK_PREP_THREADS", false);
  prep_kernel<<<f.n_clusters, std::min(sh.threads, kPrepThreads), prep_dyn_bytes(sh.cap), st>>>(
      f.n_clusters, f.offsets, f.azimuth, f.doppler, scale, s.xy64, s.xy32, s.stat, s.norm,
      sh.cap);
  count_launch();
}

void launch_mad_exact(const FrameDev& f, double scale, const Scratch& s, cudaStream_t st) {
  if (f.n_clusters == 0) return;
  mad_exact_kernel<<<(f.n_clusters + 7) / 8, 256, 0, st>>>(f.n_clusters, f.offsets, s.xy64,
                                                           scale, s.stat);
  count_launch();
}

int sm_count() {
  static const int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

// The fused warp-per-cluster kernel removes every intermediate HBM round
// trip and two launches, but on full batches it is slower on B200 than the
// three-kernel pipeline -- config 4, 4 frames: 0.42 vs 0.35 ms -- because
// warps in different phases of the ~7.5k-instruction kernel thrash the
// instruction cache (ncu: stall_no_instruction is its top stall reason, 3.0
// cycles per issue; profiles/r2_fused_summary.md). For a call of at most one
// imaging frame of small clusters the single launch wins (config 4, one
// frame: 0.135 vs 0.147 ms; config 1: 0.034 vs 0.037 ms), so it is chosen
// for those; RVK_FUSED=1/0 forces it on/off.
constexpr int kFusedAutoMaxClusters = 6144;
bool fused_path(const FrameDev& f, const rvk_ransac_params& p) {
  if (f.n_clusters == 0 || p.max_trials > kFusedMaxT) return false;
  static const int forced = env_int("RVK_FUSED", -1);
  if (forced >= 0) return forced != 0;
  const int64_t avg = f.n_points / f.n_clusters;
  return avg < 384 && f.n_clusters <= kFusedAutoMaxClusters;
}

// Whether the CTA path has clusters to take after the fused kernel: unknown
// (device-side sizes) unless the host passed the largest cluster size.
bool fused_leaves_big(const FrameDev& f, int cap = kFusedCap) {
  return f.max_cluster < 0 || f.max_cluster > cap;
}

// Prep + score fused per warp for the clusters of <= 384 points (the
// hypotheses go from registers straight into the scoring loop; the
// latency-bound prep of some warps overlaps the FMA-bound scoring of the
// others), select by select_warp_kernel, larger clusters by the CTA path.
// Measured on B200 (bench.py, 16 frames per step): config 4 step 1.263 ->
// 1.169 ms at T = 256, 3.190 -> 2.979 ms at T = 1024. The default takes it
// for calls whose mean cluster is small (as the warp prep it replaces);
// RVK_PREP_SCORE=1/0 forces it on/off.
bool prep_score_path(const FrameDev& f, const rvk_ransac_params& p) {
  if (f.n_clusters == 0 || fused_path(f, p)) return false;
  static const int forced = env_int("RVK_PREP_SCORE", -1);
  if (forced >= 0) return forced != 0;
  const int64_t avg = f.n_points / f.n_clusters;
  return avg < 384;
}

int fused_resident_ctas(bool select);

void launch_prep_score(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                       cudaStream_t st) {
  if (f.n_clusters == 0) return;
  ScoreGeom g = score_geom(p.max_trials);
  cudaMemsetAsync(s.big_ctl, 0, sizeof(int32_t) * 4, st);

  const int64_t want = (static_cast<int64_t>(f.n_clusters) + kFusedWarps - 1) / kFusedWarps;
  const int grid = static_cast<int>(std::min<int64_t>(fused_resident_ctas(false), want));
  const PrepScoreOut ps{s.xy64, s.xy32, s.stat, s.upper, g.Tg};
  fused_warp_kernel<false, FusedPrepScore, RVK_FUSED_PS_MINB><<<grid, kFusedWarps * 32, FusedPrepScore::smem,
                                                 st>>>(
      f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, f.cluster_ids,
      f.frame_id, p.max_trials, p.rng_seed, nullptr, nullptr, nullptr, nullptr, s.big_list,
      s.big_ctl, ps);
  count_launch();
}

void launch_prep_hyps(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                      cudaStream_t st) {
  if (f.n_clusters == 0) return;
  ScoreGeom g = score_geom(p.max_trials);
  set_ppt(g, s.ppt);
  cudaMemsetAsync(s.tile_count, 0, sizeof(int32_t) * (kTileBuckets + 1), st);
  if (prep_score_path(f, p)) {  // the clusters launch_prep_score listed, by persistent CTAs
    if (!fused_leaves_big(f, FusedPrepScore::cap)) return;
    prep_hyp_kernel<256, 4><<<std::min<int64_t>(2 * sm_count(), f.n_clusters), 256,
                              prep_dyn_bytes(2048), st>>>(
        f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, g, p.rng_seed,
        s.xy64, s.xy32, s.stat, s.hyp, s.upper, s.tiles, s.tile_count, s.tile_cap, 2048,
        s.big_list, s.big_ctl);
    count_launch();
    return;
  }
  if (fused_path(f, p)) {
    // the clusters the fused kernel listed, by persistent CTAs
    if (!fused_leaves_big(f)) return;
    prep_hyp_kernel<256, 4><<<std::min<int64_t>(2 * sm_count(), f.n_clusters), 256,
                              prep_dyn_bytes(2048), st>>>(
        f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, g, p.rng_seed,
        s.xy64, s.xy32, s.stat, s.hyp, s.upper, s.tiles, s.tile_count, s.tile_cap, 2048,
        s.big_list, s.big_ctl);
    count_launch();
    return;
  }
  const CtaShape sh = cluster_cta_shape(f.n_points, f.n_clusters, "RVK_PREP_THREADS", false);
  const int64_t avg = f.n_points / f.n_clusters;
  if (env_int("RVK_PREP_WARP", avg < 384 ? 1 : 0) != 0) {
    // warp per cluster up to kWarpCap points; the rest by persistent CTAs
    cudaMemsetAsync(s.big_ctl, 0, sizeof(int32_t) * 4, st);
    prep_warp_kernel<<<(f.n_clusters + kPrepWarps - 1) / kPrepWarps, kPrepWarps * 32, 0, st>>>(
        f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, g, p.rng_seed,
        s.xy64, s.xy32, s.stat, s.hyp, s.upper, s.tiles, s.tile_count, s.tile_cap,
        s.big_list, s.big_ctl);
    count_launch();
    prep_hyp_kernel<256, 4><<<std::min<int64_t>(2 * sm_count(), f.n_clusters), 256,
                              prep_dyn_bytes(2048), st>>>(
        f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, g, p.rng_seed,
        s.xy64, s.xy32, s.stat, s.hyp, s.upper, s.tiles, s.tile_count, s.tile_cap, 2048,
        s.big_list, s.big_ctl);
    count_launch();
    return;
  }
  auto k = sh.threads > 256 ? prep_hyp_kernel<512, 2> : prep_hyp_kernel<256, 4>;
  k<<<f.n_clusters, sh.threads, prep_dyn_bytes(sh.cap), st>>>(
      f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, g, p.rng_seed,
      s.xy64, s.xy32, s.stat, s.hyp, s.upper, s.tiles, s.tile_count, s.tile_cap, sh.cap, nullptr,
      nullptr);
  count_launch();
}

namespace {
// Persistent grid: every SM filled to the scoring kernel's occupancy.
int score_resident_ctas() {
  static int grid = 0;
  if (grid == 0) {
    int per_sm = 0;
    cudaFuncSetAttribute(score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kScoreSmemBytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score_kernel, kScoreThreads,
                                                  kScoreSmemBytes);
    per_sm = std::max(1, std::min(per_sm, env_int("RVK_SCORE_CTAS", per_sm)));
    grid = sm_count() * per_sm;
  }
  return grid;
}
int score_grid(int64_t max_units) {
  const int grid = score_resident_ctas();
  const int64_t warps_per_cta = kScoreThreads / 32;
  return static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(grid, (max_units + warps_per_cta - 1) / warps_per_cta)));
}
}  // namespace

int fused_resident_ctas(bool select) {
  static int grid[2] = {0, 0};
  int& g = grid[select ? 1 : 0];
  if (g == 0) {
    int per_sm = 0;
    auto k = select ? fused_warp_kernel<true, FusedFull, 4>
                    : fused_warp_kernel<false, FusedPrepScore, RVK_FUSED_PS_MINB>;
    const size_t smem = select ? FusedFull::smem : FusedPrepScore::smem;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kFusedWarps * 32, smem);
    per_sm = std::max(1, std::min(per_sm, env_int("RVK_FUSED_CTAS", per_sm)));
    g = sm_count() * per_sm;
  }
  return g;
}

int score_ppt(const ScoreGeom& g, int64_t n_points, int32_t n_clusters) {
  static const int forced = env_int("RVK_SCORE_PPT", 0);
  if (forced > 0) {  // a power of two in [16, kScorePPT]
    int ppt = 16;
    while (ppt < forced && ppt < kScorePPT) ppt <<= 1;
    return ppt;
  }
  const int64_t warps = static_cast<int64_t>(score_resident_ctas()) * (kScoreThreads / 32);
  int ppt = kScorePPT;  // at least two units per resident warp (measured, one frame of config 2)
  while (ppt > 32 && static_cast<int64_t>(g.nhb) * (n_points / ppt + n_clusters) < 2 * warps)
    ppt >>= 1;
  return ppt;
}

void launch_fused(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                  const Outputs& o, cudaStream_t st) {
  if (f.n_clusters == 0) return;
  cudaMemsetAsync(s.big_ctl, 0, sizeof(int32_t) * 4, st);
  const int64_t want = (static_cast<int64_t>(f.n_clusters) + kFusedWarps - 1) / kFusedWarps;
  const int grid = static_cast<int>(std::min<int64_t>(fused_resident_ctas(true), want));
  fused_warp_kernel<true, FusedFull, 4><<<grid, kFusedWarps * 32, FusedFull::smem, st>>>(
      f.n_clusters, f.offsets, f.azimuth, f.doppler, p.threshold_scale, f.keys, f.cluster_ids,
      f.frame_id, p.max_trials, p.rng_seed, o.inlier_count, o.winning_trial, o.mask, o.est,
      s.big_list, s.big_ctl, PrepScoreOut{});
  count_launch();
}

void launch_score(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                  cudaStream_t st) {
  if (f.n_clusters == 0) return;
  if (fused_path(f, p) && !fused_leaves_big(f)) return;
  if (prep_score_path(f, p) && !fused_leaves_big(f, FusedPrepScore::cap)) return;
  ScoreGeom g = score_geom(p.max_trials);
  set_ppt(g, s.ppt);
  const int64_t max_units = static_cast<int64_t>(g.nhb) * (f.n_points / g.ppt + f.n_clusters);
  const bool listed = fused_path(f, p) || prep_score_path(f, p);
  score_kernel<<<score_grid(max_units), kScoreThreads, kScoreSmemBytes, st>>>(
      s.tile_count, s.tiles, s.tile_cap, s.xy32, s.hyp, g, s.upper,
      listed ? s.big_ctl : nullptr);
  count_launch();
}

void launch_select(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                   const Outputs& o, cudaStream_t st) {
  if (f.n_clusters == 0) return;
  const int64_t avg = f.n_points / f.n_clusters;
  if (fused_path(f, p)) {  // the CTA path's share: the listed clusters
    if (!fused_leaves_big(f)) return;
    select_kernel<<<std::min<int64_t>(2 * sm_count(), f.n_clusters), 256, 0, st>>>(
        f.offsets, f.azimuth, f.doppler, f.keys, f.cluster_ids, f.frame_id, s.xy64, s.xy32,
        s.stat, p.threshold_scale, s.upper, p.max_trials, p.rng_seed, o.inlier_count,
        o.winning_trial, o.mask, o.est, s.big_list, s.big_ctl);
    count_launch();
    return;
  }
  if (prep_score_path(f, p) || env_int("RVK_SELECT_WARP", avg < 384 ? 1 : 0) != 0) {
    select_warp_kernel<<<(f.n_clusters + kSelectWarps - 1) / kSelectWarps, kSelectWarps * 32,
                         kSelSmem, st>>>(f.n_clusters, f.offsets, f.azimuth, f.doppler, f.keys,
                               f.cluster_ids, f.frame_id, s.xy64, s.xy32, s.stat,
                               p.threshold_scale, s.upper, p.max_trials, p.rng_seed,
                               o.inlier_count, o.winning_trial, o.mask, o.est);
    count_launch();
    return;
  }
  const CtaShape sh = cluster_cta_shape(f.n_points, f.n_clusters, "RVK_SELECT_THREADS", true);
  select_kernel<<<f.n_clusters, sh.threads, 0, st>>>(
      f.offsets, f.azimuth, f.doppler, f.keys, f.cluster_ids, f.frame_id, s.xy64, s.xy32, s.stat,
      p.threshold_scale, s.upper, p.max_trials, p.rng_seed, o.inlier_count, o.winning_trial,
      o.mask, o.est, nullptr, nullptr);
  count_launch();
}

void launch_refit(const FrameDev& f, const uint8_t* mask, rvk_estimate* est, cudaStream_t st) {
  if (f.n_clusters == 0) return;
  refit_kernel<<<f.n_clusters, kSelectThreads, 0, st>>>(f.offsets, f.azimuth, f.doppler,
                                                        f.cluster_ids, f.frame_id, mask, est);
  count_launch();
}

void launch_exact_counts(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                         int32_t* counts, cudaStream_t st) {
  if (f.n_clusters == 0) return;
  exact_counts_kernel<<<f.n_clusters, kSelectThreads, 0, st>>>(
      f.offsets, f.keys, s.xy64, s.xy32, s.stat, p.max_trials, p.rng_seed, counts);
  count_launch();
}

void launch_pack_mask(const uint8_t* mask, int64_t n_points, uint8_t* bits, cudaStream_t st) {
  const int64_t nb = (n_points + 7) / 8;
  if (nb == 0) return;
  pack_mask_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, st>>>(mask, n_points, bits);
  count_launch();
}

void launch_seed_pairs(const FrameDev& f, const rvk_ransac_params& p, int32_t* pairs,
                       cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(f.n_clusters) * p.max_trials;
  if (total == 0) return;
  seed_pairs_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      f.offsets, f.keys, f.n_clusters, p.max_trials, p.rng_seed, pairs);
  count_launch();
}

}  // namespace rvk_gpu
