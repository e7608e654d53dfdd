// Device-side building blocks shared by the sm_100a kernels (rvk_kernels.cu).
//
// Exactness contract: every quantity the reference
// computes in FP64 and that feeds a discrete decision (normalized
// coordinates, median, MAD threshold, line (m, c, den), point distance) is
// recomputed here with explicit round-to-nearest intrinsics (__dadd_rn,
// __dmul_rn, __ddiv_rn, __dsqrt_rn) in the reference's operation order, so no
// FMA contraction can change a bit. The FP32 fast filter is only ever used
// with a rigorous guard band; anything inside the band is decided by the
// exact FP64 sequence.
#pragma once

#include <cstdint>

namespace rvk_dev {

constexpr double kSeedEpsilon = 1e-12;          // include/rvk/ransac.hpp:17
constexpr double kRankEpsilon = 1e-8;           // include/rvk/velocity.hpp:18
constexpr double kZeroVelocityEpsilon = 1e-9;   // include/rvk/velocity.hpp:21
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;  // include/rvk/rng.hpp:58
constexpr double kPi = 3.141592653589793238462643383279502884;

// ---- KeyedRng (include/rvk/rng.hpp:16-67), bit-for-bit ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// High 64 bits of z * n for a 32-bit n (== __umul64hi(z, n)) in two
// IMAD.WIDE.U32: floor(z n / 2^64) = floor((zh n + floor(zl n / 2^32)) / 2^32),
// and zh n + (zl n >> 32) < 2^64.
__device__ __forceinline__ uint32_t mulhi_64x32(uint64_t z, uint32_t n) {
  const uint64_t lo = static_cast<uint64_t>(static_cast<uint32_t>(z)) * n;
  const uint64_t t = (z >> 32) * static_cast<uint64_t>(n) + (lo >> 32);
  return static_cast<uint32_t>(t >> 32);
}

// draw_seed_pair (src/ransac.cpp:111-123): KeyedRng(seed, (u32)cluster,
// (u32)trial); i = next_below(n); j = next_below(n-1), ++j if j >= i.
// next_below is the high word of the 64x32 product (rng.hpp:34-38).
// The trial-independent first step of the key (hoisted by per-cluster loops).
__device__ __forceinline__ uint64_t seed_key(uint32_t cluster) {
  return mix64(static_cast<uint64_t>(cluster) + kGamma);
}
// seed_pair with k1 = seed_key(cluster) precomputed.
__device__ __forceinline__ void seed_pair_k(uint64_t seed, uint64_t k1, uint32_t trial, uint32_t n,
                                            int& i, int& j) {
  const uint64_t k = mix64(k1 ^ static_cast<uint64_t>(trial));
  uint64_t state = mix64(k ^ seed);
  state += kGamma;
  const uint64_t z1 = mix64(state);
  state += kGamma;
  const uint64_t z2 = mix64(state);
  i = static_cast<int>(mulhi_64x32(z1, n));
  j = static_cast<int>(mulhi_64x32(z2, n - 1));
  if (j >= i) ++j;
}

__device__ __forceinline__ void seed_pair(uint64_t seed, uint32_t cluster, uint32_t trial,
                                          uint32_t n, int& i, int& j) {
  uint64_t k = mix64(static_cast<uint64_t>(cluster) + kGamma);
  k = mix64(k ^ static_cast<uint64_t>(trial));
  uint64_t state = mix64(k ^ seed);
  state += kGamma;
  const uint64_t z1 = mix64(state);
  state += kGamma;
  const uint64_t z2 = mix64(state);
  i = static_cast<int>(mulhi_64x32(z1, n));
  j = static_cast<int>(mulhi_64x32(z2, n - 1));
  if (j >= i) ++j;
}

// Line through the seeds in the normalized plane, exactly as run_trial
// (src/ransac.cpp:39-45): dx = x2 - x1; |dx| < eps -> degenerate;
// m = (y2 - y1) / dx; c = y1 - m * x1; den = sqrt(m * m + 1).
struct Line {
  double m, c, den;
  bool degenerate;
};

__device__ __forceinline__ Line make_line(double x1, double y1, double x2, double y2) {
  Line L;
  const double dx = __dsub_rn(x2, x1);
  L.degenerate = fabs(dx) < kSeedEpsilon;
  L.m = __ddiv_rn(__dsub_rn(y2, y1), dx);
  L.c = __dsub_rn(y1, __dmul_rn(L.m, x1));
  L.den = __dsqrt_rn(__dadd_rn(__dmul_rn(L.m, L.m), 1.0));
  return L;
}

// The reference's per-point decision (src/ransac.cpp:56-57):
// |(-m) * x + y - c| / den <= threshold, all FP64 round-to-nearest.
__device__ __forceinline__ bool exact_inlier(const Line& L, double x, double y, double thr) {
  const double r = __dsub_rn(__dadd_rn(__dmul_rn(-L.m, x), y), L.c);
  return __ddiv_rn(fabs(r), L.den) <= thr;
}

// The corridor half-width is known as an interval [thr_lo, thr_hi] that
// contains the reference's FP64 threshold exactly: the prep kernel sums the
// MAD deviations in parallel and bounds the difference to the reference's
// left-to-right sum (see prep_kernel); thr_lo == thr_hi once the exact
// sequential sum has been taken (exact_threshold()).

// FP32 affine form of the same distance, e = A x + B y + C with
// (A, B, C) = (-m, 1, -c) / den, and two squared corridor bounds:
//   e^2 <  t2lo  => certainly an inlier of the FP64 test,
//   e^2 >= t2hi  => certainly an outlier,
// otherwise the point is decided by exact_decide(). With x, y in [0, 1]
// the FP32 evaluation error of e is <= 4u * S, S = |A| + |B| + |C|,
// u = 2^-24, and the FP64 reference's own error is <= 4 * 2^-53 * S; the
// band 2^-21 * S (= 8u S) covers both with a factor ~2 margin, and the
// (1 -/+ 2^-30) factors cover the FP64 rounding of the squared bounds.
struct FastHyp {
  float A, B, C;
  float t2hi;  // e^2 < t2hi: possible inlier (upper-bound count)
  float t2lo;  // e^2 < t2lo: certain inlier
  float thi;   // |e| <= thi: possible inlier (linear form of t2hi, same band)
};

// Coefficients from (m, c) and r ~= 1/den. r may carry a few FP64 ulps of
// error (rsqrt in the setup kernel): that perturbs A, B, C by ~1e-16
// relative, far inside the band's factor-2 margin.
__device__ __forceinline__ FastHyp fast_coeffs(double m, double c, double r, double thr_lo,
                                               double thr_hi) {
  FastHyp h;
  const double A = -m * r;
  const double B = r;
  const double C = -c * r;
  const double S = fabs(A) + fabs(B) + fabs(C);
  const double band = S * 0x1p-21;
  h.A = __double2float_rn(A);
  h.B = __double2float_rn(B);
  h.C = __double2float_rn(C);
  const double hi = (thr_hi + band) * (1.0 + 0x1p-30);
  h.t2hi = __double2float_ru(hi * hi);
  h.thi = __double2float_ru(hi);
  if (thr_lo > band) {
    const double lo = (thr_lo - band) * (1.0 - 0x1p-30);
    h.t2lo = __double2float_rd(lo * lo);
  } else {
    h.t2lo = 0.f;  // e^2 < 0 never holds: no certain inliers
  }
  return h;
}

__device__ __forceinline__ FastHyp inert_fast() {
  FastHyp h;  // degenerate seeds score 0 (src/ransac.cpp:40-42): nothing passes
  h.A = h.B = h.C = 0.f;
  h.t2hi = -1.f;
  h.t2lo = -1.f;
  h.thi = -1.f;
  return h;
}

__device__ __forceinline__ FastHyp make_fast(const Line& L, double thr_lo, double thr_hi) {
  if (L.degenerate) return inert_fast();
  return fast_coeffs(L.m, L.c, __ddiv_rn(1.0, L.den), thr_lo, thr_hi);
}

// 1/d to ~1 FP64 ulp: the MUFU seed and two Newton steps (no IEEE divide).
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  return fma(r, fma(-d, r, 1.0), r);
}

// a / s rounded to nearest, bit-identical to __ddiv_rn(a, s), for a divisor
// s shared by many dividends (normalize_cluster's spans) with r ~= 1/s
// precomputed once: Markstein's correction step q1 = q0 + (a - s q0) r, then
// a verification -- q1 is the correctly rounded quotient iff
// |a - s q1| < ulp(q1)/2 * s (the residual is exact when q1 is within one ulp;
// a quotient can never lie exactly on a midpoint) -- and __ddiv_rn for the
// rare rest (zero or tiny quotients, failed checks). Requires
// s in [2^-60, 2^60] (div_span_ok) so that the scaled half-ulp is normal.
__device__ __forceinline__ bool div_span_ok(double s) {
  return s >= 0x1p-60 && s <= 0x1p60;
}
__device__ __forceinline__ double div_rn_shared(double a, double s, double r) {
  const double q0 = a * r;
  const double q1 = fma(fma(-q0, s, a), r, q0);
  const long long e = __double_as_longlong(q1) & 0x7ff0000000000000LL;  // biased exponent
  if (e >= (0x3ffLL - 900) << 52) {                                     // |q1| >= 2^-900
    const double half_ulp = __longlong_as_double(e - (53LL << 52));
    if (fabs(fma(-q1, s, a)) < half_ulp * s) return q1;
  }
  return __ddiv_rn(a, s);
}

// Fast-pass hypothesis straight from the seeds: the same line as make_line
// (degeneracy decided on the exact dx), but the slope by a refined
// reciprocal and 1/den by rsqrt instead of correctly rounded divides and sqrt
// -- a few FP64 ulps, far inside the guard band (see fast_coeffs); used where
// only the FP32 filter is needed. |dx| >= kSeedEpsilon keeps the
// reciprocal clear of the flush-to-zero range.
__device__ __forceinline__ FastHyp make_fast_from_seeds(double x1, double y1, double x2,
                                                        double y2, double thr_lo, double thr_hi) {
  const double dx = __dsub_rn(x2, x1);
  if (fabs(dx) < kSeedEpsilon) return inert_fast();
  const double m = __dsub_rn(y2, y1) * fast_rcp(dx);
  const double c = __dsub_rn(y1, __dmul_rn(m, x1));
  return fast_coeffs(m, c, rsqrt(__dadd_rn(__dmul_rn(m, m), 1.0)), thr_lo, thr_hi);
}

// Full per-hypothesis state for the exact (verification / mask) passes.
struct ExactHyp {
  Line L;
  FastHyp f;
  int a, b;
};

__device__ __forceinline__ ExactHyp make_exact(const double2* __restrict__ xy64, uint64_t seed,
                                               uint32_t key, uint32_t trial, int n,
                                               double thr_lo, double thr_hi) {
  ExactHyp H;
  seed_pair(seed, key, trial, static_cast<uint32_t>(n), H.a, H.b);
  const double2 p = xy64[H.a];
  const double2 q = xy64[H.b];
  H.L = make_line(p.x, p.y, q.x, q.y);
  H.f = make_fast(H.L, thr_lo, thr_hi);
  return H;
}

enum Decision : int { kOut = 0, kIn = 1, kUndecided = 2 };

// Exact inlier decision of point k for a non-degenerate hypothesis
// (run_trial, src/ransac.cpp:47-63: seeds counted without evaluation).
// kUndecided only when the FP64 distance falls inside [thr_lo, thr_hi],
// i.e. the threshold's last bits matter and the exact sequential MAD sum is
// needed.
__device__ __forceinline__ int classify(const ExactHyp& H, int k, float2 p32,
                                        const double2* __restrict__ xy64, double thr_lo,
                                        double thr_hi) {
  if (k == H.a || k == H.b) return kIn;
  const float e = __fmaf_rn(H.f.A, p32.x, __fmaf_rn(H.f.B, p32.y, H.f.C));
  if (__fmaf_rn(e, e, -H.f.t2lo) < 0.f) return kIn;
  if (!(__fmaf_rn(e, e, -H.f.t2hi) < 0.f)) return kOut;
  const double2 q = xy64[k];
  const double r = __dsub_rn(__dadd_rn(__dmul_rn(-H.L.m, q.x), q.y), H.L.c);
  const double d = __ddiv_rn(fabs(r), H.L.den);
  if (d <= thr_lo) return kIn;
  if (d > thr_hi) return kOut;
  return kUndecided;
}

// The reference's threshold bit for bit: mean_abs_deviation's left-to-right
// sum (include/rvk/ransac.hpp:74-84) then mad_threshold's scale
// (src/ransac.cpp:89-94). One thread; n dependent FP64 adds.
__device__ __forceinline__ double exact_threshold(const double2* xy64, int n, double med,
                                                  double scale) {
  double acc = 0.0;
  int k = 0;
  for (; k + 8 <= n; k += 8) {
    double d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = fabs(__dsub_rn(xy64[k + q].y, med));
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, d[q]);
  }
  for (; k < n; ++k) acc = __dadd_rn(acc, fabs(__dsub_rn(xy64[k].y, med)));
  return __dmul_rn(scale, __ddiv_rn(acc, static_cast<double>(n)));
}

// sin and cos of an azimuth for the LSQ design matrix (build_design_matrix,
// src/velocity.cpp:9-17, which takes Eigen's cos()/sin()). Azimuths are
// atan2 outputs in (-pi, pi] (src/scene.cpp, the frame reader's check), so
// the general range reduction of libdevice's sincos is not needed: one
// Cody-Waite step with the fdlibm split of pi/2 (|q| <= 2, FMA products
// exact) and the fdlibm kernel polynomials on [-pi/4, pi/4]: within
// 1.1e-16 absolute of libdevice's sincos over 4e8 points of [-4, 4]
// (tools/sincos_check.cu; the reference's own libm differs from any other by
// an ulp too, and the refit is tolerance-checked), in ~25 FP64
// instructions instead of ~60 plus table loads. Outside [-4, 4]: libdevice.
__device__ __forceinline__ void sincos_az(double x, double* s, double* c) {
  if (!(fabs(x) <= 4.0)) {
    sincos(x, s, c);
    return;
  }
  const double q = rint(x * 0.63661977236758134308);  // 2/pi
  double r = fma(-q, 1.57079632673412561417e+00, x);  // pi/2, first 33 bits
  r = fma(-q, 6.07710050650619224932e-11, r);          // next 33 bits
  r = fma(-q, 2.02226624879595063154e-21, r);          // tail
  const double z = r * r;
  const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10,
                                                      -2.50507602534068634195e-08),
                                               2.75573137070700676789e-06),
                                        -1.98412698298579493134e-04),
                                 8.33333333332248946124e-03),
                          -1.66666666666666324348e-01);
  const double sr = fma(r * z, ps, r);
  const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11,
                                                      2.08757232129817482790e-09),
                                               -2.75573143513906633035e-07),
                                        2.48015872894767294178e-05),
                                 -1.38888888888741095749e-03),
                          4.16666666666666019037e-02);
  const double cr = fma(z * z, pc, fma(-0.5, z, 1.0));
  const int iq = static_cast<int>(q) & 3;
  const double ss = (iq & 1) ? cr : sr, cc = (iq & 1) ? sr : cr;
  *s = (iq & 2) ? -ss : ss;
  *c = ((iq + 1) & 2) ? -cc : cc;
}

// Packs (count, trial) so that a max picks the largest count and, on ties,
// the lowest trial -- the ascending strict-> scan of src/ransac.cpp:181-189.
__device__ __forceinline__ unsigned long long pack_best(int count, int trial) {
  return (static_cast<unsigned long long>(static_cast<uint32_t>(count)) << 32) |
         static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(trial));
}
__device__ __forceinline__ int unpack_count(unsigned long long v) {
  return static_cast<int>(v >> 32);
}
__device__ __forceinline__ int unpack_trial(unsigned long long v) {
  return static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(v & 0xFFFFFFFFull));
}

}  // namespace rvk_dev
