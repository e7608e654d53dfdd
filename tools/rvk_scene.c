/*
 * Host-side synthetic frame generator (workload source for bench.py and the
 * tests; not on the accelerated path).
 *
 * Restates rvk::generate_frame (/root/reference/proj/src/scene.cpp:105-189)
 * and the KeyedRng it draws from (include/rvk/rng.hpp:16-67) so that for any
 * spec the reference accepts, the frame is bit-identical to the reference's
 * (tests/test_workloads.py checks this against oracle/_ref). Differences:
 *   - no spec validation (scene.cpp:34-64, :68-103); in particular
 *     outlier_fraction may reach 0.5, which BASELINE config 3 needs and the
 *     reference rejects (scene.cpp:39);
 *   - no noise points (the bench workloads take clusters from the truth
 *     table, src/bench.cpp:57-63, so n_noise_points = 0).
 * Object i's points are contiguous in the output, objects in order, exactly
 * as generate_frame lays them out.
 *
 * objects: n_objects rows of 10 doubles: center_x, center_y, extent_x,
 * extent_y, v_x, v_y, n_points, outlier_fraction, doppler_noise_sigma, unused.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define K_GAMMA 0x9E3779B97F4A7C15ull
#define K_PI 3.14159265358979323846

typedef struct {
  uint64_t s;
} krng;

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void krng_init(krng* r, uint64_t seed, uint64_t hi, uint64_t lo) {
  uint64_t k = mix(hi + K_GAMMA);
  k = mix(k ^ lo);
  r->s = mix(k ^ seed);
}
static uint64_t next_u64(krng* r) {
  uint64_t z = (r->s += K_GAMMA);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint32_t next_below(krng* r, uint32_t n) {
  return (uint32_t)(((unsigned __int128)next_u64(r) * n) >> 64);
}
static double next_unit(krng* r) { return (double)(next_u64(r) >> 11) * 0x1p-53; }
static double next_range(krng* r, double lo, double hi) { return lo + next_unit(r) * (hi - lo); }
static double next_gaussian(krng* r) {
  const double u1 = (double)((next_u64(r) >> 11) + 1) * 0x1p-53;
  const double u2 = next_unit(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * K_PI * u2);
}
static double half_open(double a) { return a == -K_PI ? K_PI : a; }

/* Public helpers so Python builds specs from the same stream (workloads.py). */
uint64_t rvk_scene_rng_u64(uint64_t seed, uint64_t hi, uint64_t lo, int32_t k) {
  krng r;
  krng_init(&r, seed, hi, lo);
  uint64_t v = 0;
  for (int32_t i = 0; i <= k; ++i) v = next_u64(&r);
  return v;
}

/* Fills n draws of next_unit() from KeyedRng(seed, hi, lo). */
void rvk_scene_rng_units(uint64_t seed, uint64_t hi, uint64_t lo, int64_t n, double* out) {
  krng r;
  krng_init(&r, seed, hi, lo);
  for (int64_t i = 0; i < n; ++i) out[i] = next_unit(&r);
}

int rvk_scene_generate(uint64_t seed, int32_t n_objects, const double* objects,
                       double offset_lo, double offset_hi, double* x, double* y, double* doppler,
                       double* azimuth, int32_t* outlier_flag) {
  int64_t first = 0;
  int32_t* idx = NULL;
  int64_t idx_cap = 0;
  for (int32_t i = 0; i < n_objects; ++i) {
    const double* o = objects + 10 * (int64_t)i;
    const int32_t n = (int32_t)o[6];
    krng rng;
    krng_init(&rng, seed, (uint64_t)i + 1, 0); /* scene.cpp:120: stream i+1 */
    for (int32_t k = 0; k < n; ++k) {          /* scene.cpp:124-132 */
      const int64_t q = first + k;
      x[q] = o[0] + o[2] * (next_unit(&rng) - 0.5);
      y[q] = o[1] + o[3] * (next_unit(&rng) - 0.5);
      azimuth[q] = half_open(atan2(y[q], x[q]));
      doppler[q] = o[4] * cos(azimuth[q]) + o[5] * sin(azimuth[q]); /* types.hpp:68-71 */
      if (outlier_flag) outlier_flag[q] = 0;
    }
    for (int32_t k = 0; k < n; ++k) /* scene.cpp:137-140 */
      doppler[first + k] += o[8] * next_gaussian(&rng);
    /* scene.cpp:143-151: partial Fisher-Yates prefix, sorted ascending */
    const int32_t m = (int32_t)floor(o[7] * n);
    if (n > idx_cap) {
      free(idx);
      idx_cap = n;
      idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)idx_cap);
    }
    for (int32_t k = 0; k < n; ++k) idx[k] = k;
    for (int32_t t = 0; t < m; ++t) {
      const int32_t pick = t + (int32_t)next_below(&rng, (uint32_t)(n - t));
      const int32_t tmp = idx[t];
      idx[t] = idx[pick];
      idx[pick] = tmp;
    }
    /* ascending order of the chosen prefix (std::sort) */
    uint8_t* chosen = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
    for (int32_t t = 0; t < m; ++t) chosen[idx[t]] = 1;
    for (int32_t local = 0; local < n; ++local) { /* scene.cpp:165-171 */
      if (!chosen[local]) continue;
      const double sign = next_unit(&rng) < 0.5 ? -1.0 : 1.0;
      const double magnitude = next_range(&rng, offset_lo, offset_hi);
      doppler[first + local] += sign * magnitude;
      if (outlier_flag) outlier_flag[first + local] = 1;
    }
    free(chosen);
    first += n;
  }
  free(idx);
  return 0;
}
