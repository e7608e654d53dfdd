/*
 * TEST INFRASTRUCTURE ONLY -- CPU checker, see rvk_oracle.h. Restates the
 * reference (/root/reference/proj) in C; every function cites the lines it
 * follows. Compiled with -ffp-contract=off and no -march (oracle/Makefile),
 * so each FP64 operation rounds exactly as in the reference build.
 */
#include "rvk_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_SEED_EPSILON 1e-12        /* include/rvk/ransac.hpp:17 */
#define K_RANK_EPSILON 1e-8         /* include/rvk/velocity.hpp:18 */
#define K_ZERO_VELOCITY_EPSILON 1e-9 /* include/rvk/velocity.hpp:21 */
#define K_MIN_CLUSTER_SIZE 3        /* include/rvk/types.hpp:20 */
#define K_GAMMA 0x9E3779B97F4A7C15ull /* include/rvk/rng.hpp:58 */
#define K_PI 3.14159265358979323846 /* std::numbers::pi, include/rvk/types.hpp:13 */

static _Thread_local char g_err[256];

const char* rvk_or_last_error(void) { return g_err; }

/* ---- KeyedRng, include/rvk/rng.hpp:16-67 ---- */

static uint64_t mix(uint64_t z) { /* rng.hpp:60-64 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void rvk_or_rng_init(rvk_or_rng* r, uint64_t seed, uint64_t hi, uint64_t lo) { /* rng.hpp:18-23 */
  uint64_t k = mix(hi + K_GAMMA);
  k = mix(k ^ lo);
  r->state = mix(k ^ seed);
}

uint64_t rvk_or_rng_next_u64(rvk_or_rng* r) { /* rng.hpp:25-30 */
  uint64_t z = (r->state += K_GAMMA);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint32_t rvk_or_rng_next_below(rvk_or_rng* r, uint32_t n) { /* rng.hpp:34-38 */
  const unsigned __int128 wide = (unsigned __int128)rvk_or_rng_next_u64(r) * n;
  return (uint32_t)(wide >> 64);
}

double rvk_or_rng_next_unit(rvk_or_rng* r) { /* rng.hpp:41 */
  return (double)(rvk_or_rng_next_u64(r) >> 11) * 0x1p-53;
}

double rvk_or_rng_next_range(rvk_or_rng* r, double lo, double hi) { /* rng.hpp:44-46 */
  return lo + rvk_or_rng_next_unit(r) * (hi - lo);
}

double rvk_or_rng_next_gaussian(rvk_or_rng* r) { /* rng.hpp:49-55 */
  const double u1 = (double)((rvk_or_rng_next_u64(r) >> 11) + 1) * 0x1p-53;
  const double u2 = rvk_or_rng_next_unit(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * K_PI * u2);
}

uint64_t rvk_or_rng_u64(uint64_t seed, uint64_t hi, uint64_t lo, int32_t k) {
  rvk_or_rng r;
  rvk_or_rng_init(&r, seed, hi, lo);
  uint64_t v = 0;
  for (int32_t i = 0; i <= k; ++i) v = rvk_or_rng_next_u64(&r);
  return v;
}

/* ---- draw_seed_pair, src/ransac.cpp:111-123 ---- */
int rvk_or_seed_pair(uint64_t seed, int32_t cluster, int32_t trial, int32_t n, int32_t* i,
                     int32_t* j) {
  if (n < 2) {
    snprintf(g_err, sizeof g_err, "draw_seed_pair: need at least 2 points");
    return RVK_EINVAL;
  }
  rvk_or_rng r;
  rvk_or_rng_init(&r, seed, (uint64_t)(uint32_t)cluster, (uint64_t)(uint32_t)trial);
  const int32_t a = (int32_t)rvk_or_rng_next_below(&r, (uint32_t)n);
  int32_t b = (int32_t)rvk_or_rng_next_below(&r, (uint32_t)(n - 1));
  if (b >= a) ++b;
  *i = a;
  *j = b;
  return RVK_OK;
}

/* ---- median / mean_abs_deviation, include/rvk/ransac.hpp:53-84 ---- */
static int cmp_double(const void* pa, const void* pb) {
  const double a = *(const double*)pa, b = *(const double*)pb;
  return (a > b) - (a < b);
}

static double median_of(const double* v, int64_t n, int64_t stride) { /* ransac.hpp:53-70 */
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) s[i] = v[i * stride];
  qsort(s, (size_t)n, sizeof(double), cmp_double);
  const int64_t mid = n / 2;
  const double m = (n % 2 == 1) ? s[mid] : (s[mid - 1] + s[mid]) / 2.0;
  free(s);
  return m;
}

static double mean_abs_deviation(const double* v, int64_t n, int64_t stride) { /* ransac.hpp:74-84 */
  const double med = median_of(v, n, stride);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) { /* sequential, index order */
    const double dev = v[i * stride] - med;
    acc += dev < 0.0 ? -dev : dev;
  }
  return acc / (double)n;
}

/* normalize_cluster (src/ransac.cpp:69-87) + mad_threshold (:234-239). */
double rvk_or_prepare_cluster(int64_t n, const double* az, const double* dop, double scale,
                              double* xy, double* norm4) {
  const double* axis_src[2] = {az, dop};
  for (int axis = 0; axis < 2; ++axis) {
    const double* v = axis_src[axis];
    double lo = v[0], hi = v[0];
    for (int64_t k = 1; k < n; ++k) { /* Eigen minCoeff/maxCoeff */
      lo = v[k] < lo ? v[k] : lo;
      hi = v[k] > hi ? v[k] : hi;
    }
    const double s = hi - lo;
    if (norm4) {
      norm4[axis] = lo;
      norm4[2 + axis] = s;
    }
    for (int64_t k = 0; k < n; ++k) xy[2 * k + axis] = (s == 0.0) ? 0.5 : (v[k] - lo) / s;
  }
  return scale * mean_abs_deviation(xy + 1, n, 2);
}

/* run_trial, src/ransac.cpp:32-65 (count_trial_inliers / evaluate_trial). */
int32_t rvk_or_run_trial(int64_t n, const double* xy, int32_t a, int32_t b, double thr,
                         uint8_t* mask) {
  const double x1 = xy[2 * a], y1 = xy[2 * a + 1];
  const double x2 = xy[2 * b], y2 = xy[2 * b + 1];
  const double dx = x2 - x1;
  if (fabs(dx) < K_SEED_EPSILON) return 0;
  const double m = (y2 - y1) / dx;
  const double c = y1 - m * x1;
  const double denom = sqrt(m * m + 1.0);
  int32_t count = 2;
  if (mask) {
    mask[a] = 1;
    mask[b] = 1;
  }
  for (int64_t k = 0; k < n; ++k) {
    if (k == a || k == b) continue;
    const double dist = fabs(-m * xy[2 * k] + xy[2 * k + 1] - c) / denom;
    if (dist <= thr) {
      ++count;
      if (mask) mask[k] = 1;
    }
  }
  return count;
}

static int validate(int32_t n_clusters, const int64_t* offsets, const rvk_ransac_params* p,
                    const char* who) {
  /* src/ransac.cpp:140-154 / src/baseline.cpp:13-27 */
  if (p->max_trials < 1) {
    snprintf(g_err, sizeof g_err, "%s: max_trials must be at least 1", who);
    return RVK_EINVAL;
  }
  if (!(p->threshold_scale > 0.0)) {
    snprintf(g_err, sizeof g_err, "%s: threshold_scale must be positive", who);
    return RVK_EINVAL;
  }
  for (int32_t c = 0; c < n_clusters; ++c) {
    const int64_t n = offsets[c + 1] - offsets[c];
    if (n < K_MIN_CLUSTER_SIZE) {
      snprintf(g_err, sizeof g_err, "%s: cluster %d has %lld points, need %d", who, c,
               (long long)n, K_MIN_CLUSTER_SIZE);
      return RVK_ECLUSTER_TOO_SMALL;
    }
  }
  return RVK_OK;
}

/* sequential_ransac, src/baseline.cpp:11-51, for one cluster. */
static void ransac_one(int64_t n, const double* az, const double* dop,
                       const rvk_ransac_params* p, int32_t key, int32_t* count, int32_t* trial,
                       uint8_t* mask, double* xy) {
  const double thr = rvk_or_prepare_cluster(n, az, dop, p->threshold_scale, xy, NULL);
  int32_t best_count = -1, best_trial = -1;
  for (int32_t t = 0; t < p->max_trials; ++t) {
    int32_t a, b;
    rvk_or_seed_pair(p->rng_seed, key, t, (int32_t)n, &a, &b);
    const int32_t cnt = rvk_or_run_trial(n, xy, a, b, thr, NULL);
    if (cnt > best_count) { /* strict >: lowest trial wins ties */
      best_count = cnt;
      best_trial = t;
    }
  }
  int32_t a, b;
  rvk_or_seed_pair(p->rng_seed, key, best_trial, (int32_t)n, &a, &b);
  if (mask) memset(mask, 0, (size_t)n);
  uint8_t* tmp = mask ? mask : (uint8_t*)calloc((size_t)n, 1);
  const int32_t cnt = rvk_or_run_trial(n, xy, a, b, thr, tmp); /* evaluate_trial */
  if (!mask) free(tmp);
  if (count) *count = cnt;
  if (trial) *trial = best_trial;
}

int rvk_or_sequential_ransac(int32_t n_clusters, const int64_t* offsets, const double* az,
                             const double* dop, const rvk_ransac_params* p,
                             const int32_t* key, int32_t* inlier_count, int32_t* winning_trial,
                             uint8_t* mask) {
  const int st = validate(n_clusters, offsets, p, "sequential_ransac");
  if (st != RVK_OK) return st;
  int64_t nmax = 0;
  for (int32_t c = 0; c < n_clusters; ++c)
    if (offsets[c + 1] - offsets[c] > nmax) nmax = offsets[c + 1] - offsets[c];
  double* xy = (double*)malloc(sizeof(double) * 2 * (size_t)(nmax > 0 ? nmax : 1));
  for (int32_t c = 0; c < n_clusters; ++c) {
    const int64_t b = offsets[c];
    ransac_one(offsets[c + 1] - b, az + b, dop + b, p, key ? key[c] : c,
               inlier_count ? inlier_count + c : NULL, winning_trial ? winning_trial + c : NULL,
               mask ? mask + b : NULL, xy);
  }
  free(xy);
  return RVK_OK;
}

int rvk_or_trial_counts(int32_t n_clusters, const int64_t* offsets, const double* az,
                        const double* dop, const rvk_ransac_params* p, const int32_t* key,
                        int32_t* counts) {
  const int st = validate(n_clusters, offsets, p, "run_ransac");
  if (st != RVK_OK) return st;
  for (int32_t c = 0; c < n_clusters; ++c) {
    const int64_t b = offsets[c], n = offsets[c + 1] - b;
    double* xy = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    const double thr = rvk_or_prepare_cluster(n, az + b, dop + b, p->threshold_scale, xy, NULL);
    for (int32_t t = 0; t < p->max_trials; ++t) {
      int32_t i, j;
      rvk_or_seed_pair(p->rng_seed, key ? key[c] : c, t, (int32_t)n, &i, &j);
      counts[(int64_t)c * p->max_trials + t] = rvk_or_run_trial(n, xy, i, j, thr, NULL);
    }
    free(xy);
  }
  return RVK_OK;
}

int rvk_or_cluster_thresholds(int32_t n_clusters, const int64_t* offsets, const double* az,
                              const double* dop, double scale, double* norm, double* thr,
                              double* normalized) {
  for (int32_t c = 0; c < n_clusters; ++c) {
    const int64_t b = offsets[c], n = offsets[c + 1] - b;
    if (n < 1) {
      snprintf(g_err, sizeof g_err, "normalize_cluster: empty cluster");
      return RVK_EINVAL;
    }
    double* xy = normalized ? normalized + 2 * b : (double*)malloc(sizeof(double) * 2 * (size_t)n);
    thr[c] = rvk_or_prepare_cluster(n, az + b, dop + b, scale, xy, norm ? norm + 4 * c : NULL);
    if (!normalized) free(xy);
  }
  return RVK_OK;
}

/* ---- velocity, src/velocity.cpp + include/rvk/velocity.hpp ---- */

static double to_half_open_angle(double a) { return a == -K_PI ? K_PI : a; } /* types.hpp:74-77 */

/* estimate_cluster_velocity, src/velocity.cpp:26-90. Reductions are
 * sequential in index order (Eigen squaredNorm/dot/mean). */
static void estimate_cluster(int64_t frame_id, int32_t cluster_id, int64_t n, const double* az,
                             const double* dop, const uint8_t* mask, rvk_estimate* est) {
  est->frame_id = frame_id;
  est->cluster_id = cluster_id;
  int64_t n_in = 0;
  for (int64_t k = 0; k < n; ++k) n_in += mask[k] ? 1 : 0;
  est->inlier_count = (int32_t)n_in;
  est->has_heading = 0;
  est->heading = 0.0;
  if (n_in == 0) { /* velocity.cpp:56-62 */
    est->v_x = 0.0;
    est->v_y = 0.0;
    est->condition_ok = 0;
    return;
  }
  if (n_in == 1) { /* velocity.cpp:63-67 */
    for (int64_t k = 0; k < n; ++k)
      if (mask[k]) {
        est->v_x = dop[k] * cos(az[k]);
        est->v_y = dop[k] * sin(az[k]);
      }
    est->condition_ok = 0;
  } else {
    /* build_design_matrix velocity.cpp:9-17; solve_velocity velocity.hpp:46-73 */
    double g00 = 0.0, g01 = 0.0, g11 = 0.0, b0 = 0.0, b1 = 0.0, dsum = 0.0;
    double c0 = 0.0, s0 = 0.0;
    int first = 1;
    for (int64_t k = 0; k < n; ++k) {
      if (!mask[k]) continue;
      const double c = cos(az[k]), s = sin(az[k]);
      if (first) {
        c0 = c;
        s0 = s;
        first = 0;
      }
      g00 += c * c;
      g01 += c * s;
      g11 += s * s;
      b0 += c * dop[k];
      b1 += s * dop[k];
      dsum += dop[k];
    }
    const double det = g00 * g11 - g01 * g01;
    const double half_trace = (g00 + g11) / 2.0;
    if (det >= K_RANK_EPSILON * half_trace * half_trace) {
      est->v_x = (g11 * b0 - g01 * b1) / det;
      est->v_y = (g00 * b1 - g01 * b0) / det;
      est->condition_ok = 1;
    } else { /* min_norm_fallback velocity.hpp:79-105 */
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
      const double nrm = sqrt(u0 * u0 + u1 * u1);
      if (nrm > 0.0) {
        u0 /= nrm;
        u1 /= nrm;
      }
      if (u0 * c0 + u1 * s0 < 0.0) {
        u0 = -u0;
        u1 = -u1;
      }
      const double mean = dsum / (double)n_in;
      est->v_x = mean * u0;
      est->v_y = mean * u1;
      est->condition_ok = 0;
    }
  }
  /* heading_angle velocity.cpp:19-24 */
  if (!(fabs(est->v_x) < K_ZERO_VELOCITY_EPSILON && fabs(est->v_y) < K_ZERO_VELOCITY_EPSILON)) {
    est->heading = to_half_open_angle(atan2(est->v_y, est->v_x));
    est->has_heading = 1;
  }
}

int rvk_or_estimate_all(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                        const double* az, const double* dop, const int32_t* ids,
                        const uint8_t* mask, rvk_estimate* out) {
  for (int32_t c = 0; c < n_clusters; ++c) {
    const int64_t b = offsets[c];
    estimate_cluster(frame_id, ids ? ids[c] : c, offsets[c + 1] - b, az + b, dop + b, mask + b,
                     out + c);
  }
  return RVK_OK;
}

int rvk_or_ransac_estimate_range(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                                 const double* az, const double* dop, const int32_t* ids,
                                 const rvk_ransac_params* p, int32_t c_begin, int32_t c_end,
                                 int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                                 rvk_estimate* out) {
  const int st = validate(n_clusters, offsets, p, "run_ransac");
  if (st != RVK_OK) return st;
  for (int32_t c = c_begin; c < c_end; ++c) {
    const int64_t b = offsets[c], n = offsets[c + 1] - b;
    double* xy = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    ransac_one(n, az + b, dop + b, p, c, inlier_count + c, winning_trial + c, mask + b, xy);
    free(xy);
    estimate_cluster(frame_id, ids ? ids[c] : c, n, az + b, dop + b, mask + b, out + c);
  }
  return RVK_OK;
}

/* ---- DBSCAN + extract_clusters (src/clustering.cpp) ---------------------
 * Restated from the reference, O(n^2) neighbour tests like it. Any
 * breadth-first order visits the same component, so the queue-based
 * labelling here equals the reference's (:62-89) exactly. */

/* squared_distance, clustering.cpp:11-20 (compiled -ffp-contract=off) */
static double sq_dist(const double* x, const double* y, const double* z, int features, int64_t a,
                      int64_t b) {
  const double dx = x[a] - x[b];
  const double dy = y[a] - y[b];
  double d2 = dx * dx + dy * dy;
  if (features) {
    const double dz = z[a] - z[b];
    d2 += dz * dz;
  }
  return d2;
}

int rvk_or_dbscan(int64_t n, const double* x, const double* y, const double* z, double eps,
                  int32_t min_pts, int32_t features, int32_t* labels) {
  if (!(eps > 0.0)) { /* clustering.cpp:25-27 */
    snprintf(g_err, sizeof g_err, "dbscan: eps must be positive");
    return 1;
  }
  if (min_pts < 1) { /* :28-30 */
    snprintf(g_err, sizeof g_err, "dbscan: min_pts must be at least 1");
    return 1;
  }
  for (int64_t i = 0; i < n; ++i) labels[i] = -1;
  if (n == 0) return 0;
  const double eps2 = eps * eps; /* :37 */
  /* |N_eps(p)| including p itself (:39-60) */
  char* core = (char*)calloc((size_t)n, 1);
  for (int64_t i = 0; i < n; ++i) {
    int64_t cnt = 0;
    for (int64_t j = 0; j < n; ++j) cnt += sq_dist(x, y, z, features, i, j) <= eps2;
    core[i] = cnt >= min_pts;
  }
  /* core-core components, ids in order of the smallest core index (:62-89) */
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int32_t next_id = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!core[i] || labels[i] != -1) continue;
    const int32_t id = next_id++;
    int64_t head = 0, tail = 0;
    labels[i] = id;
    queue[tail++] = i;
    while (head < tail) {
      const int64_t p = queue[head++];
      for (int64_t q = 0; q < n; ++q)
        if (core[q] && labels[q] == -1 && sq_dist(x, y, z, features, p, q) <= eps2) {
          labels[q] = id;
          queue[tail++] = q;
        }
    }
  }
  /* border points: nearest core neighbour, ties to the lowest index (:91-113) */
  for (int64_t i = 0; i < n; ++i) {
    if (core[i]) continue;
    int64_t best = -1;
    double best_d2 = 0.0;
    for (int64_t q = 0; q < n; ++q) {
      if (q == i || !core[q]) continue;
      const double d2 = sq_dist(x, y, z, features, i, q);
      if (d2 > eps2) continue;
      if (best == -1 || d2 < best_d2 || (d2 == best_d2 && q < best)) {
        best = q;
        best_d2 = d2;
      }
    }
    if (best != -1) labels[i] = labels[best];
  }
  free(queue);
  free(core);
  return 0;
}

/* extract_clusters (src/clustering.cpp:116-155) */
int rvk_or_extract_clusters(int64_t n, int32_t* labels, int32_t min_cluster_size,
                            int32_t* n_clusters, int64_t* offsets, int32_t* point_indices) {
  if (min_cluster_size < 1) {
    snprintf(g_err, sizeof g_err, "extract_clusters: min_cluster_size must be at least 1");
    return 1;
  }
  int32_t max_label = -1;
  for (int64_t i = 0; i < n; ++i) max_label = labels[i] > max_label ? labels[i] : max_label;
  const int64_t k = (int64_t)max_label + 1;
  int64_t* size = (int64_t*)calloc((size_t)(k > 0 ? k : 1), sizeof(int64_t));
  int32_t* remap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
  for (int64_t i = 0; i < n; ++i)
    if (labels[i] >= 0) ++size[labels[i]];
  int32_t m = 0;
  offsets[0] = 0;
  for (int64_t l = 0; l < k; ++l) {
    remap[l] = -1;
    if (size[l] < min_cluster_size) continue;
    remap[l] = m;
    offsets[m + 1] = offsets[m] + size[l];
    ++m;
  }
  int64_t* fill = (int64_t*)calloc((size_t)(m > 0 ? m : 1), sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) { /* members in ascending point order */
    if (labels[i] < 0) continue;
    const int32_t c = remap[labels[i]];
    labels[i] = c;
    if (c >= 0) point_indices[offsets[c] + fill[c]++] = (int32_t)i;
  }
  *n_clusters = m;
  free(fill);
  free(remap);
  free(size);
  return 0;
}

/* combine_masks (src/ransac.cpp:217-242): a point's position within its
 * label counts the earlier points of that label (:227-239); the first mask
 * with a given cluster_id wins (unordered_map::emplace, :223-226). */
int rvk_or_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks,
                         const int32_t* mask_ids, const int64_t* mask_offsets,
                         const uint8_t* masks, uint8_t* result) {
  for (int64_t i = 0; i < n; ++i) result[i] = 0;
  if (n_masks == 0) return 0;
  int32_t max_label = -1;
  for (int64_t i = 0; i < n; ++i) max_label = labels[i] > max_label ? labels[i] : max_label;
  if (max_label < 0) return 0;
  int64_t* seen = (int64_t*)calloc((size_t)max_label + 1, sizeof(int64_t));
  int32_t* by_id = (int32_t*)malloc(sizeof(int32_t) * ((size_t)max_label + 1));
  for (int32_t l = 0; l <= max_label; ++l) by_id[l] = -1;
  for (int32_t k = 0; k < n_masks; ++k)
    if (mask_ids[k] >= 0 && mask_ids[k] <= max_label && by_id[mask_ids[k]] < 0)
      by_id[mask_ids[k]] = k;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t l = labels[i];
    if (l < 0) continue;
    const int64_t pos = seen[l]++;
    const int32_t k = by_id[l];
    if (k >= 0 && pos < mask_offsets[k + 1] - mask_offsets[k])
      result[i] = masks[mask_offsets[k] + pos] ? 1 : 0;
  }
  free(by_id);
  free(seen);
  return 0;
}
