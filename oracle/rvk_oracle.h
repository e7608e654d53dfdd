/*
 * TEST INFRASTRUCTURE ONLY -- the CPU checker. Never linked into, called by,
 * or shipped with the product path (paper_2012_12618_b200/); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 *
 * Plain-C restatement of the reference's per-cluster RANSAC + LSQ path
 * (/root/reference/proj, C++20/Eigen), function by function; each definition
 * in rvk_oracle.c cites the reference file:line it follows. Pinned against
 * the reference itself: tests/golden/ holds vectors produced by the
 * unmodified reference (oracle/_ref/librvk_ref.so, script
 * tests/golden/make_golden.py) and tests/test_oracle.py checks this oracle
 * against every one of them, bit-exact.
 *
 * Same CSR conventions and entry-point shapes as include/rvk_gpu.h.
 */
#ifndef RVK_ORACLE_H_
#define RVK_ORACLE_H_

#include <stdint.h>

#include "../include/rvk_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rvk_or_rng {
  uint64_t state;
} rvk_or_rng;

void rvk_or_rng_init(rvk_or_rng* r, uint64_t seed, uint64_t hi, uint64_t lo);
uint64_t rvk_or_rng_next_u64(rvk_or_rng* r);
uint32_t rvk_or_rng_next_below(rvk_or_rng* r, uint32_t n);
double rvk_or_rng_next_unit(rvk_or_rng* r);
double rvk_or_rng_next_range(rvk_or_rng* r, double lo, double hi);
double rvk_or_rng_next_gaussian(rvk_or_rng* r);
uint64_t rvk_or_rng_u64(uint64_t seed, uint64_t hi, uint64_t lo, int32_t k);

int rvk_or_seed_pair(uint64_t seed, int32_t cluster, int32_t trial, int32_t n, int32_t* i,
                     int32_t* j);

/* normalize_cluster + mad_threshold for one cluster; xy[2*k+{0,1}] receives
 * the normalized (azimuth, doppler) of point k. Returns the threshold. */
double rvk_or_prepare_cluster(int64_t n, const double* az, const double* dop, double scale,
                              double* xy, double* norm4);
/* run_trial (count only when mask == NULL). */
int32_t rvk_or_run_trial(int64_t n, const double* xy, int32_t a, int32_t b, double thr,
                         uint8_t* mask);

const char* rvk_or_last_error(void);

int rvk_or_sequential_ransac(int32_t n_clusters, const int64_t* offsets, const double* az,
                             const double* dop, const rvk_ransac_params* params,
                             const int32_t* rng_cluster_index, int32_t* inlier_count,
                             int32_t* winning_trial, uint8_t* mask);
int rvk_or_trial_counts(int32_t n_clusters, const int64_t* offsets, const double* az,
                        const double* dop, const rvk_ransac_params* params,
                        const int32_t* rng_cluster_index, int32_t* counts);
int rvk_or_cluster_thresholds(int32_t n_clusters, const int64_t* offsets, const double* az,
                              const double* dop, double scale, double* norm, double* thr,
                              double* normalized);
int rvk_or_estimate_all(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                        const double* az, const double* dop, const int32_t* cluster_ids,
                        const uint8_t* mask, rvk_estimate* out);
/* Sequential RANSAC + LSQ over clusters [c_begin, c_end) only (bounded
 * CPU-baseline samples); outputs are indexed like the full call. */
int rvk_or_ransac_estimate_range(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                                 const double* az, const double* dop, const int32_t* cluster_ids,
                                 const rvk_ransac_params* params, int32_t c_begin, int32_t c_end,
                                 int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                                 rvk_estimate* out);

/* DBSCAN + extract_clusters (src/clustering.cpp:24-155), O(n^2) like the
 * reference; features 0 = XY, 1 = XYZ (z may be NULL for XY). */
int rvk_or_dbscan(int64_t n, const double* x, const double* y, const double* z, double eps,
                  int32_t min_pts, int32_t features, int32_t* labels);
int rvk_or_extract_clusters(int64_t n, int32_t* labels, int32_t min_cluster_size,
                            int32_t* n_clusters, int64_t* offsets, int32_t* point_indices);

/* combine_masks (src/ransac.cpp:217-242): frame labels + CSR masks. */
int rvk_or_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks,
                         const int32_t* mask_ids, const int64_t* mask_offsets,
                         const uint8_t* masks, uint8_t* result);

#ifdef __cplusplus
}
#endif

#endif /* RVK_ORACLE_H_ */
