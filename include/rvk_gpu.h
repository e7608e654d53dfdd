/*
 * rvk_gpu.h -- C-ABI of the B200 (sm_100a) per-cluster velocity-profile
 * estimator: RANSAC inlier selection + least-squares (v_x, v_y) refit +
 * heading.
 *
 * This is the drop-in boundary. Each entry point replaces one call of the
 * reference C++ API (proj/include/rvk, citations are relative to
 * /root/reference/proj) with plain pointers and sizes:
 *
 *   rvk_run_ransac     <- rvk::run_ransac      include/rvk/ransac.hpp:128-129
 *                                               (impl src/ransac.cpp:138-199)
 *   rvk_estimate_all   <- rvk::estimate_all    include/rvk/velocity.hpp:123-125
 *                                               (impl src/velocity.cpp:92-121)
 *   rvk_ransac_estimate   run_ransac followed by estimate_all on the same
 *                         clusters (the pipeline of tools/rvk_main.cpp:134-144
 *                         and src/bench.cpp:132-143), masks never leave HBM.
 *   rvk_trial_counts   <- per-(cluster, trial) count_trial_inliers
 *                         (src/ransac.cpp:125-127) as scored inside run_ransac
 *                         (src/ransac.cpp:164-174); exact for every trial.
 *   rvk_seed_pairs     <- rvk::draw_seed_pair  src/ransac.cpp:111-123
 *   rvk_cluster_thresholds <- normalize_cluster + mad_threshold
 *                         (src/ransac.cpp:69-94, ransac.hpp:53-84)
 *   rvk_stream_*          the per-frame loop of run_estimate
 *                         (tools/rvk_main.cpp:125-149), pipelined
 *   rvk_dbscan         <- rvk::dbscan          src/clustering.cpp:24-114
 *   rvk_extract_clusters <- rvk::extract_clusters src/clustering.cpp:116-155
 *   rvk_combine_masks  <- rvk::combine_masks  src/ransac.cpp:217-242
 *   rvk_estimate_frame    one frame of run_estimate: dbscan -> extract_clusters
 *                         -> gather -> run_ransac -> estimate_all
 *                         (tools/rvk_main.cpp:128-141), all on the device
 *
 * The C++ layer paper_2012_12618_b200/csrc/rvk_dropin.cpp re-exports the
 * reference's own C++ signatures on top of these, so unchanged callers link
 * against it.
 *
 * Data layout (CSR, one "frame" per call):
 *   offsets[n_clusters + 1]  int64, offsets[0] == 0, ascending; cluster c owns
 *                            points [offsets[c], offsets[c+1]).
 *   azimuth[P], doppler[P]   float64, P = offsets[n_clusters]; the points of
 *                            each cluster in the order gather_cluster_points
 *                            produces (src/ransac.cpp:201-215): this is exactly
 *                            Eigen::ArrayX2d's column-major [az(n) | dop(n)]
 *                            split into two SoA arrays.
 *   mask[P]                  uint8 0/1, aligned with the points (InlierMask::mask).
 *
 * Host entry points take HOST pointers, copy to the device, run, and copy back
 * before returning (synchronous, like the reference). The *_device variants
 * take DEVICE pointers and a cudaStream_t (as void*) and are asynchronous.
 *
 * Errors: every entry point returns an rvk_status. The message is available
 * from rvk_last_error() (thread-local). Validation order and messages follow
 * the reference so the C++ layer can rethrow the same exception types:
 *   RVK_EINVAL              -> std::invalid_argument   (ransac.cpp:140-145,
 *                                                        velocity.cpp:95-97,231-233)
 *   RVK_ECLUSTER_TOO_SMALL  -> rvk::ClusterTooSmall     (ransac.cpp:150-154);
 *                              rvk_last_error_cluster() = offending cluster.
 *   RVK_ECUDA / RVK_ENOMEM  -> std::runtime_error (no CPU fallback exists).
 *
 * Threading: re-entrant; one lazily created device context per (process,
 * device) under a mutex; each calling thread gets its own stream and
 * workspace. `workers` is accepted for signature parity with the reference
 * and ignored: the device grid replaces the std::thread team
 * (include/rvk/parallel.hpp:23-54). Results are bit-identical for any
 * device, grid or batch composition (the reference's worker-count
 * invariance, ransac.hpp:124-125).
 */
#ifndef RVK_GPU_H_
#define RVK_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RVK_GPU_ABI_VERSION 1

typedef enum rvk_status {
  RVK_OK = 0,
  RVK_EINVAL = 1,
  RVK_ECLUSTER_TOO_SMALL = 2,
  RVK_ECUDA = 3,
  RVK_ENOMEM = 4
} rvk_status;

/* Mirrors rvk::RansacParams (include/rvk/ransac.hpp:19-23). */
typedef struct rvk_ransac_params {
  int32_t max_trials;      /* line hypotheses per cluster, >= 1 (default 256) */
  int32_t reserved;        /* must be 0 */
  double threshold_scale;  /* > 0 (default 1.0) */
  uint64_t rng_seed;       /* KeyedRng seed (default 0) */
} rvk_ransac_params;

/* Mirrors rvk::VelocityEstimate (include/rvk/types.hpp:57-65). */
typedef struct rvk_estimate {
  int64_t frame_id;
  int32_t cluster_id;
  int32_t inlier_count;
  double v_x;
  double v_y;
  double heading;        /* valid iff has_heading */
  int32_t has_heading;   /* std::optional<double>::has_value() */
  int32_t condition_ok;
} rvk_estimate;

/* Library / device info. */
int32_t rvk_abi_version(void);
const char* rvk_last_error(void);
int32_t rvk_last_error_cluster(void);
/* Number of device kernels this thread launched since the last reset. */
int64_t rvk_kernel_launches(void);
void rvk_reset_kernel_launches(void);

/* rvk::run_ransac (src/ransac.cpp:138-199).
 *   rng_cluster_index: optional [n_clusters] RNG key per cluster; NULL means
 *   the positional index c, as in the reference (ransac.cpp:169). Batched
 *   multi-frame calls pass the frame-local index.
 *   Outputs (caller-allocated): inlier_count[C], winning_trial[C], mask[P]. */
int rvk_run_ransac(int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                   const double* doppler, const rvk_ransac_params* params,
                   const int32_t* rng_cluster_index, int32_t workers, int32_t* inlier_count,
                   int32_t* winning_trial, uint8_t* mask);

/* rvk::estimate_all (src/velocity.cpp:92-121) over CSR-gathered clusters.
 *   cluster_ids[C] = Cluster::cluster_id (copied to the estimates). */
int rvk_estimate_all(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                     const double* azimuth, const double* doppler, const int32_t* cluster_ids,
                     const uint8_t* mask, int32_t workers, rvk_estimate* out);

/* run_ransac + estimate_all fused; any output pointer may be NULL. */
int rvk_ransac_estimate(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                        const double* azimuth, const double* doppler, const int32_t* cluster_ids,
                        const rvk_ransac_params* params, const int32_t* rng_cluster_index,
                        int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                        rvk_estimate* out);

/* rvk_ransac_estimate with the masks bit-packed (the
 * InlierMask payload of include/rvk/types.hpp:50-55 at 1 bit per point):
 * mask_bits[ceil(P/8)], point k of the CSR = bit (k & 7) of byte k >> 3
 * (numpy.packbits(mask, bitorder="little")). The D2H of the mask is P/8
 * bytes instead of P. Everything else as rvk_ransac_estimate. */
int rvk_ransac_estimate_packed(int64_t frame_id, int32_t n_clusters, const int64_t* offsets,
                               const double* azimuth, const double* doppler,
                               const int32_t* cluster_ids, const rvk_ransac_params* params,
                               const int32_t* rng_cluster_index, int32_t* inlier_count,
                               int32_t* winning_trial, uint8_t* mask_bits, rvk_estimate* out);

/* rvk_ransac_estimate with one frame's clusters split over several GPUs for
 * latency: contiguous cluster ranges of about equal points,
 * one host thread per range, each on devices[i] (a device may repeat); the RNG
 * keys and cluster ids stay frame-positional, so the outputs are byte-identical
 * to the single-device call. Validation and messages as rvk_ransac_estimate,
 * on the whole frame. */
int rvk_ransac_estimate_multi(int32_t n_devices, const int32_t* devices, int64_t frame_id,
                              int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                              const double* doppler, const int32_t* cluster_ids,
                              const rvk_ransac_params* params, const int32_t* rng_cluster_index,
                              int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                              rvk_estimate* out);

/* Device-pointer variant of rvk_ransac_estimate (all arrays in HBM, async on
 * `stream`, a cudaStream_t or NULL for the legacy default stream). The
 * caller must keep the inputs alive until the stream reaches this point.
 * Preconditions (the offsets live in HBM, so they are not checked on the
 * host): d_offsets[0] == 0, non-decreasing, d_offsets[n_clusters] ==
 * n_points. A cluster with fewer than 3 points -- which the host API rejects
 * with RVK_ECLUSTER_TOO_SMALL like the reference (src/ransac.cpp:147-156) --
 * is never read: its outputs are a sentinel, inlier_count = winning_trial =
 * -1, an all-zero mask and an estimate with v = 0, inlier_count 0,
 * condition_ok 0 and no heading; every other cluster's outputs are
 * unaffected. */
int rvk_ransac_estimate_device(int64_t frame_id, int32_t n_clusters, int64_t n_points,
                               const int64_t* d_offsets, const double* d_azimuth,
                               const double* d_doppler, const int32_t* d_cluster_ids,
                               const rvk_ransac_params* params, const int32_t* d_rng_cluster_index,
                               int32_t* d_inlier_count, int32_t* d_winning_trial, uint8_t* d_mask,
                               rvk_estimate* d_out, void* stream);

/* Exact per-(cluster, trial) inlier counts, counts[c * max_trials + t]
 * (the `counts` vector of src/ransac.cpp:163-174). */
int rvk_trial_counts(int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                     const double* doppler, const rvk_ransac_params* params,
                     const int32_t* rng_cluster_index, int32_t* counts);

/* Seed pairs drawn on the device: pairs[2*(c*max_trials+t)+{0,1}] = (i, j)
 * of draw_seed_pair(seed, key_c, t, n_c) (src/ransac.cpp:111-123). */
int rvk_seed_pairs(int32_t n_clusters, const int64_t* offsets, const rvk_ransac_params* params,
                   const int32_t* rng_cluster_index, int32_t* pairs);

/* Per-cluster normalization offsets/scales and the MAD corridor, computed on
 * the device exactly as normalize_cluster + mad_threshold: norm[4*c+{0..3}] =
 * (offset_az, offset_dop, scale_az, scale_dop), threshold[c]. */
int rvk_cluster_thresholds(int32_t n_clusters, const int64_t* offsets, const double* azimuth,
                           const double* doppler, double threshold_scale, double* norm,
                           double* threshold);

/* Pipelined frame stream: the per-frame loop of the reference's estimate
 * pipeline (tools/rvk_main.cpp:125-149 -- for each frame, run_ransac then
 * estimate_all) with up to `depth` frames in flight, so the H2D copy of
 * frame k+1 overlaps the kernels of frame k and the D2H of frame k-1.
 * Results are identical to rvk_ransac_estimate on the same frame.
 *
 *   rvk_stream_create   params are validated once (src/ransac.cpp:140-145);
 *                       depth in [1, 8] (0 = default 3).
 *   rvk_stream_submit   validates the frame like run_ransac
 *                       (src/ransac.cpp:147-156) and enqueues it; returns a
 *                       ticket. Pinned (cudaHostAlloc / cudaHostRegister)
 *                       input and output arrays are read / written by DMA
 *                       directly and must stay valid until the ticket is
 *                       waited for; pageable inputs are staged during the
 *                       call. Blocks only when all `depth` slots are busy
 *                       (it then completes the oldest frame).
 *   rvk_stream_wait     blocks until the ticket's outputs are in the caller's
 *                       arrays (idempotent; completed tickets return RVK_OK).
 *   rvk_stream_destroy  completes every in-flight frame and frees the stream.
 *
 * A stream belongs to the device that was current at creation and is used
 * by one host thread at a time. */
typedef struct rvk_frame_stream rvk_frame_stream;
int rvk_stream_create(const rvk_ransac_params* params, int32_t depth, rvk_frame_stream** out);
int rvk_stream_submit(rvk_frame_stream* s, int64_t frame_id, int32_t n_clusters,
                      const int64_t* offsets, const double* azimuth, const double* doppler,
                      const int32_t* cluster_ids, const int32_t* rng_cluster_index,
                      int32_t* inlier_count, int32_t* winning_trial, uint8_t* mask,
                      rvk_estimate* out, int64_t* ticket);
/* rvk_stream_submit with the mask delivered bit-packed (mask_bits[ceil(P/8)],
 * layout of rvk_ransac_estimate_packed). */
int rvk_stream_submit_packed(rvk_frame_stream* s, int64_t frame_id, int32_t n_clusters,
                             const int64_t* offsets, const double* azimuth,
                             const double* doppler, const int32_t* cluster_ids,
                             const int32_t* rng_cluster_index, int32_t* inlier_count,
                             int32_t* winning_trial, uint8_t* mask_bits, rvk_estimate* out,
                             int64_t* ticket);
int rvk_stream_wait(rvk_frame_stream* s, int64_t ticket);
int rvk_stream_destroy(rvk_frame_stream* s);

/* ---- Clustering: the stage upstream of the path (tools/rvk_main.cpp:128-129) ----
 * Mirrors rvk::ClusteringParams (include/rvk/clustering.hpp:13-17). */
typedef struct rvk_clustering_params {
  double eps;        /* neighbourhood radius, > 0 (default 2.0) */
  int32_t min_pts;   /* neighbours incl. the point itself for a core point, >= 1 (default 3) */
  int32_t features;  /* RVK_FEATURES_XY (default) or RVK_FEATURES_XYZ */
} rvk_clustering_params;
#define RVK_FEATURES_XY 0
#define RVK_FEATURES_XYZ 1

/* rvk::dbscan (src/clustering.cpp:24-114) on the device, bit-exact: x, y
 * (and z for XYZ; may be NULL for XY) of n points -> labels[n] (cluster ids
 * 0..k-1 in order of each cluster's smallest core index, or -1 = noise). */
int rvk_dbscan(int64_t n, const double* x, const double* y, const double* z,
               const rvk_clustering_params* params, int32_t* labels);

/* rvk::extract_clusters (src/clustering.cpp:116-155): labels[n] rewritten in
 * place (small clusters -> -1, survivors compacted in order); outputs the
 * clusters as CSR: *n_clusters = m, offsets[m + 1] (capacity n + 1),
 * point_indices[n] (members of cluster c at offsets[c] .. offsets[c+1], in
 * ascending point order; entries past offsets[m] are unspecified). */
int rvk_extract_clusters(int64_t n, int32_t* labels, int32_t min_cluster_size,
                         int32_t* n_clusters, int64_t* offsets, int32_t* point_indices);

/* One frame of run_estimate's loop (tools/rvk_main.cpp:128-141), all on the
 * device: dbscan -> extract_clusters -> gather_cluster_points -> run_ransac
 * -> estimate_all. Point arrays are SoA (z may be NULL for XY). Outputs are
 * caller-allocated for the worst case: labels[n], offsets[n + 1],
 * point_indices[n], mask[n] (CSR-aligned with point_indices), and per cluster
 * (capacity n / min_cluster_size + 1) inlier_count, winning_trial, out
 * (cluster_id = the compact cluster id, frame_id = frame_id). Errors as the
 * reference's calls in that order (dbscan, extract_clusters, run_ransac). */
int rvk_estimate_frame(int64_t frame_id, int64_t n, const double* x, const double* y,
                       const double* z, const double* doppler, const double* azimuth,
                       const rvk_clustering_params* cparams, int32_t min_cluster_size,
                       const rvk_ransac_params* rparams, int32_t* labels, int32_t* n_clusters,
                       int64_t* offsets, int32_t* point_indices, int32_t* inlier_count,
                       int32_t* winning_trial, uint8_t* mask, rvk_estimate* out);

/* rvk::combine_masks (src/ransac.cpp:217-242): the frame-level union of the
 * cluster masks. labels[n] = Frame::labels; masks are CSR: mask k has
 * cluster_id mask_ids[k] and bytes masks[mask_offsets[k] .. mask_offsets[k+1]].
 * result[n]: point i is set iff its label is >= 0, a mask with that
 * cluster_id exists (the first such mask if ids repeat) and that mask is set
 * at i's position among the points of its label in ascending frame order.
 * n_masks == 0 gives all zeros. */
int rvk_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks, const int32_t* mask_ids,
                      const int64_t* mask_offsets, const uint8_t* masks, uint8_t* result);

/* Stage timing for benchmarking/profiling. When enabled, CUDA events bracket
 * every pipeline stage launch on its stream (0 = prep + hypothesis setup +
 * tile plan, 1 = a fused warp-per-cluster kernel -- the whole path for a
 * single frame of small clusters, or prep + score for batches of them --,
 * 2 = score, 3 = select + refit); rvk_profile_read waits for them, returns the
 * accumulated device milliseconds and launch counts per stage, and clears the
 * record. */
void rvk_profile_enable(int32_t on);
int rvk_profile_read(double* ms, int64_t* launches, int32_t n_stages);

#ifdef __cplusplus
}
#endif

#endif /* RVK_GPU_H_ */
