// Host-side launchers for the sm_100a kernels in rvk_kernels.cu.
// All launchers are asynchronous on `stream` and count their launches in
// the calling thread's counter (rvk_kernel_launches()).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/rvk_gpu.h"

namespace rvk_gpu {

struct FrameDev {
  int32_t n_clusters = 0;
  int64_t n_points = 0;
  const int64_t* offsets = nullptr;   // [C+1]
  const double* azimuth = nullptr;    // [P]
  const double* doppler = nullptr;    // [P]
  const int32_t* keys = nullptr;      // [C] RNG cluster key or null (positional)
  const int32_t* cluster_ids = nullptr;  // [C] or null (positional)
  const int32_t* order = nullptr;     // [C] scoring order (largest first) or null
  int64_t frame_id = 0;
  int64_t max_cluster = -1;           // largest cluster size if the host knows it, else -1
};

// Scoring geometry for a given max_trials T (host and device agree on it).
// Hypotheses are processed in groups of 8 (one scoring lane each); a scoring
// unit is one warp's work: kUnitGroups groups (256 hypotheses) of one cluster
// against up to kScorePPT of its points.
constexpr int kScoreThreads = 256;
constexpr int kUnitGroups = 32;                   // groups of 8 hypotheses per unit (one per lane)
constexpr int kScorePPT = 512;                    // points per scoring unit (max)
constexpr int kTileBuckets = kScorePPT / 4 + 1;   // 0: full units; 1..128: by size, descending
static_assert(kScorePPT == 512, "ScoreGeom::ppt_shift default");

struct ScoreGeom {
  int T = 0;    // max_trials
  int Tg = 0;   // hypothesis groups of 8 per cluster
  int TS = 0;   // groups per unit (kUnitGroups)
  int nhb = 0;  // hypothesis blocks per cluster = ceil(Tg / TS)
  int ppt = kScorePPT;  // points per unit of this call: a power of two <= kScorePPT (score_ppt())
  int ppt_shift = 9;    // log2(ppt)
};

inline void set_ppt(ScoreGeom& g, int ppt) {
  g.ppt = ppt;
  g.ppt_shift = 0;
  while ((1 << g.ppt_shift) < ppt) ++g.ppt_shift;
}

inline __host__ __device__ ScoreGeom score_geom(int T) {
  ScoreGeom g;
  g.T = T;
  g.Tg = (T + 7) / 8;
  g.TS = kUnitGroups;
  g.nhb = (g.Tg + g.TS - 1) / g.TS;
  return g;
}

// Capacity of one tile bucket: bounds the total tile count of a frame.
inline int64_t tile_capacity(const ScoreGeom& g, int64_t n_points, int32_t n_clusters) {
  return static_cast<int64_t>(g.nhb) * (n_points / g.ppt + n_clusters) + 1;
}

// Points per scoring unit for a call: kScorePPT when the call has enough
// units to give every resident scoring warp two, else the largest of 256 /
// 128 / 64 / 32 that does (a single small frame: more, shorter units ->
// better balance, lower latency). RVK_SCORE_PPT overrides (tests).
int score_ppt(const ScoreGeom& g, int64_t n_points, int32_t n_clusters);

struct Scratch {
  double2* xy64 = nullptr;   // [P] normalized (x, y), FP64
  float2* xy32 = nullptr;    // [P + 2C + 10] normalized (x, y), FP32, each cluster
                             // starting at an even index, odd sizes padded (+8
                             // slack: the scoring loop reads ahead)
  double4* stat = nullptr;   // [C] (thr_lo, thr_hi, median, thr_exact|NaN)
  double* norm = nullptr;    // [4C] (offset_az, offset_dop, scale_az, scale_dop)
  int32_t* upper = nullptr;  // [C*Tg*8] fast-pass upper-bound counts
  float* hyp = nullptr;      // [C*Tg*32] per group of 8: A[8] B[8] C[8] K[8]
  int4* tiles = nullptr;     // [kTileBuckets * tile_cap] scoring tile descriptors
  int32_t* tile_count = nullptr;  // [kTileBuckets + 1] tiles per bucket + claim counter (zeroed per call)
  int32_t* big_list = nullptr;    // [C] clusters too large for the warp-per-cluster kernels
  int32_t* big_ctl = nullptr;     // [4] big_list count, CTA-prep claim counter, fused-kernel
                                  // claim counter (zeroed per call)
  int64_t tile_cap = 0;
  int ppt = kScorePPT;            // points per scoring unit of this call (score_ppt)
};

struct Outputs {
  int32_t* inlier_count = nullptr;   // [C]
  int32_t* winning_trial = nullptr;  // [C]
  uint8_t* mask = nullptr;           // [P] (required by the select kernel)
  rvk_estimate* est = nullptr;       // [C] or null (no refit)
};

void count_launch();

// normalize_cluster + median + mad_threshold per cluster.
void launch_prep(const FrameDev& f, double threshold_scale, const Scratch& s, cudaStream_t st);
// Exact (left-to-right) MAD threshold into stat[c].w (and .x = .y).
void launch_mad_exact(const FrameDev& f, double threshold_scale, const Scratch& s,
                      cudaStream_t st);
// normalize + median + MAD + hypothesis setup (seed pairs, FP64 lines, FP32
// coefficients) + scoring-tile registration, one CTA per cluster.
void launch_prep_hyps(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                      cudaStream_t st);
// Whether a call takes the fused warp-per-cluster kernel (launch_fused) for its
// clusters of <= 512 points; the CTA path (prep_hyps -> score -> select) then
// runs on the clusters the fused kernel lists.
bool fused_path(const FrameDev& f, const rvk_ransac_params& p);
// The whole path for every cluster of <= 512 points, one warp each: normalize,
// median/MAD, hypotheses, FP32 upper-bound scoring, exact select, mask, refit.
void launch_fused(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                  const Outputs& o, cudaStream_t st);
// Whether a call takes the fused prep + score warp kernel (launch_prep_score)
// for its clusters of <= 384 points; select_warp_kernel then selects.
bool prep_score_path(const FrameDev& f, const rvk_ransac_params& p);
void launch_prep_score(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                       cudaStream_t st);
// Upper-bound inlier counts for every (cluster, trial): FFMA2 scoring.
void launch_score(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                  cudaStream_t st);
// Exact argmax (verifying every candidate that could win), winner mask,
// optional LSQ refit + heading.
void launch_select(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                   const Outputs& o, cudaStream_t st);
// mask[P] (0/1 bytes) -> bits[ceil(P/8)], point k = bit (k & 7) of byte k >> 3.
void launch_pack_mask(const uint8_t* mask, int64_t n_points, uint8_t* bits, cudaStream_t st);
// estimate_all on caller masks.
void launch_refit(const FrameDev& f, const uint8_t* mask, rvk_estimate* est, cudaStream_t st);
// Exact count of every (cluster, trial).
void launch_exact_counts(const FrameDev& f, const rvk_ransac_params& p, const Scratch& s,
                         int32_t* counts, cudaStream_t st);
void launch_seed_pairs(const FrameDev& f, const rvk_ransac_params& p, int32_t* pairs,
                       cudaStream_t st);

// ---- clustering (rvk_dbscan.cu): dbscan + extract_clusters
struct DbscanLayout {
  int table_bits = 0;
  size_t o_keys = 0, o_idx = 0, o_skeys = 0, o_sidx = 0, o_sx = 0, o_sy = 0, o_sz = 0;
  size_t o_cstart = 0, o_cend = 0, o_core = 0, o_parent = 0, o_root = 0, o_rep = 0, o_rank = 0;
  size_t o_count = 0, o_keep = 0, o_kept = 0, o_start = 0, o_small = 0, o_cub = 0;
  size_t cub_bytes = 0, total = 0;
};
DbscanLayout dbscan_layout(int64_t n, bool xyz);
// rvk::dbscan on device arrays x, y (z or null for XY) -> labels[n].
void launch_dbscan(int64_t n, const double* x, const double* y, const double* z, double eps,
                   int min_pts, const DbscanLayout& L, char* ws, int32_t* labels, cudaStream_t st);
// rvk::extract_clusters on device labels (rewritten in place); labels < n_labels_max.
// offsets[m+1], point_indices[n] (kept members first, ascending per cluster), *d_n_clusters = m.
void launch_extract(int64_t n, int32_t* labels, int32_t n_labels_max, int min_size,
                    const DbscanLayout& L, char* ws, int64_t* offsets, int32_t* point_indices,
                    int32_t* d_n_clusters, cudaStream_t st);
// rvk::combine_masks: result[n] from frame labels and CSR masks (ids sorted
// ascending with the first mask index per id in mask_of).
void launch_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks,
                          const int32_t* ids_sorted, const int32_t* mask_of,
                          const int64_t* moff, const uint8_t* masks, const DbscanLayout& L,
                          char* ws, uint8_t* result, cudaStream_t st);
// Gathers azimuth/doppler of the clusters' members (gather_cluster_points).
void launch_gather(int64_t p, const int32_t* point_indices, const double* az, const double* dop,
                   double* gaz, double* gdop, cudaStream_t st);

}  // namespace rvk_gpu
