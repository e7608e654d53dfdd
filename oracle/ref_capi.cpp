// TEST INFRASTRUCTURE ONLY -- never on the product path.
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled from
// /root/reference/proj/src/{ransac,velocity,baseline,scene,bench,clustering}.cpp
// by oracle/Makefile into oracle/_ref/librvk_ref.so (with the Eigen stand-in
// compat/eigen_shim). The entry points mirror include/rvk_gpu.h with an
// rvk_ref_ prefix so the tests and bench.py --impl reference drive both
// implementations with the same marshalling.
//
// Every function here only converts CSR arrays <-> the reference's Eigen /
// std::vector types and calls the reference:
//   rvk::run_ransac         src/ransac.cpp:138-199
//   rvk::sequential_ransac  src/baseline.cpp:11-51
//   rvk::estimate_all       src/velocity.cpp:92-121
//   rvk::sequential_lsq     src/baseline.cpp:53-79
//   rvk::draw_seed_pair / normalize_cluster / mad_threshold /
//   count_trial_inliers     src/ransac.cpp:69-127
//   rvk::generate_frame     src/scene.cpp:105-189 (workload synthesis)
#include <rvk/baseline.hpp>
#include <rvk/clustering.hpp>
#include <rvk/frame_io.hpp>
#include <rvk/ransac.hpp>
#include <rvk/rng.hpp>
#include <rvk/scene.hpp>
#include <rvk/velocity.hpp>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/rvk_gpu.h"

namespace {

thread_local std::string g_error;
thread_local int g_error_cluster = -1;

std::vector<Eigen::ArrayX2d> to_clusters(int32_t n, const int64_t* off, const double* az,
                                         const double* dop) {
  std::vector<Eigen::ArrayX2d> out(static_cast<std::size_t>(n));
  for (int32_t c = 0; c < n; ++c) {
    const int64_t b = off[c], e = off[c + 1];
    Eigen::ArrayX2d pts(e - b, 2);
    for (int64_t k = b; k < e; ++k) {
      pts(k - b, 0) = az[k];
      pts(k - b, 1) = dop[k];
    }
    out[static_cast<std::size_t>(c)] = std::move(pts);
  }
  return out;
}

rvk::RansacParams to_params(const rvk_ransac_params* p) {
  rvk::RansacParams r;
  r.max_trials = p->max_trials;
  r.threshold_scale = p->threshold_scale;
  r.rng_seed = p->rng_seed;
  return r;
}

void from_masks(const std::vector<rvk::InlierMask>& masks, const int64_t* off, int32_t* count,
                int32_t* trial, uint8_t* mask) {
  for (std::size_t c = 0; c < masks.size(); ++c) {
    if (count) count[c] = masks[c].inlier_count;
    if (trial) trial[c] = masks[c].winning_trial;
    if (mask)
      for (Eigen::Index k = 0; k < masks[c].mask.size(); ++k)
        mask[off[c] + k] = masks[c].mask(k) ? 1 : 0;
  }
}

// A frame whose points are the CSR arrays in order, one Cluster per range.
void to_frame(int64_t frame_id, int32_t n, const int64_t* off, const double* az, const double* dop,
              const int32_t* ids, rvk::Frame& frame, std::vector<rvk::Cluster>& clusters) {
  frame.frame_id = frame_id;
  frame.points.resize(static_cast<std::size_t>(off[n]));
  for (int64_t k = 0; k < off[n]; ++k) {
    frame.points[static_cast<std::size_t>(k)].azimuth = az[k];
    frame.points[static_cast<std::size_t>(k)].doppler = dop[k];
  }
  clusters.resize(static_cast<std::size_t>(n));
  for (int32_t c = 0; c < n; ++c) {
    clusters[static_cast<std::size_t>(c)].cluster_id = ids ? ids[c] : c;
    auto& idx = clusters[static_cast<std::size_t>(c)].point_indices;
    idx.clear();
    for (int64_t k = off[c]; k < off[c + 1]; ++k) idx.push_back(static_cast<int>(k));
  }
}

std::vector<rvk::InlierMask> to_masks(int32_t n, const int64_t* off, const uint8_t* mask) {
  std::vector<rvk::InlierMask> masks(static_cast<std::size_t>(n));
  for (int32_t c = 0; c < n; ++c) {
    auto& m = masks[static_cast<std::size_t>(c)];
    m.cluster_id = c;
    m.mask = rvk::BoolArray::Constant(off[c + 1] - off[c], false);
    int cnt = 0;
    for (int64_t k = off[c]; k < off[c + 1]; ++k) {
      m.mask(k - off[c]) = mask[k] != 0;
      cnt += mask[k] != 0;
    }
    m.inlier_count = cnt;
    m.winning_trial = -1;
  }
  return masks;
}

void from_estimates(const std::vector<rvk::VelocityEstimate>& est, rvk_estimate* out) {
  for (std::size_t c = 0; c < est.size(); ++c) {
    out[c].frame_id = est[c].frame_id;
    out[c].cluster_id = est[c].cluster_id;
    out[c].inlier_count = est[c].inlier_count;
    out[c].v_x = est[c].v_x;
    out[c].v_y = est[c].v_y;
    out[c].has_heading = est[c].heading.has_value() ? 1 : 0;
    out[c].heading = est[c].heading.value_or(0.0);
    out[c].condition_ok = est[c].condition_ok ? 1 : 0;
  }
}

template <class F>
int guarded(F&& f) {
  g_error.clear();
  g_error_cluster = -1;
  try {
    f();
    return RVK_OK;
  } catch (const rvk::ClusterTooSmall& e) {
    g_error = e.what();
    // "run_ransac: cluster <c> has ..." (src/ransac.cpp:151)
    const std::string s = e.what();
    const auto p = s.find("cluster ");
    if (p != std::string::npos) g_error_cluster = std::atoi(s.c_str() + p + 8);
    return RVK_ECLUSTER_TOO_SMALL;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return RVK_EINVAL;
  } catch (const std::exception& e) {
    g_error = e.what();
    return RVK_EINVAL;
  }
}

}  // namespace

extern "C" {

const char* rvk_ref_last_error(void) { return g_error.c_str(); }
int32_t rvk_ref_last_error_cluster(void) { return g_error_cluster; }

int rvk_ref_run_ransac(int32_t n, const int64_t* off, const double* az, const double* dop,
                       const rvk_ransac_params* p, int32_t workers, int32_t* count, int32_t* trial,
                       uint8_t* mask) {
  return guarded([&] {
    const auto masks = rvk::run_ransac(to_clusters(n, off, az, dop), to_params(p), workers);
    from_masks(masks, off, count, trial, mask);
  });
}

int rvk_ref_sequential_ransac(int32_t n, const int64_t* off, const double* az, const double* dop,
                              const rvk_ransac_params* p, int32_t* count, int32_t* trial,
                              uint8_t* mask) {
  return guarded([&] {
    const auto masks = rvk::sequential_ransac(to_clusters(n, off, az, dop), to_params(p));
    from_masks(masks, off, count, trial, mask);
  });
}

int rvk_ref_estimate_all(int64_t frame_id, int32_t n, const int64_t* off, const double* az,
                         const double* dop, const int32_t* ids, const uint8_t* mask,
                         int32_t workers, rvk_estimate* out) {
  return guarded([&] {
    rvk::Frame frame;
    std::vector<rvk::Cluster> clusters;
    to_frame(frame_id, n, off, az, dop, ids, frame, clusters);
    const auto est = rvk::estimate_all(frame, clusters, to_masks(n, off, mask), workers);
    from_estimates(est, out);
  });
}

int rvk_ref_sequential_lsq(int64_t frame_id, int32_t n, const int64_t* off, const double* az,
                           const double* dop, const int32_t* ids, const uint8_t* mask,
                           rvk_estimate* out) {
  return guarded([&] {
    rvk::Frame frame;
    std::vector<rvk::Cluster> clusters;
    to_frame(frame_id, n, off, az, dop, ids, frame, clusters);
    const auto est = rvk::sequential_lsq(frame, clusters, to_masks(n, off, mask));
    from_estimates(est, out);
  });
}

// The reference pipeline (tools/rvk_main.cpp:134-144): gather is implicit in
// the CSR layout, then run_ransac + estimate_all with `workers` threads.
int rvk_ref_ransac_estimate(int64_t frame_id, int32_t n, const int64_t* off, const double* az,
                            const double* dop, const int32_t* ids, const rvk_ransac_params* p,
                            int32_t workers, int32_t* count, int32_t* trial, uint8_t* mask,
                            rvk_estimate* out) {
  return guarded([&] {
    rvk::Frame frame;
    std::vector<rvk::Cluster> clusters;
    to_frame(frame_id, n, off, az, dop, ids, frame, clusters);
    const auto pts = rvk::gather_cluster_points(frame, clusters);
    const auto masks = rvk::run_ransac(pts, to_params(p), workers);
    const auto est = rvk::estimate_all(frame, clusters, masks, workers);
    from_masks(masks, off, count, trial, mask);
    if (out) from_estimates(est, out);
  });
}

int rvk_ref_trial_counts(int32_t n, const int64_t* off, const double* az, const double* dop,
                         const rvk_ransac_params* p, int32_t* counts) {
  return guarded([&] {
    const auto clusters = to_clusters(n, off, az, dop);
    for (int32_t c = 0; c < n; ++c) {
      const auto nc = rvk::normalize_cluster(clusters[static_cast<std::size_t>(c)]);
      const double thr = rvk::mad_threshold(nc.pts.col(1), p->threshold_scale);
      const int np = static_cast<int>(nc.pts.rows());
      for (int t = 0; t < p->max_trials; ++t) {
        const auto [a, b] = rvk::draw_seed_pair(p->rng_seed, c, t, np);
        counts[static_cast<int64_t>(c) * p->max_trials + t] = rvk::count_trial_inliers(nc, a, b, thr);
      }
    }
  });
}

int rvk_ref_seed_pair(uint64_t seed, int32_t cluster, int32_t trial, int32_t n, int32_t* i,
                      int32_t* j) {
  return guarded([&] {
    const auto [a, b] = rvk::draw_seed_pair(seed, cluster, trial, n);
    *i = a;
    *j = b;
  });
}

// n draws of KeyedRng(seed, hi, lo).next_unit() (workload layout draws).
void rvk_ref_rng_units(uint64_t seed, uint64_t hi, uint64_t lo, int64_t n, double* out) {
  rvk::KeyedRng rng(seed, hi, lo);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next_unit();
}

uint64_t rvk_ref_rng_u64(uint64_t seed, uint64_t hi, uint64_t lo, int32_t k) {
  rvk::KeyedRng rng(seed, hi, lo);
  uint64_t v = 0;
  for (int32_t i = 0; i <= k; ++i) v = rng.next_u64();
  return v;
}

int rvk_ref_cluster_thresholds(int32_t n, const int64_t* off, const double* az, const double* dop,
                               double scale, double* norm, double* thr, double* normalized) {
  return guarded([&] {
    const auto clusters = to_clusters(n, off, az, dop);
    for (int32_t c = 0; c < n; ++c) {
      const auto nc = rvk::normalize_cluster(clusters[static_cast<std::size_t>(c)]);
      norm[4 * c + 0] = nc.offset(0);
      norm[4 * c + 1] = nc.offset(1);
      norm[4 * c + 2] = nc.scale(0);
      norm[4 * c + 3] = nc.scale(1);
      thr[c] = rvk::mad_threshold(nc.pts.col(1), scale);
      if (normalized)
        for (int64_t k = off[c]; k < off[c + 1]; ++k) {
          normalized[2 * k + 0] = nc.pts(k - off[c], 0);
          normalized[2 * k + 1] = nc.pts(k - off[c], 1);
        }
    }
  });
}

// One synthetic object per row of `objects` (10 doubles each):
// center_x, center_y, extent_x, extent_y, v_x, v_y, n_points,
// outlier_fraction, doppler_noise_sigma, (unused). Outlier offset range is
// `offset_lo..offset_hi`. Writes P points (x, y, doppler, azimuth) and the
// per-object first_point; returns the status. scene.cpp:105-189.
int rvk_ref_generate_frame(uint64_t seed, int32_t n_objects, const double* objects,
                           double offset_lo, double offset_hi, double* x, double* y,
                           double* doppler, double* azimuth, int32_t* outlier_flag) {
  return guarded([&] {
    rvk::SceneSpec spec;
    spec.rng_seed = seed;
    for (int32_t i = 0; i < n_objects; ++i) {
      const double* o = objects + 10 * i;
      rvk::ObjectSpec obj;
      obj.center = Eigen::Vector2d(o[0], o[1]);
      obj.extent = Eigen::Vector2d(o[2], o[3]);
      obj.v_x = o[4];
      obj.v_y = o[5];
      obj.n_points = static_cast<int>(o[6]);
      obj.outlier_fraction = o[7];
      obj.doppler_noise_sigma = o[8];
      obj.outlier_offset_range = Eigen::Vector2d(offset_lo, offset_hi);
      spec.objects.push_back(obj);
    }
    const auto scene = rvk::generate_frame(spec);
    for (std::size_t k = 0; k < scene.frame.points.size(); ++k) {
      x[k] = scene.frame.points[k].x;
      y[k] = scene.frame.points[k].y;
      doppler[k] = scene.frame.points[k].doppler;
      azimuth[k] = scene.frame.points[k].azimuth;
      if (outlier_flag) outlier_flag[k] = 0;
    }
    if (outlier_flag)
      for (const auto& t : scene.truth)
        for (int idx : t.outlier_indices) outlier_flag[idx] = 1;
  });
}

// rvk::dbscan (src/clustering.cpp:24-114) on SoA points; features 0 = XY, 1 = XYZ.
int rvk_ref_dbscan(int64_t n, const double* x, const double* y, const double* z, double eps,
                   int32_t min_pts, int32_t features, int32_t* labels) {
  return guarded([&] {
    rvk::Frame frame;
    frame.points.resize(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      frame.points[static_cast<std::size_t>(i)].x = x[i];
      frame.points[static_cast<std::size_t>(i)].y = y[i];
      frame.points[static_cast<std::size_t>(i)].z = z ? z[i] : 0.0;
    }
    rvk::ClusteringParams cp;
    cp.eps = eps;
    cp.min_pts = min_pts;
    cp.features = features ? rvk::ClusterFeatures::XYZ : rvk::ClusterFeatures::XY;
    rvk::dbscan(frame, cp);
    for (int64_t i = 0; i < n; ++i) labels[i] = frame.labels[static_cast<std::size_t>(i)];
  });
}

// rvk::extract_clusters (src/clustering.cpp:116-155): labels in/out, CSR out.
int rvk_ref_extract_clusters(int64_t n, int32_t* labels, int32_t min_cluster_size,
                             int32_t* n_clusters, int64_t* offsets, int32_t* point_indices) {
  return guarded([&] {
    rvk::Frame frame;
    frame.points.resize(static_cast<std::size_t>(n));
    frame.labels.assign(labels, labels + n);
    const auto clusters = rvk::extract_clusters(frame, min_cluster_size);
    *n_clusters = static_cast<int32_t>(clusters.size());
    offsets[0] = 0;
    int64_t k = 0;
    for (std::size_t c = 0; c < clusters.size(); ++c) {
      for (int idx : clusters[c].point_indices) point_indices[k++] = idx;
      offsets[c + 1] = k;
    }
    for (int64_t i = 0; i < n; ++i) labels[i] = frame.labels[static_cast<std::size_t>(i)];
  });
}

// rvk::combine_masks (src/ransac.cpp:217-242): frame labels + CSR masks.
int rvk_ref_combine_masks(int64_t n, const int32_t* labels, int32_t n_masks,
                          const int32_t* mask_ids, const int64_t* mask_offsets,
                          const uint8_t* masks, uint8_t* result) {
  return guarded([&] {
    rvk::Frame frame;
    frame.points.resize(static_cast<std::size_t>(n));
    frame.labels.assign(labels, labels + n);
    std::vector<rvk::InlierMask> ms(static_cast<std::size_t>(n_masks));
    for (int32_t k = 0; k < n_masks; ++k) {
      auto& m = ms[static_cast<std::size_t>(k)];
      m.cluster_id = mask_ids[k];
      const int64_t len = mask_offsets[k + 1] - mask_offsets[k];
      m.mask = rvk::BoolArray::Constant(len, false);
      for (int64_t q = 0; q < len; ++q) m.mask(q) = masks[mask_offsets[k] + q] != 0;
    }
    const rvk::BoolArray r = rvk::combine_masks(frame, ms);
    for (int64_t i = 0; i < n; ++i) result[i] = r(i) ? 1 : 0;
  });
}

// The body of run_estimate (tools/rvk_main.cpp:104-158) without CLI11:
// read_frames -> per frame dbscan, extract_clusters, gather, run_ransac +
// estimate_all (mode 0 "parallel") or all_true_masks + estimate_all (mode 2
// "lsq-only") -> write_estimates. Per-frame errors are skipped like the CLI.
int rvk_ref_run_estimate_csv(const char* frames_path, const char* out_path, int32_t mode,
                             double eps, int32_t min_pts, int32_t max_trials,
                             double threshold_scale, uint64_t seed) {
  return guarded([&] {
    rvk::ClusteringParams cp;
    cp.eps = eps;
    cp.min_pts = min_pts;
    rvk::RansacParams rp;
    rp.max_trials = max_trials;
    rp.threshold_scale = threshold_scale;
    rp.rng_seed = seed;
    std::vector<rvk::Frame> frames = rvk::read_frames(frames_path);
    std::vector<rvk::VelocityEstimate> all;
    for (rvk::Frame& frame : frames) {
      try {
        rvk::dbscan(frame, cp);
        const auto clusters = rvk::extract_clusters(frame);
        if (clusters.empty()) continue;
        const auto pts = rvk::gather_cluster_points(frame, clusters);
        std::vector<rvk::VelocityEstimate> est;
        if (mode == 0) {
          const auto masks = rvk::run_ransac(pts, rp, 0);
          est = rvk::estimate_all(frame, clusters, masks, 0);
        } else {
          est = rvk::estimate_all(frame, clusters, rvk::all_true_masks(clusters), 0);
        }
        all.insert(all.end(), est.begin(), est.end());
      } catch (const std::exception&) {
      }
    }
    rvk::write_estimates(all, out_path);
  });
}

// rvk::write_frames (src/frame_io.cpp:141-156) of one frame of SoA points.
int rvk_ref_write_frames(int32_t n_frames, const int64_t* frame_ids, const int64_t* offsets,
                         const double* x, const double* y, const double* z, const double* dop,
                         const double* az, const char* path) {
  return guarded([&] {
    std::vector<rvk::Frame> frames(static_cast<std::size_t>(n_frames));
    for (int32_t f = 0; f < n_frames; ++f) {
      frames[static_cast<std::size_t>(f)].frame_id = frame_ids[f];
      for (int64_t i = offsets[f]; i < offsets[f + 1]; ++i) {
        rvk::RadarPoint p;
        p.x = x[i];
        p.y = y[i];
        p.z = z[i];
        p.doppler = dop[i];
        p.azimuth = az[i];
        frames[static_cast<std::size_t>(f)].points.push_back(p);
      }
    }
    rvk::write_frames(frames, path);
  });
}

}  // extern "C"
