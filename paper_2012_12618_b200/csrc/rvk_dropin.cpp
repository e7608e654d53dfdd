// C++ drop-in for the reference API: strong definitions of
//
//   std::vector<InlierMask> rvk::run_ransac(const std::vector<Eigen::ArrayX2d>&,
//                                           const RansacParams&, int workers)
//       -- include/rvk/ransac.hpp:128-129, replaces src/ransac.cpp:138-199
//   std::vector<VelocityEstimate> rvk::estimate_all(const Frame&,
//                                                   const std::vector<Cluster>&,
//                                                   const std::vector<InlierMask>&, int workers)
//       -- include/rvk/velocity.hpp:123-125, replaces src/velocity.cpp:92-121
//   BoolArray rvk::combine_masks(const Frame&, const std::vector<InlierMask>&)
//       -- include/rvk/ransac.hpp:140, replaces src/ransac.cpp:217-242
//   void rvk::dbscan(Frame&, const ClusteringParams&)
//       -- include/rvk/clustering.hpp:24, replaces src/clustering.cpp:24-114
//   std::vector<Cluster> rvk::extract_clusters(Frame&, int)
//       -- include/rvk/clustering.hpp:31, replaces src/clustering.cpp:116-155
//
// with the reference's exact signatures, compiled against the reference's
// public headers (proj/include/rvk) and Eigen. Both marshal into the CSR
// layout of include/rvk_gpu.h and call the sm_100a pipeline; no CPU
// arithmetic of the path remains here. Errors are rethrown with the
// reference's types and messages (std::invalid_argument,
// rvk::ClusterTooSmall). `workers` is accepted and ignored.
//
// Link-time substitution (oracle/Makefile `dropin`): make
// the reference's definitions of these symbols file-local in its ransac.o /
// velocity.o / clustering.o (objcopy --localize-symbol, one object at a time)
// and link this library; every other reference symbol (primitives,
// sequential baselines, gather) stays the reference's own.
#include <rvk/clustering.hpp>
#include <rvk/ransac.hpp>
#include <rvk/types.hpp>
#include <rvk/velocity.hpp>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "rvk_gpu.h"

namespace rvk {
namespace {

[[noreturn]] void rethrow(int status) {
  const std::string msg = rvk_last_error();
  if (status == RVK_EINVAL) throw std::invalid_argument(msg);
  if (status == RVK_ECLUSTER_TOO_SMALL) throw ClusterTooSmall(msg);
  throw std::runtime_error(msg);
}

}  // namespace

std::vector<InlierMask> run_ransac(const std::vector<Eigen::ArrayX2d>& clusters,
                                   const RansacParams& params, int /*workers*/) {
  const int32_t n = static_cast<int32_t>(clusters.size());
  std::vector<int64_t> offsets(static_cast<std::size_t>(n) + 1, 0);
  for (int32_t c = 0; c < n; ++c)
    offsets[c + 1] = offsets[c] + static_cast<int64_t>(clusters[static_cast<std::size_t>(c)].rows());
  const int64_t P = offsets[n];
  // ArrayX2d is column-major: col(0) = azimuth[n], col(1) = doppler[n].
  std::vector<double> az(static_cast<std::size_t>(P)), dop(static_cast<std::size_t>(P));
  for (int32_t c = 0; c < n; ++c) {
    const auto& m = clusters[static_cast<std::size_t>(c)];
    for (Eigen::Index k = 0; k < m.rows(); ++k) {
      az[static_cast<std::size_t>(offsets[c] + k)] = m(k, 0);
      dop[static_cast<std::size_t>(offsets[c] + k)] = m(k, 1);
    }
  }
  rvk_ransac_params p{params.max_trials, 0, params.threshold_scale, params.rng_seed};
  std::vector<int32_t> count(static_cast<std::size_t>(n)), trial(static_cast<std::size_t>(n));
  std::vector<uint8_t> mask(static_cast<std::size_t>(P));
  const int st = rvk_run_ransac(n, offsets.data(), az.data(), dop.data(), &p, nullptr, 0,
                                count.data(), trial.data(), mask.data());
  if (st != RVK_OK) rethrow(st);
  std::vector<InlierMask> out(static_cast<std::size_t>(n));
  for (int32_t c = 0; c < n; ++c) {
    InlierMask& im = out[static_cast<std::size_t>(c)];
    im.cluster_id = c;
    im.inlier_count = count[static_cast<std::size_t>(c)];
    im.winning_trial = trial[static_cast<std::size_t>(c)];
    im.mask = BoolArray::Constant(offsets[c + 1] - offsets[c], false);
    for (int64_t k = offsets[c]; k < offsets[c + 1]; ++k)
      im.mask(k - offsets[c]) = mask[static_cast<std::size_t>(k)] != 0;
  }
  return out;
}

std::vector<VelocityEstimate> estimate_all(const Frame& frame, const std::vector<Cluster>& clusters,
                                           const std::vector<InlierMask>& masks,
                                           int /*workers*/) {
  if (clusters.size() != masks.size())  // src/velocity.cpp:95-97
    throw std::invalid_argument("estimate_all: one mask per cluster required");
  const int32_t n = static_cast<int32_t>(clusters.size());
  std::vector<int64_t> offsets(static_cast<std::size_t>(n) + 1, 0);
  for (int32_t c = 0; c < n; ++c) {
    const auto& cl = clusters[static_cast<std::size_t>(c)];
    if (masks[static_cast<std::size_t>(c)].mask.size() !=
        static_cast<Eigen::Index>(cl.point_indices.size()))  // velocity.cpp:104-106
      throw std::invalid_argument("estimate_all: mask size does not match cluster size");
    offsets[c + 1] = offsets[c] + static_cast<int64_t>(cl.point_indices.size());
  }
  const int64_t P = offsets[n];
  std::vector<double> az(static_cast<std::size_t>(P)), dop(static_cast<std::size_t>(P));
  std::vector<uint8_t> mask(static_cast<std::size_t>(P));
  std::vector<int32_t> ids(static_cast<std::size_t>(n));
  for (int32_t c = 0; c < n; ++c) {
    const auto& cl = clusters[static_cast<std::size_t>(c)];
    ids[static_cast<std::size_t>(c)] = cl.cluster_id;
    for (std::size_t k = 0; k < cl.point_indices.size(); ++k) {
      const RadarPoint& pt = frame.points[static_cast<std::size_t>(cl.point_indices[k])];
      const std::size_t q = static_cast<std::size_t>(offsets[c]) + k;
      az[q] = pt.azimuth;
      dop[q] = pt.doppler;
      mask[q] = masks[static_cast<std::size_t>(c)].mask(static_cast<Eigen::Index>(k)) ? 1 : 0;
    }
  }
  std::vector<rvk_estimate> est(static_cast<std::size_t>(n));
  const int st = rvk_estimate_all(frame.frame_id, n, offsets.data(), az.data(), dop.data(),
                                  ids.data(), mask.data(), 0, est.data());
  if (st != RVK_OK) rethrow(st);
  std::vector<VelocityEstimate> out(static_cast<std::size_t>(n));
  for (int32_t c = 0; c < n; ++c) {
    const rvk_estimate& e = est[static_cast<std::size_t>(c)];
    VelocityEstimate& v = out[static_cast<std::size_t>(c)];
    v.frame_id = e.frame_id;
    v.cluster_id = e.cluster_id;
    v.v_x = e.v_x;
    v.v_y = e.v_y;
    v.heading = e.has_heading ? std::optional<double>(e.heading) : std::nullopt;
    v.inlier_count = e.inlier_count;
    v.condition_ok = e.condition_ok != 0;
  }
  return out;
}

void dbscan(Frame& frame, const ClusteringParams& params) {
  const int64_t n = static_cast<int64_t>(frame.points.size());
  std::vector<double> x(static_cast<std::size_t>(n)), y(x.size()), z(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) {
    x[i] = frame.points[i].x;
    y[i] = frame.points[i].y;
    z[i] = frame.points[i].z;
  }
  const rvk_clustering_params p{params.eps, params.min_pts,
                                params.features == ClusterFeatures::XYZ ? RVK_FEATURES_XYZ
                                                                        : RVK_FEATURES_XY};
  std::vector<int32_t> labels(x.size());
  const int st = rvk_dbscan(n, x.data(), y.data(), z.data(), &p, labels.data());
  if (st != RVK_OK) rethrow(st);  // clustering.cpp:25-30, before labels change
  frame.labels.assign(labels.begin(), labels.end());
}

std::vector<Cluster> extract_clusters(Frame& frame, int min_cluster_size) {
  if (min_cluster_size < 1)  // clustering.cpp:117-119
    throw std::invalid_argument("extract_clusters: min_cluster_size must be at least 1");
  if (frame.labels.size() != frame.points.size())  // :120-122
    throw std::invalid_argument("extract_clusters: frame labels missing; run dbscan first");
  const int64_t n = static_cast<int64_t>(frame.labels.size());
  std::vector<int32_t> labels(frame.labels.begin(), frame.labels.end());
  std::vector<int64_t> offsets(static_cast<std::size_t>(n) + 2, 0);
  std::vector<int32_t> pi(static_cast<std::size_t>(n) + 1);
  int32_t m = 0;
  const int st = rvk_extract_clusters(n, labels.data(), min_cluster_size, &m, offsets.data(),
                                      pi.data());
  if (st != RVK_OK) rethrow(st);
  frame.labels.assign(labels.begin(), labels.end());
  std::vector<Cluster> out(static_cast<std::size_t>(m));
  for (int32_t c = 0; c < m; ++c) {
    out[static_cast<std::size_t>(c)].cluster_id = c;
    out[static_cast<std::size_t>(c)].point_indices.assign(pi.begin() + offsets[c],
                                                          pi.begin() + offsets[c + 1]);
  }
  return out;
}

BoolArray combine_masks(const Frame& frame, const std::vector<InlierMask>& masks) {
  const int64_t n = static_cast<int64_t>(frame.points.size());
  BoolArray result = BoolArray::Constant(n, false);
  if (masks.empty() || frame.labels.size() != frame.points.size()) return result;  // :220-222
  std::vector<int32_t> ids(masks.size());
  std::vector<int64_t> off(masks.size() + 1, 0);
  for (std::size_t k = 0; k < masks.size(); ++k) {
    ids[k] = masks[k].cluster_id;
    off[k + 1] = off[k] + masks[k].mask.size();
  }
  std::vector<uint8_t> flat(static_cast<std::size_t>(off.back()));
  for (std::size_t k = 0; k < masks.size(); ++k)
    for (Eigen::Index q = 0; q < masks[k].mask.size(); ++q)
      flat[static_cast<std::size_t>(off[k] + q)] = masks[k].mask(q) ? 1 : 0;
  std::vector<int32_t> labels(frame.labels.begin(), frame.labels.end());
  std::vector<uint8_t> out(static_cast<std::size_t>(n));
  const int st = rvk_combine_masks(n, labels.data(), static_cast<int32_t>(masks.size()),
                                   ids.data(), off.data(), flat.data(), out.data());
  if (st != RVK_OK) rethrow(st);
  for (int64_t i = 0; i < n; ++i) result(i) = out[static_cast<std::size_t>(i)] != 0;
  return result;
}

}  // namespace rvk
