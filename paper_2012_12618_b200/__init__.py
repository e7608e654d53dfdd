"""B200-native (sm_100a) per-cluster radar velocity-profile estimator.

The hot path of arXiv 2012.12618 / the `rvk` reference: per-cluster RANSAC
inlier selection on the min-max-normalized (azimuth, Doppler) profile, the
least-squares (v_x, v_y) refit on the winning inliers, and the heading.
Kernels live in csrc/ and are reached through the C-ABI include/rvk_gpu.h;
this package is the Python mirror of the reference API on top of it.
"""
from .api import (ClusterTooSmall, Cluster, ClusteringParams, DeviceError, Frame,  # noqa: F401
                  FrameStream, InlierMask, RansacParams, combine_masks, combine_masks_labels,
                  dbscan, dbscan_points, estimate_frame,
                  extract_clusters, extract_clusters_labels,
                  RansacResult, VelocityEstimate, clusters_to_csr, cluster_thresholds_csr,
                  draw_seed_pair, estimate_all, estimate_all_csr, gather_cluster_points,
                  ransac_estimate_csr, ransac_estimate_device, ransac_estimate_multi_csr,
                  run_ransac, run_ransac_csr,
                  seed_pairs_csr, trial_counts_csr)

__all__ = [
    "ClusterTooSmall", "Cluster", "ClusteringParams", "DeviceError", "Frame", "FrameStream",
    "InlierMask", "RansacParams", "combine_masks", "combine_masks_labels", "dbscan",
    "dbscan_points", "estimate_frame", "extract_clusters",
    "extract_clusters_labels",
    "RansacResult", "VelocityEstimate", "clusters_to_csr", "cluster_thresholds_csr",
    "draw_seed_pair", "estimate_all", "estimate_all_csr", "gather_cluster_points",
    "ransac_estimate_csr", "ransac_estimate_device", "ransac_estimate_multi_csr",
    "run_ransac", "run_ransac_csr",
    "seed_pairs_csr", "trial_counts_csr",
]
