"""Clustering stage: rvk::dbscan + extract_clusters.

CPU: the C restatement (oracle/rvk_oracle.c) against the golden vectors of
the unmodified reference (tests/golden/dbscan.npz, make_golden_dbscan.py)
and live against the reference build. GPU (-m gpu): the sm_100a grid-hash
DBSCAN and extract_clusters through the C-ABI, bit-exact against the
golden vectors and the oracle, and the whole frame path rvk_estimate_frame
(dbscan -> extract -> gather -> run_ransac -> estimate_all) against the
reference pipeline of tools/rvk_main.cpp:128-141.
"""
import numpy as np
import pytest

from conftest import assert_estimates_close

FEATS = {0: "xy", 1: "xyz"}


def _frames(seed, n_frames, with_z=False):
    rng = np.random.default_rng(seed)
    for _ in range(n_frames):
        n_blobs = int(rng.integers(1, 12))
        size = int(rng.integers(3, 80))
        c = rng.uniform(-40, 40, (n_blobs, 2))
        pts = [c[b] + rng.normal(0, rng.uniform(0.2, 1.5), (size, 2)) for b in range(n_blobs)]
        pts.append(rng.uniform(-40, 40, (int(rng.integers(0, 60)), 2)))
        p = np.concatenate(pts)
        p = p[rng.permutation(len(p))]
        if rng.random() < 0.3:  # quantized: ties and exactly-eps distances
            p = np.round(p * 2) / 2
        z = rng.normal(0, 1.0, len(p)) if with_z else None
        yield p[:, 0].copy(), p[:, 1].copy(), z, float(rng.uniform(0.5, 3.0)), \
            int(rng.integers(1, 7))


# ------------------------------------------------------------------ CPU

def test_oracle_dbscan_matches_reference_golden(oracle, golden_dbscan):
    for g in golden_dbscan:
        lab = oracle.dbscan(g["x"], g["y"], g["z"], g["eps"], g["min_pts"], g["features"])
        np.testing.assert_array_equal(lab, g["labels"], err_msg=g["name"])
        lab2, off, pi = oracle.extract_clusters(lab, g["min_cluster_size"])
        np.testing.assert_array_equal(lab2, g["extracted"], err_msg=g["name"])
        np.testing.assert_array_equal(off, g["offsets"], err_msg=g["name"])
        np.testing.assert_array_equal(pi, g["point_indices"], err_msg=g["name"])


def test_oracle_dbscan_live_against_reference(oracle, reference):
    for x, y, z, eps, mp in _frames(11, 40, with_z=True):
        for feat in (0, 1):
            np.testing.assert_array_equal(oracle.dbscan(x, y, z, eps, mp, feat),
                                          reference.dbscan(x, y, z, eps, mp, feat))


def test_oracle_dbscan_validation(oracle):
    from oracle.binding import CheckerError
    with pytest.raises(CheckerError, match="eps must be positive"):
        oracle.dbscan([0.0], [0.0], None, 0.0, 3)
    with pytest.raises(CheckerError, match="min_pts must be at least 1"):
        oracle.dbscan([0.0], [0.0], None, 1.0, 0)
    with pytest.raises(CheckerError, match="min_cluster_size must be at least 1"):
        oracle.extract_clusters(np.zeros(3, np.int32), 0)


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_gpu_dbscan_golden(gpu_lib, golden_dbscan):
    import paper_2012_12618_b200 as rvk
    for g in golden_dbscan:
        p = rvk.ClusteringParams(g["eps"], g["min_pts"], FEATS[g["features"]])
        lab = rvk.dbscan_points(g["x"], g["y"], g["z"], p)
        np.testing.assert_array_equal(lab, g["labels"], err_msg=g["name"])
        lab2, off, pi = rvk.extract_clusters_labels(lab, g["min_cluster_size"])
        np.testing.assert_array_equal(lab2, g["extracted"], err_msg=g["name"])
        np.testing.assert_array_equal(off, g["offsets"], err_msg=g["name"])
        np.testing.assert_array_equal(pi, g["point_indices"], err_msg=g["name"])


@pytest.mark.gpu
def test_gpu_dbscan_random_frames_vs_oracle(gpu_lib, oracle):
    import paper_2012_12618_b200 as rvk
    for k, (x, y, z, eps, mp) in enumerate(_frames(5, 60, with_z=True)):
        feat = k % 2
        want = oracle.dbscan(x, y, z, eps, mp, feat)
        got = rvk.dbscan_points(x, y, z, rvk.ClusteringParams(eps, mp, FEATS[feat]))
        np.testing.assert_array_equal(got, want, err_msg=f"frame {k}")
        mcs = 1 + k % 4
        for a, b in zip(rvk.extract_clusters_labels(got, mcs), oracle.extract_clusters(want, mcs)):
            np.testing.assert_array_equal(a, b, err_msg=f"frame {k} extract")


@pytest.mark.gpu
def test_gpu_dbscan_edge_cases(gpu_lib, oracle):
    import paper_2012_12618_b200 as rvk
    P = rvk.ClusteringParams
    assert rvk.dbscan_points(np.zeros(0), np.zeros(0)).size == 0
    np.testing.assert_array_equal(rvk.dbscan_points([1.0], [2.0], params=P(1.0, 1)), [0])
    np.testing.assert_array_equal(rvk.dbscan_points([1.0], [2.0], params=P(1.0, 2)), [-1])
    # identical points, a chain exactly eps apart, negative and large coordinates
    same = np.full(10, 3.25)
    np.testing.assert_array_equal(rvk.dbscan_points(same, same, params=P(0.1, 10)), np.zeros(10))
    chain = np.arange(30) * 0.5 - 1e4
    np.testing.assert_array_equal(rvk.dbscan_points(chain, np.zeros(30), params=P(0.5, 3)),
                                  oracle.dbscan(chain, np.zeros(30), None, 0.5, 3))
    # a border point equidistant from two cores of different clusters
    x = np.array([0.0, 0.1, 0.2, 2.0, 3.8, 3.9, 4.0])
    y = np.zeros(7)
    np.testing.assert_array_equal(rvk.dbscan_points(x, y, params=P(1.8, 3)),
                                  oracle.dbscan(x, y, None, 1.8, 3))
    with pytest.raises(ValueError, match="eps must be positive"):
        rvk.dbscan_points([0.0], [0.0], params=P(0.0, 3))
    with pytest.raises(ValueError, match="min_pts must be at least 1"):
        rvk.dbscan_points([0.0], [0.0], params=P(1.0, 0))
    with pytest.raises(ValueError, match="min_cluster_size must be at least 1"):
        rvk.extract_clusters_labels(np.zeros(3, np.int32), 0)


@pytest.mark.gpu
def test_gpu_dbscan_large_radar_frame(gpu_lib, reference):
    """A 20k-point radar frame from the reference's generate_frame."""
    import paper_2012_12618_b200 as rvk
    from tools import workloads as W
    w = W.imaging(seed=77, n_clusters=100, total=20000)
    x, y = w.x, w.y
    want = reference.dbscan(x, y, None, 2.0, 3, 0)
    got = rvk.dbscan_points(x, y, params=rvk.ClusteringParams(2.0, 3))
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_gpu_estimate_frame_matches_reference_pipeline(gpu_lib, reference):
    """rvk_estimate_frame == the reference's frame loop body
    (tools/rvk_main.cpp:128-141) on radar frames."""
    import paper_2012_12618_b200 as rvk
    from oracle.binding import make_params
    from tools import workloads as W
    for s in range(3):
        w = W.automotive(seed=300 + s, n_clusters=40)
        fr = rvk.Frame(frame_id=s, x=w.x, y=w.y, z=np.zeros(w.n_points), doppler=w.doppler,
                       azimuth=w.azimuth)
        rp = rvk.RansacParams(256, 1.0, 9)
        labels, off, pi, res, est = rvk.estimate_frame(fr, rvk.ClusteringParams(2.0, 3), rp)
        rl = reference.dbscan(w.x, w.y, None, 2.0, 3, 0)
        rl2, roff, rpi = reference.extract_clusters(rl, 3)
        np.testing.assert_array_equal(labels, rl2)
        np.testing.assert_array_equal(off, roff)
        np.testing.assert_array_equal(pi, rpi)
        az, dop = w.azimuth[rpi], w.doppler[rpi]
        r, e = reference.ransac_estimate(roff, az, dop, make_params(256, 1.0, 9), frame_id=s,
                                         cluster_ids=np.arange(roff.size - 1, dtype=np.int32))
        np.testing.assert_array_equal(res.mask, r.mask)
        np.testing.assert_array_equal(res.winning_trial, r.winning_trial)
        np.testing.assert_array_equal(res.inlier_count, r.inlier_count)
        assert_estimates_close(est, e, label=f"frame {s}", frame=(roff, az, r.mask))


# ------------------------------------------------------------ combine_masks

def _random_masks(rng):
    n = int(rng.integers(0, 300))
    labels = rng.integers(-1, 8, n).astype(np.int32)
    m = int(rng.integers(0, 10))
    ids = rng.integers(-1, 9, m).astype(np.int32)  # duplicates and unknown ids too
    sizes = rng.integers(0, 60, m)
    off = np.zeros(m + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    masks = rng.integers(0, 2, int(off[-1])).astype(np.uint8)
    return labels, ids, off, masks


def test_oracle_combine_masks_live_against_reference(oracle, reference):
    rng = np.random.default_rng(21)
    for _ in range(200):
        args = _random_masks(rng)
        np.testing.assert_array_equal(oracle.combine_masks(*args), reference.combine_masks(*args))


@pytest.mark.gpu
def test_gpu_combine_masks_vs_oracle(gpu_lib, oracle):
    import paper_2012_12618_b200 as rvk
    rng = np.random.default_rng(22)
    for k in range(200):
        args = _random_masks(rng)
        np.testing.assert_array_equal(rvk.combine_masks_labels(*args), oracle.combine_masks(*args),
                                      err_msg=f"case {k}")
    # frame-level: the masks of the device pipeline on a clustered frame
    from tools import workloads as W
    w = W.automotive(seed=5, n_clusters=30)
    fr = rvk.Frame(frame_id=0, x=w.x, y=w.y, doppler=w.doppler, azimuth=w.azimuth)
    labels, off, pi, res, _ = rvk.estimate_frame(fr, rvk.ClusteringParams(2.0, 3),
                                                 rvk.RansacParams(256, 1.0, 1))
    ids = np.arange(off.size - 1, dtype=np.int32)
    got = rvk.combine_masks_labels(labels, ids, off, res.mask)
    want = np.zeros(labels.size, np.uint8)
    want[pi] = res.mask  # members in ascending order == the label ranks
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got, oracle.combine_masks(labels, ids, off, res.mask))
