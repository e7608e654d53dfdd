"""CPU: workload generator pinned to the reference; C-ABI library surface.

* tools/rvk_scene.c == rvk::generate_frame (src/scene.cpp:105-189), bit-exact,
  on the golden specs and (live) on the bench shapes; the two generator
  backends of tools/workloads.py give identical frames.
* librvk_gpu.so loads without a GPU and exports every function declared in
  include/rvk_gpu.h; host-side validation (which runs before any CUDA call)
  returns the reference's status and messages.
* librvk_dropin.so exports the reference's own C++ symbols.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def test_scene_generator_matches_reference_golden(golden_scene):
    from conftest import _ensure_built
    _ensure_built()
    from tools import workloads as W
    for g in golden_scene:
        x, y, d, a, flag = W.generate(g["seed"], g["objects"])
        np.testing.assert_array_equal(x, g["x"])
        np.testing.assert_array_equal(y, g["y"])
        np.testing.assert_array_equal(d, g["doppler"])
        np.testing.assert_array_equal(a, g["azimuth"])
        np.testing.assert_array_equal(flag, g["outlier"])


def test_bench_workloads_match_reference_live(reference):
    from tools import workloads as W
    for w in (W.single_frame(), W.automotive(n_clusters=40)):
        objs = np.zeros((w.n_clusters, 10))
        # rebuild the spec the workload used and ask the reference for it
        w2 = w
        sizes = np.diff(w.offsets)
        assert sizes.min() >= 3
        _, _, d, a, flag = reference.generate_frame(w.meta["scene_seed"], _spec_of(w))
        np.testing.assert_array_equal(a, w2.azimuth)
        np.testing.assert_array_equal(d, w2.doppler)
        np.testing.assert_array_equal(flag, w2.outlier)
        del objs


def test_generator_backends_identical(reference):
    """bench.py --impl reference draws its frames through oracle/_ref's
    generate_frame + KeyedRng; our arm through tools/rvk_scene.c: the same
    arrays for every config the reference can generate (config 3's 50%
    outliers are beyond generate_frame's check, scene.cpp:39)."""
    from tools import workloads as W
    makers = [lambda: W.single_frame(seed=9), lambda: W.automotive(seed=4, n_clusters=30),
              lambda: W.imaging(seed=4003, n_clusters=300, total=60_000)]
    try:
        for mk in makers:
            W.set_generator("scene")
            a = mk()
            W.set_generator("reference")
            b = mk()
            for f in ("offsets", "azimuth", "doppler", "outlier", "truth_v"):
                np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    finally:
        W.set_generator("scene")


def _spec_of(w):
    from tools import workloads as W
    if w.name == "single":
        vx, vy = W._velocities(w.meta["scene_seed"], w.n_clusters)
        objs = np.zeros((w.n_clusters, 10))
        for i in range(w.n_clusters):
            col, row = divmod(i, 8)
            objs[i] = [15.0 + 10.0 * col, -35.0 + 10.0 * row, 2.0, 2.0, vx[i], vy[i],
                       w.offsets[i + 1] - w.offsets[i], 0.2, 0.1, 0.0]
        return objs
    u = W.rng_units(w.meta["scene_seed"], 998, 0, w.n_clusters)
    vx, vy = W._velocities(w.meta["scene_seed"], w.n_clusters, 0.5, 30.0)
    objs = np.zeros((w.n_clusters, 10))
    for i in range(w.n_clusters):
        col, row = i % 10, i // 10
        objs[i] = [10.0 + 8.0 * col, -160.0 + 16.0 * row, 0.5 + 2.0 * u[i], 0.5 + 9.5 * u[i],
                   vx[i], vy[i], w.offsets[i + 1] - w.offsets[i], 0.25, 0.1, 0.0]
    return objs


def test_workload_shapes():
    from conftest import _ensure_built
    _ensure_built()
    from tools import workloads as W
    w1 = W.single_frame()
    assert w1.n_clusters == 8 and w1.n_points == 1024 and w1.evals == 262144
    w2 = W.automotive()
    sizes = np.diff(w2.offsets)
    assert w2.n_clusters == 200 and sizes.min() >= 64 and sizes.max() <= 2048
    w4 = W.imaging()
    s4 = np.diff(w4.offsets)
    assert w4.n_clusters == 5000 and w4.n_points == 1_000_000
    assert s4.min() >= 50 and s4.max() <= 350
    w3 = W.stress()
    assert w3.max_trials == 4096 and w3.threshold_scale == 0.25
    # 50% outliers: floor(0.5 * n) per cluster
    per = np.add.reduceat(w3.outlier, w3.offsets[:-1])
    np.testing.assert_array_equal(per, np.floor(0.5 * np.diff(w3.offsets)))


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "rvk_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rvk_[a-z_0-9]+)\s*\(", text)))


def test_gpu_library_exports_every_declared_symbol():
    from conftest import _ensure_built
    _ensure_built()
    from paper_2012_12618_b200 import _native
    declared = _declared_functions()
    assert len(declared) >= 12
    lib = C.CDLL(_native.GPU_SO)
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.GPU_SIGNATURES), "binding table out of date"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.GPU_SO], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (rvk_[a-z_0-9]+)$", out, flags=re.M))
    assert set(declared) <= exported


def test_host_validation_without_gpu():
    """Validation runs before any CUDA call, in the reference's order."""
    from conftest import _ensure_built
    _ensure_built()
    import paper_2012_12618_b200 as rvk
    off = np.array([0, 3, 5], np.int64)
    az = np.zeros(5)
    with pytest.raises(ValueError, match="max_trials must be at least 1"):
        rvk.run_ransac_csr(off, az, az, rvk.RansacParams(max_trials=0))
    with pytest.raises(ValueError, match="threshold_scale must be positive"):
        rvk.run_ransac_csr(off, az, az, rvk.RansacParams(threshold_scale=0.0))
    with pytest.raises(rvk.ClusterTooSmall, match="run_ransac: cluster 1 has 2 points, need 3") \
            as e:
        rvk.run_ransac_csr(off, az, az, rvk.RansacParams())
    assert e.value.cluster == 1
    # params are checked before cluster sizes (src/ransac.cpp:140-154)
    with pytest.raises(ValueError):
        rvk.run_ransac_csr(off, az, az, rvk.RansacParams(max_trials=0))
    # the multi-device split validates the whole frame first: the index is frame-global
    off4 = np.array([0, 5, 10, 15, 17], np.int64)
    with pytest.raises(rvk.ClusterTooSmall, match="cluster 3 has 2 points") as e:
        rvk.ransac_estimate_multi_csr(off4, np.zeros(17), np.zeros(17), rvk.RansacParams(),
                                      [0, 0])
    assert e.value.cluster == 3
    with pytest.raises(ValueError, match="at least one device"):
        rvk.ransac_estimate_multi_csr(off, az, az, rvk.RansacParams(), [])
    # empty input -> empty output, no device work
    r = rvk.run_ransac_csr(np.array([0], np.int64), np.zeros(0), np.zeros(0), rvk.RansacParams())
    assert r.inlier_count.size == 0
    with pytest.raises(ValueError, match="one mask per cluster"):
        rvk.estimate_all(rvk.Frame(), [rvk.Cluster(0, np.array([0]))], [])


def test_dropin_exports_reference_symbols():
    from conftest import _ensure_built
    _ensure_built()
    so = os.path.join(ROOT, "paper_2012_12618_b200", "lib", "librvk_dropin.so")
    if not os.path.exists(so):
        pytest.skip("drop-in not built (needs the reference headers)")
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True,
                         text=True).stdout
    assert "rvk::run_ransac(std::vector<" in out
    assert "rvk::estimate_all(rvk::Frame const&" in out
