"""Synthetic clustered radar frames of the BASELINE.json shapes (bench and test
infrastructure; not part of the product package).

Points come from rvk::generate_frame (/root/reference/proj/src/scene.cpp:105-189):
object points uniform in a box, azimuth = atan2(y, x), Doppler = radial
projection + sigma * N(0, 1), floor(f * n) outliers offset by +-U[2, 5] m/s.
Clusters are taken from the truth table (one cluster per object, no DBSCAN),
as src/bench.cpp:57-63 does. All layout/velocity draws use the reference's
KeyedRng, so a (config, seed) pair names a bit-identical frame everywhere.

Two interchangeable generators (tests/test_workloads_abi.py pins them equal):
  "scene"     tools/rvk_scene.c, a C restatement of generate_frame, built into
              tools/_build/librvk_scene.so -- travels with the repo and allows
              outlier_fraction 0.5 (config 3), which the reference rejects
              (scene.cpp:39);
  "reference" oracle/_ref/librvk_ref.so, the unmodified reference build
              (bench.py --impl reference uses it, so that arm maps no repo
              library besides the reference itself).

Configs (BASELINE.json "configs"):
  1 single   8 objects x 128 pts, 20% outliers, T=256   (bench.cpp:38-51 lattice)
  2 auto     200 objects, n_i = round(64 * 32^u) (64..2048), 25% outliers, T=1024
  3 stress   config-2 shapes, 50% outliers, T=4096, threshold_scale 0.25
  4 imaging  5000 objects, n_i ~ U[50, 350] summing to exactly 1,000,000, T=256
  5 stream   10k config-2 frames (scene seed = frame index), T=1024
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SCENE_SRC = os.path.join(HERE, "rvk_scene.c")
SCENE_SO = os.path.join(HERE, "_build", "librvk_scene.so")

_lock = threading.Lock()
_scene = None
_generator = os.environ.get("RVK_WORKLOAD_GENERATOR", "scene")


def build_scene(force: bool = False) -> str:
    """gcc tools/rvk_scene.c -> tools/_build/librvk_scene.so (flags of the
    reference build: no FMA contraction)."""
    os.makedirs(os.path.dirname(SCENE_SO), exist_ok=True)
    if force or not os.path.exists(SCENE_SO) or \
            os.path.getmtime(SCENE_SO) < os.path.getmtime(SCENE_SRC):
        r = subprocess.run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                            "-o", SCENE_SO, SCENE_SRC, "-lm"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("scene build failed: " + r.stderr[-3000:])
    return SCENE_SO


def _scene_lib():
    global _scene
    with _lock:
        if _scene is None:
            if not os.path.exists(SCENE_SO):
                build_scene()
            lib = C.CDLL(SCENE_SO)
            lib.rvk_scene_generate.restype = C.c_int
            lib.rvk_scene_generate.argtypes = [C.c_uint64, C.c_int32] + [C.c_void_p] + \
                [C.c_double] * 2 + [C.c_void_p] * 5
            lib.rvk_scene_rng_units.restype = None
            lib.rvk_scene_rng_units.argtypes = [C.c_uint64] * 3 + [C.c_int64, C.c_void_p]
            _scene = lib
        return _scene


def set_generator(name: str) -> None:
    """"scene" (default) or "reference" (oracle/_ref's generate_frame)."""
    global _generator
    if name not in ("scene", "reference"):
        raise ValueError(name)
    _generator = name


def generator() -> str:
    return _generator


@dataclass
class Workload:
    name: str
    offsets: np.ndarray      # int64 [C+1]
    azimuth: np.ndarray      # float64 [P]
    doppler: np.ndarray      # float64 [P]
    outlier: np.ndarray      # int32 [P] (1 = planted outlier)
    truth_v: np.ndarray      # float64 [C, 2]
    max_trials: int
    threshold_scale: float = 1.0
    rng_seed: int = 0
    meta: dict = field(default_factory=dict)
    x: np.ndarray = field(default_factory=lambda: np.zeros(0))  # float64 [P], m (frame order)
    y: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @property
    def n_clusters(self) -> int:
        return self.offsets.size - 1

    @property
    def n_points(self) -> int:
        return int(self.offsets[-1])

    @property
    def evals(self) -> int:
        """Hypothesis x point evaluations of one RANSAC pass (T * P)."""
        return self.max_trials * self.n_points


def rng_units(seed: int, hi: int, lo: int, n: int) -> np.ndarray:
    """n draws of KeyedRng(seed, hi, lo).next_unit() (include/rvk/rng.hpp:40-41)."""
    out = np.zeros(n)
    if _generator == "reference":
        from oracle.binding import Reference
        Reference().rng_units(seed, hi, lo, out)
    else:
        _scene_lib().rvk_scene_rng_units(seed & (2**64 - 1), hi, lo, n, out.ctypes.data)
    return out


def generate(seed: int, objects: np.ndarray, offset_range=(2.0, 5.0)):
    """generate_frame: objects [k, 10] -> (x, y, doppler, azimuth, outlier_flag)."""
    objects = np.ascontiguousarray(objects, dtype=np.float64).reshape(-1, 10)
    if _generator == "reference":
        from oracle.binding import Reference
        return Reference().generate_frame(seed & (2**64 - 1), objects, offset_range)
    p = int(objects[:, 6].sum())
    x, y, d, a = (np.zeros(p) for _ in range(4))
    flag = np.zeros(p, np.int32)
    st = _scene_lib().rvk_scene_generate(seed & (2**64 - 1), objects.shape[0],
                                         objects.ctypes.data, offset_range[0], offset_range[1],
                                         x.ctypes.data, y.ctypes.data, d.ctypes.data,
                                         a.ctypes.data, flag.ctypes.data)
    if st != 0:
        raise RuntimeError("rvk_scene_generate failed")
    return x, y, d, a, flag


def _frame(name, seed, objects, max_trials, threshold_scale=1.0, rng_seed=0, **meta):
    x, y, d, a, flag = generate(seed, objects)
    sizes = objects[:, 6].astype(np.int64)
    offsets = np.zeros(sizes.size + 1, np.int64)
    np.cumsum(sizes, out=offsets[1:])
    return Workload(name, offsets, a, d, flag, objects[:, 4:6].copy(), max_trials,
                    threshold_scale, rng_seed, dict(scene_seed=seed, **meta), x, y)


def _velocities(seed: int, k: int, lo=3.0, hi=18.0):
    u = rng_units(seed, 999, 0, 2 * k).reshape(k, 2)
    speed = lo + u[:, 0] * (hi - lo)
    direction = -math.pi + u[:, 1] * (2 * math.pi)
    return speed * np.cos(direction), speed * np.sin(direction)


def single_frame(seed: int = 7, n_clusters: int = 8, points: int = 128,
                 outlier_fraction: float = 0.20, max_trials: int = 256) -> Workload:
    """Config 1: make_workload's lattice (src/bench.cpp:38-51): 8 rows in y,
    columns marching out in x, 2 x 2 m boxes, sigma 0.1 m/s."""
    vx, vy = _velocities(seed, n_clusters)
    objs = np.zeros((n_clusters, 10))
    for i in range(n_clusters):
        col, row = divmod(i, 8)
        objs[i] = [15.0 + 10.0 * col, -35.0 + 10.0 * row, 2.0, 2.0, vx[i], vy[i], points,
                   outlier_fraction, 0.1, 0.0]
    return _frame("single", seed, objs, max_trials)


def automotive(seed: int = 11, n_clusters: int = 200, outlier_fraction: float = 0.25,
               max_trials: int = 1024, threshold_scale: float = 1.0, name="automotive",
               lo_pts: int = 64, hi_pts: int = 2048) -> Workload:
    """Config 2: n_i = round(64 * 32^u) (pedestrians to trucks), extent
    growing with n_i from 0.5 x 0.5 m to 2.5 x 10 m, on a 10-column lattice
    with >= 4 m gaps (x pitch 8 m, y pitch 16 m)."""
    u = rng_units(seed, 998, 0, n_clusters)
    n_pts = np.rint(lo_pts * (hi_pts / lo_pts) ** u).astype(np.int64)
    vx, vy = _velocities(seed, n_clusters, 0.5, 30.0)
    objs = np.zeros((n_clusters, 10))
    for i in range(n_clusters):
        col, row = i % 10, i // 10
        objs[i] = [10.0 + 8.0 * col, -160.0 + 16.0 * row, 0.5 + 2.0 * u[i], 0.5 + 9.5 * u[i],
                   vx[i], vy[i], n_pts[i], outlier_fraction, 0.1, 0.0]
    return _frame(name, seed, objs, max_trials, threshold_scale)


def stress(seed: int = 13, max_trials: int = 4096) -> Workload:
    """Config 3: automotive shapes with 50% micro-Doppler outliers and a tight
    corridor (threshold_scale 0.25). The reference's generate_frame rejects
    outlier_fraction >= 0.5 (scene.cpp:39); the same recipe is run without
    that check and the identical arrays are fed to both implementations."""
    return automotive(seed, 200, 0.5, max_trials, 0.25, name="stress")


def imaging(seed: int = 17, n_clusters: int = 5000, total: int = 1_000_000,
            max_trials: int = 256) -> Workload:
    """Config 4: 5000 objects, n_i ~ U[50, 350], adjusted to sum to exactly
    `total`, on a 100 x 50 lattice of 1.5 x 1.5 m boxes, 25% outliers."""
    u = rng_units(seed, 997, 0, n_clusters)
    n_pts = (50 + np.floor(u * 301)).astype(np.int64)
    diff = total - int(n_pts.sum())
    i = 0
    while diff != 0:  # deterministic round-robin fix-up inside [50, 350]
        step = 1 if diff > 0 else -1
        if 50 <= n_pts[i % n_clusters] + step <= 350:
            n_pts[i % n_clusters] += step
            diff -= step
        i += 1
    vx, vy = _velocities(seed, n_clusters, 0.5, 30.0)
    objs = np.zeros((n_clusters, 10))
    for k in range(n_clusters):
        col, row = k % 100, k // 100
        objs[k] = [8.0 + 6.0 * col, -150.0 + 6.0 * row, 1.5, 1.5, vx[k], vy[k], n_pts[k], 0.25,
                   0.1, 0.0]
    return _frame("imaging", seed, objs, max_trials)


def stream_frame(frame_index: int, max_trials: int = 1024) -> Workload:
    """Config 5 frame: config-2 shapes with scene seed = frame index."""
    w = automotive(seed=frame_index, max_trials=max_trials, name="stream")
    w.meta["frame_index"] = frame_index
    return w


CONFIGS = {
    1: single_frame,
    2: automotive,
    3: stress,
    4: imaging,
}


def random_clusters(rng: np.random.Generator, n_clusters: int, lo: int = 5, hi: int = 40,
                    az_range=(-1.3, 1.3), dop_range=(-25.0, 25.0)):
    """Uniform random clusters (acceptance C3 style, acceptance_test.cpp:264-279)."""
    sizes = rng.integers(lo, hi + 1, size=n_clusters)
    offsets = np.zeros(n_clusters + 1, np.int64)
    np.cumsum(sizes, out=offsets[1:])
    p = int(offsets[-1])
    az = rng.uniform(az_range[0], az_range[1], size=p)
    dop = rng.uniform(dop_range[0], dop_range[1], size=p)
    return offsets, az, dop
