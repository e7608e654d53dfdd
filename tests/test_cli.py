"""lib/rvk_gpu: the reference CLI's `estimate` command (tools/rvk_main.cpp:104-158)
on the device path. Modeled on the reference's
test_cli.cpp: exit codes and messages (CPU), and on the GPU the estimate CSV
against the reference's own run_estimate body (read_frames -> dbscan ->
extract -> run_ransac/estimate_all or lsq-only -> write_estimates) on the
same frames file: ids, inlier counts and heading presence exact, velocities
and headings within the north_star tolerance."""
import math
import os
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT, _ensure_built

CLI = os.path.join(ROOT, "paper_2012_12618_b200", "lib", "rvk_gpu")


def _run(*args):
    _ensure_built()
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


def test_cli_usage_errors():
    code, out = _run()
    assert code == 2 and "usage" in out
    code, out = _run("estimate", "x.csv")
    assert code == 2 and "-o are required" in out
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "f.csv")
        open(f, "w").write("frame_id,x,y,z,doppler,azimuth\n0,1,2,0,1,0.5\n")
        code, out = _run("estimate", f, "-o", os.path.join(d, "o.csv"), "--mode", "fast")
        assert code == 2 and "mode must be parallel, sequential, gpu or lsq-only" in out
        code, out = _run("estimate", f, "-o", os.path.join(d, "o.csv"), "--eps", "0")
        assert code == 2 and "invalid estimation parameters" in out


def test_cli_frame_file_errors():
    """read_frames' messages (src/frame_io.cpp:86-139), exit 2, no device work."""
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "o.csv")
        cases = [("", "empty frame file"),
                 ("frame_id,x,y\n", "expected header"),
                 ("frame_id,x,y,z,doppler,azimuth\n0,1,2,3\n", "line 2: expected 6 fields"),
                 ("frame_id,x,y,z,doppler,azimuth\nq,1,2,3,4,0\n", "line 2: bad frame_id 'q'"),
                 ("frame_id,x,y,z,doppler,azimuth\n0,1,2,3,4,0\n0,1,inf,3,4,0\n",
                  "line 3: bad y 'inf'"),
                 ("frame_id,x,y,z,doppler,azimuth\n0,1,2,3,4,4\n", "azimuth outside (-pi, pi]")]
        for i, (text, msg) in enumerate(cases):
            f = os.path.join(d, f"f{i}.csv")
            open(f, "w").write(text)
            code, log = _run("estimate", f, "-o", out)
            assert code == 2 and msg in log, (text, log)
        code, log = _run("estimate", os.path.join(d, "missing.csv"), "-o", out)
        assert code == 2 and "cannot open for reading" in log


def _read_est(path):
    lines = open(path).read().splitlines()
    assert lines[0] == "frame_id,cluster_id,v_x,v_y,heading_deg,inlier_count"
    return [ln.split(",") for ln in lines[1:]]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["gpu", "parallel", "sequential", "lsq-only"])
def test_cli_estimate_matches_reference_run_estimate(gpu_lib, reference, mode):
    from tools import workloads as W
    frames = []
    for k in range(4):
        w = W.automotive(seed=500 + k, n_clusters=25)
        frames.append((100 + k, w.x, w.y, np.zeros(w.n_points), w.doppler, w.azimuth))
    with tempfile.TemporaryDirectory() as d:
        fp = os.path.join(d, "frames.csv")
        reference.write_frames(fp, frames)
        ours, theirs = os.path.join(d, "ours.csv"), os.path.join(d, "ref.csv")
        code, log = _run("estimate", fp, "-o", ours, "--mode", mode, "--seed", "7",
                         "--max-trials", "128")
        assert code == 0, log
        reference.run_estimate_csv(fp, theirs, "lsq-only" if mode == "lsq-only" else "parallel",
                                   max_trials=128, seed=7)
        a, b = _read_est(ours), _read_est(theirs)
    assert len(a) == len(b) > 0
    for ra, rb in zip(a, b):
        assert ra[0] == rb[0] and ra[1] == rb[1] and ra[5] == rb[5]  # ids, inlier_count
        for k in (2, 3):
            assert math.isclose(float(ra[k]), float(rb[k]), rel_tol=1e-4, abs_tol=1e-9)
        ha, hb = float(ra[4]), float(rb[4])
        assert math.isnan(ha) == math.isnan(hb)
        if not math.isnan(hb):
            assert abs((ha - hb + 180.0) % 360.0 - 180.0) <= math.degrees(1e-3)


def test_cli_parallel_parse_reports_first_bad_line():
    """The frame file is parsed by all host threads in line-aligned chunks;
    the reported error must still be the first malformed row in file order
    (src/frame_io.cpp:100-132), wherever the chunk boundaries fall."""
    rng = np.random.default_rng(4)
    n = 60_000
    rows = [f"{i % 7},{x:.6f},{y:.6f},0,{d:.6f},{a:.6f}" for i, (x, y, d, a) in
            enumerate(zip(rng.uniform(-50, 50, n), rng.uniform(-50, 50, n),
                          rng.uniform(-9, 9, n), rng.uniform(-3, 3, n)))]
    rows[41_234] = "3,1.0,2.0,0,zz,0.5"          # line 41236 (header = line 1)
    rows[52_000] = "3,1.0,2.0"                   # a later error in another chunk
    rows[59_000] = "4,1.0,2.0,0,1.0,9.0"
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "f.csv")
        open(f, "w").write("frame_id,x,y,z,doppler,azimuth\n" + "\n".join(rows) + "\n")
        code, out = _run("estimate", f, "-o", os.path.join(d, "o.csv"))
        assert code == 2, out
        assert "malformed row at line 41236: bad doppler 'zz'" in out, out
