"""Host mesh builder (csrc/host/frame_mesh.cpp: incremental Delaunay +
SweepOrder) against the exact reference-order sweep — CPU tests.

The engine no longer replays planestereo::delaunayTriangulate's lexicographic
sweep (proj/src/delaunay.cpp:50-325) for every frame-iteration: it extends the
previous iteration's triangulation and recovers, only where the output depends
on it, the sweep's vertex rotation (fitPlane rounding, mesh.cpp:12-26) and its
triangle order (hull-vertex pins, mesh.cpp:109-122).  tests/cpp/test_mesh.cpp
checks the result against delaunay_lex (array-for-array equal to the compiled
reference, tests/test_delaunay.py): same triangle set, bit-identical planes,
and identical D_it at every pinned hull-vertex pixel.
"""
import os
import struct
import subprocess

import numpy as np
import pytest

import paper_1511_00758_b200 as ps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_mesh")


@pytest.fixture(scope="module")
def test_mesh_bin():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return BIN


def test_synthetic_sets(test_mesh_bin):
    """Lattices and random fills grown in three batches, with d = 0 hull
    vertices (pins) and tiny fractional disparities (rotation-dependent
    planes), including sets past the query budget (replay fallback)."""
    out = subprocess.run([test_mesh_bin, "--synthetic", "300"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok ")


def _dump(path, orc, w, h, planes, nd, ground, sigma, its, cell, seed):
    L, R = ps.synth_pair(w, h, planes, nd, ground, sigma, seed=seed)
    cfg = ps.PipelineConfig(iterations=its, maxDisparity=nd, occupancyCellSize=cell)
    r = orc.run(L, R, cfg)
    assert r["status"] == 0
    u, v, d = r["supports"]
    counts = [t["supportCount"] for t in r["trace"]]
    with open(path, "wb") as f:
        f.write(struct.pack("iiiii", w, h, nd, its, len(u)))
        f.write(np.asarray(counts, np.int32).tobytes())
        f.write(u.astype(np.int32).tobytes())
        f.write(v.astype(np.int32).tobytes())
        f.write(d.astype(np.float64).tobytes())


@pytest.mark.parametrize("seed", [5, 9])
def test_pipeline_support_lists(test_mesh_bin, orc, tmp_path, seed):
    """Every iteration's support list of BASELINE config 2 frames (VGA, grid
    10, 3 iterations; seeds 5 and 9 have ambiguous d = 0 hull pins and
    rotation-dependent planes) as the restatement produces them."""
    path = str(tmp_path / f"cfg2_{seed}.sup")
    _dump(path, orc, 640, 480, 12, 64, False, 2.0, 3, 10, seed)
    out = subprocess.run([test_mesh_bin, path], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok ")


def test_device_star_triangulation_on_cpu(test_mesh_bin, orc, tmp_path):
    """The device Delaunay (kernels/star_dt.cuh: per-point stars from a grid,
    convex hull from column extremes) compiled for the CPU: the same triangle
    set as the reference-order sweep on 3,000 synthetic sets (lattices with
    cocircular cells, random points, duplicates, collinear sets) and on every
    iteration of a BASELINE config 2 frame — for each of its search paths."""
    star = os.path.join(ROOT, "tests", "cpp", "_build", "test_star")
    path = str(tmp_path / "cfg2_9.sup")
    _dump(path, orc, 640, 480, 12, 64, False, 2.0, 3, 10, 9)
    # the per-point local pass, the grid search alone (pass 2's search), and
    # the tiled pass 1 of the device (radius 2, then 4, then the grid)
    for mode in ([], ["--no-local"], ["--tiled"]):
        out = subprocess.run([star] + mode + ["--synthetic", "3000"], capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, " ".join(mode) + out.stdout + out.stderr
        out = subprocess.run([star] + mode + [path], capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, " ".join(mode) + out.stdout + out.stderr
