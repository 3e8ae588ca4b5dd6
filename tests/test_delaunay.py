"""Product Delaunay (host C++, csrc/host/delaunay.cpp) — CPU tests.

Contract: the triangle SET equals the reference's
delaunayTriangulate output (order and rotation are free).  Also re-expresses
the reference's own Delaunay unit tests (proj/tests/test_delaunay.cpp).
"""
import numpy as np
import pytest

import paper_1511_00758_b200 as ps
from conftest import load_golden


def canon(tris):
    out = set()
    for a, b, c in np.asarray(tris).reshape(-1, 3):
        out.add(min([(a, b, c), (b, c, a), (c, a, b)]))
    return out


def orient(p, q, r):
    return (q[0] - p[0]) * (r[1] - p[1]) - (q[1] - p[1]) * (r[0] - p[0])


def incircle_det(a, b, c, d):
    adx, ady = a[0] - d[0], a[1] - d[1]
    bdx, bdy = b[0] - d[0], b[1] - d[1]
    cdx, cdy = c[0] - d[0], c[1] - d[1]
    aq, bq, cq = adx * adx + ady * ady, bdx * bdx + bdy * bdy, cdx * cdx + cdy * cdy
    return adx * (bdy * cq - cdy * bq) - ady * (bdx * cq - cdx * bq) + aq * (bdx * cdy - cdx * bdy)


def tri(u, v):
    return ps.delaunay_triangulate(np.asarray(u, np.int32), np.asarray(v, np.int32))


def test_fewer_than_three_or_collinear_give_nothing():
    # test_delaunay.cpp:38-43
    assert len(tri([], [])) == 0
    assert len(tri([1, 5], [1, 9])) == 0
    assert len(tri([0, 4, 8, 12, 16], [0, 2, 4, 6, 8])) == 0
    assert len(tri([3, 3, 3, 3], [0, 9, 4, 13])) == 0


def test_three_points_and_square():
    # test_delaunay.cpp:45-58
    assert len(tri([0, 10, 4], [0, 0, 8])) == 1
    sq = [(0, 0), (8, 0), (0, 8), (8, 8)]
    t = tri([p[0] for p in sq], [p[1] for p in sq])
    assert len(t) == 2
    for a, b, c in t:
        assert orient(sq[a], sq[b], sq[c]) > 0
        for i in range(4):
            assert incircle_det(sq[a], sq[b], sq[c], sq[i]) <= 0


def test_random_sets_empty_circumcircle_and_orientation():
    # test_delaunay.cpp:60-72 (own random points; the reference's use a
    # library-specific distribution)
    rng = np.random.default_rng(0)
    for seed in range(100):
        n = 3 + seed % 48
        pts = set()
        while len(pts) < n:
            pts.add((int(rng.integers(0, 60)), int(rng.integers(0, 60))))
        pts = list(pts)
        t = tri([p[0] for p in pts], [p[1] for p in pts])
        for a, b, c in t:
            assert orient(pts[a], pts[b], pts[c]) > 0
            for i in range(n):
                assert incircle_det(pts[a], pts[b], pts[c], pts[i]) <= 0


def test_area_tiles_hull_and_edges_unique():
    # test_delaunay.cpp:74-129
    rng = np.random.default_rng(1)
    for seed in range(25):
        pts = list({(int(rng.integers(0, 50)), int(rng.integers(0, 50))) for _ in range(30)})
        t = tri([p[0] for p in pts], [p[1] for p in pts])
        area = sum(orient(pts[a], pts[b], pts[c]) for a, b, c in t)
        s = sorted(pts)

        def half(seq):
            ch = []
            for p in seq:
                while len(ch) >= 2 and orient(ch[-2], ch[-1], p) <= 0:
                    ch.pop()
                ch.append(p)
            return ch

        hull = half(s)[:-1] + half(s[::-1])[:-1]
        hull_area = sum(hull[i][0] * hull[(i + 1) % len(hull)][1] - hull[i][1] * hull[(i + 1) % len(hull)][0]
                        for i in range(len(hull)))
        assert area == hull_area
        seen = set()
        for a, b, c in t:
            for e in [(a, b), (b, c), (c, a)]:
                assert e not in seen
                seen.add(e)


def test_duplicates_keep_first_and_determinism():
    # test_delaunay.cpp:131-149
    t = tri([0, 8, 4, 8, 0], [0, 0, 6, 0, 0])
    assert len(t) == 1 and t.max() <= 2
    rng = np.random.default_rng(77)
    u = rng.integers(0, 48, 37)
    v = rng.integers(0, 48, 37)
    assert np.array_equal(tri(u, v), tri(u, v))


def test_lattice_72_triangles_matches_golden_set():
    # test_delaunay.cpp:151-164 and the reference's exact cocircular tie rule
    g = load_golden("stages_random_64x48.npz")
    t = tri(g["lattice_u"], g["lattice_v"])
    assert len(t) == 72
    assert canon(t) == canon(g["lattice_tris"])
    assert canon(tri(g["pts_u"], g["pts_v"])) == canon(g["pts_tris"])


def test_coordinate_limit():
    with pytest.raises(ps.Error):
        tri([0, 1 << 20, 3], [0, 0, 5])


def _point_sets(rng, count):
    for trial in range(count):
        kind = trial % 5
        n = int(rng.integers(3, 300))
        if kind == 0:
            u, v = rng.integers(0, 80, n), rng.integers(0, 80, n)
        elif kind == 1:  # lattice subsets: massively cocircular
            step, g = int(rng.integers(1, 5)), int(rng.integers(3, 12))
            uu, vv = np.meshgrid(np.arange(g) * step, np.arange(g) * step)
            keep = rng.random(uu.size) < 0.8
            u, v = uu.ravel()[keep], vv.ravel()[keep]
        elif kind == 2:  # jittered lattice
            uu, vv = np.meshgrid(np.arange(10) * 3, np.arange(10) * 3)
            u, v = uu.ravel() + rng.integers(-1, 2, 100), vv.ravel() + rng.integers(-1, 2, 100)
        elif kind == 3:  # tiny span, many duplicates
            u, v = rng.integers(0, 6, n), rng.integers(0, 6, n)
        else:  # wide span with negative coordinates (int128 predicate path)
            u, v = rng.integers(-30000, 30000, n), rng.integers(-20000, 20000, n)
        if len(u) < 3:
            continue
        p = rng.permutation(len(u))
        yield u[p].astype(np.int32), v[p].astype(np.int32)


def fast(u, v):
    return ps.delaunay_triangulate(np.asarray(u, np.int32), np.asarray(v, np.int32), fast=True)


def test_set_equals_oracle_restatement(orc):
    rng = np.random.default_rng(11)
    for u, v in _point_sets(rng, 1500):
        want = orc.delaunay(u, v)
        assert canon(fast(u, v)) == canon(want)        # radial sweep: same set
        assert np.array_equal(tri(u, v), want)         # lexicographic sweep: same array


def test_set_equals_compiled_reference(ref):
    rng = np.random.default_rng(12)
    for u, v in _point_sets(rng, 1500):
        want = ref.delaunay(u, v)
        assert canon(fast(u, v)) == canon(want)
        assert np.array_equal(tri(u, v), want)


def test_pipeline_support_sets_equal_reference(orc):
    """Real support lists (golden fixture runs) — fractional-d supports, s=1 lattices."""
    from conftest import golden_names

    for name in golden_names("pipe_"):
        g = load_golden(name)
        if int(g["status"]) != 0:
            continue
        u, v = g["sup_u"], g["sup_v"]
        want = orc.delaunay(u, v)
        assert canon(fast(u, v)) == canon(want), name
        assert np.array_equal(tri(u, v), want), name


def test_hull_pins_equal_all_triangle_pins():
    """The engine's hull-vertex pin walk (lex_hull_pins) equals mesh_pins over
    every triangle (tests/cpp/test_pins.cpp, 3000 random and lattice sets)."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-s", "-C", os.path.join(root, "tests", "cpp")], check=True)
    out = subprocess.run([os.path.join(root, "tests", "cpp", "_build", "test_pins")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches 0" in out.stdout
