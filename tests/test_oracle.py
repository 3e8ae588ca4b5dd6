"""The oracle (oracle/ps_oracle.c) pinned against the reference itself.

* golden fixtures (tests/golden/*.npz, generated from the compiled reference by
  tests/golden/gen_golden.py) — bit-exact, runs everywhere;
* direct diffs against oracle/_ref (the reference sources compiled in place)
  on seeded inputs — wherever that build exists.
"""
import numpy as np
import pytest

from conftest import config_of, golden_names, load_golden

PIPE = golden_names("pipe_")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("name", PIPE)
def test_oracle_matches_golden_pipeline(orc, name):
    g = load_golden(name)
    cfg = config_of(g["meta"])
    out = orc.run(g["left"], g["right"], cfg)
    assert out["status"] == int(g["status"])
    if out["status"] != 0:
        return
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert np.array_equal(bits(out[k]), bits(g[k])), k
    su, sv, sd = out["supports"]
    assert np.array_equal(su, g["sup_u"]) and np.array_equal(sv, g["sup_v"])
    assert np.array_equal(sd, g["sup_d"])
    tr = out["trace"]
    assert [t["supportCount"] for t in tr] == list(g["trace_support"])
    assert [t["triangleCount"] for t in tr] == list(g["trace_tri"])
    assert [t["occupancyCellSize"] for t in tr] == list(g["trace_cell"])
    assert [t["meanCost"] for t in tr] == list(g["trace_mean"])
    assert [t["validCount"] for t in tr] == list(g["trace_valid"])


def test_oracle_matches_golden_stages(orc):
    import paper_1511_00758_b200 as ps

    g = load_golden("stages_random_64x48.npz")
    cfg = ps.PipelineConfig()
    assert np.array_equal(orc.census(g["image"]), g["census"])
    for t in (0, 10, 20, 35):
        assert np.array_equal(orc.gradient_mask(g["image"], t)[0], g[f"mask_t{t}"])
    cu, cv, cs = orc.detect_candidates(g["image"], cfg)
    assert np.array_equal(cu, g["cand_u"]) and np.array_equal(cv, g["cand_v"])
    assert np.array_equal(cs, g["cand_score"])
    u, v, d = orc.match_epipolar(g["census"], g["census"], cu, cv, cfg)
    assert np.array_equal(u, g["self_u"]) and np.array_equal(d, g["self_d"])
    u, v, d = orc.match_epipolar(g["census"], orc.census(g["shift_image"]), cu, cv, cfg)
    assert np.array_equal(u, g["shift_u"]) and np.array_equal(d, g["shift_d"])
    assert np.array_equal(orc.delaunay(g["lattice_u"], g["lattice_v"]), g["lattice_tris"])
    assert np.array_equal(orc.delaunay(g["pts_u"], g["pts_v"]), g["pts_tris"])
    planes, lookup = orc.mesh_build(g["pts_u"] + 2, g["pts_v"] + 2, g["pts_d"], g["pts_tris"], 64, 64)
    assert np.array_equal(bits(planes), bits(g["planes"]))
    assert np.array_equal(lookup, g["lookup"])


# ------------------------------------------------------- direct reference diffs

SYNTH_CASES = [
    # (w, h, planes, nd, ground, sigma, seed, cfg kwargs)
    (640, 480, 12, 64, False, 2.0, 1, dict(iterations=2, maxDisparity=64, occupancyCellSize=10)),
    (320, 240, 8, 64, False, 4.0, 2, dict(iterations=3, maxDisparity=64, occupancyCellSize=8)),
    (311, 203, 10, 96, True, 2.0, 3, dict(iterations=4, maxDisparity=96, occupancyCellSize=6)),
    (200, 150, 6, 40, False, 2.0, 4, dict(iterations=3, maxDisparity=40, occupancyCellSize=16,
                                          perBinCap=9, costLow=0.2, costHigh=0.55)),
]


@pytest.mark.parametrize("case", SYNTH_CASES, ids=lambda c: f"{c[0]}x{c[1]}_s{c[6]}")
def test_oracle_equals_reference_full_run(orc, ref, case):
    import paper_1511_00758_b200 as ps

    w, h, npl, nd, ground, sigma, seed, kw = case
    L, R = ps.synth_pair(w, h, npl, nd, ground, sigma, seed=seed)
    cfg = ps.PipelineConfig(**kw)
    a = ref.run(L, R, cfg)
    b = orc.run(L, R, cfg)
    assert a["status"] == b["status"] == 0
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert np.array_equal(bits(a[k]), bits(b[k])), k
    for x, y in zip(a["supports"], b["supports"]):
        assert np.array_equal(x, y)
    assert [t["meanCost"] for t in a["trace"]] == [t["meanCost"] for t in b["trace"]]


def test_staged_reference_equals_run(ref):
    """The staged mirror of run() used for non-power-of-two grids equals run() itself."""
    import paper_1511_00758_b200 as ps

    L, R = ps.synth_pair(256, 192, 8, 64, False, 2.0, seed=9)
    cfg = ps.PipelineConfig(iterations=3, maxDisparity=64, occupancyCellSize=16)
    a = ref.run(L, R, cfg, validate=0)
    b = ref.run(L, R, cfg, validate=2)
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert np.array_equal(bits(a[k]), bits(b[k])), k


def test_oracle_stages_equal_reference(orc, ref):
    import paper_1511_00758_b200 as ps

    rng = np.random.default_rng(5)
    for trial in range(6):
        w, h = int(rng.integers(24, 120)), int(rng.integers(24, 100))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        img2 = rng.integers(0, 256, (h, w), dtype=np.uint8)
        cfg = ps.PipelineConfig(perBinCap=int(rng.integers(1, 12)),
                                cornerThreshold=int(rng.integers(5, 40)),
                                maxDisparity=int(rng.integers(1, 80)))
        assert np.array_equal(orc.census(img), ref.census(img))
        thr = int(rng.integers(0, 60))
        assert np.array_equal(orc.gradient_mask(img, thr)[0], ref.gradient_mask(img, thr)[0])
        a = orc.detect_candidates(img, cfg)
        b = ref.detect_candidates(img, cfg)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        cl, cr = ref.census(img), ref.census(img2)
        cu = rng.integers(0, w, 50).astype(np.int32)
        cv = rng.integers(0, h, 50).astype(np.int32)
        cu[10:14] = cu[0]  # duplicate pixels exercise the per-pixel dedup
        cv[10:14] = cv[0]
        for x, y in zip(orc.match_epipolar(cl, cr, cu, cv, cfg), ref.match_epipolar(cl, cr, cu, cv, cfg)):
            assert np.array_equal(x, y)


def test_oracle_refinement_and_resampling_equal_reference(orc, ref):
    import paper_1511_00758_b200 as ps

    rng = np.random.default_rng(8)
    w, h = 90, 70
    img = rng.integers(0, 256, (h, w), dtype=np.uint8)
    img2 = rng.integers(0, 256, (h, w), dtype=np.uint8)
    cfg = ps.PipelineConfig()
    mask = (rng.random((h, w)) < 0.7).astype(np.uint8)
    val = (rng.random((h, w)) * 30).astype(np.float32)
    ok = (rng.random((h, w)) < 0.9).astype(np.uint8)
    val = np.where(ok == 1, val, np.float32(0))  # DisparityMap: invalid pixels hold 0 (disparity.hpp:23-26)
    cost =(rng.integers(0, 25, (h, w)) / np.float32(24)).astype(np.float32)
    for cell in (1, 3, 8, 32):
        fd1 = np.zeros((h, w), np.float32); fv1 = np.zeros((h, w), np.uint8)
        fc1 = np.full((h, w), 0.5, np.float32)
        fd2, fv2, fc2 = fd1.copy(), fv1.copy(), fc1.copy()
        ga = orc.refinement(val, ok, cost, fd1, fv1, fc1, mask, cell, cfg)
        gb = ref.refinement(val, ok, cost, fd2, fv2, fc2, mask, cell, cfg)
        assert np.array_equal(fd1, fd2) and np.array_equal(fv1, fv2) and np.array_equal(fc1, fc2)
        assert np.array_equal(ga[0], gb[0]) and np.array_equal(ga[1], gb[1])
        cl, cr = ref.census(img), ref.census(img2)
        su = rng.integers(2, w - 2, 20).astype(np.int32)
        sv = rng.integers(2, h - 2, 20).astype(np.int32)
        sd = rng.integers(0, 20, 20).astype(np.float64)
        a = orc.support_resampling(ga[0], ga[1], cell, su, sv, sd, cl, cr, cfg)
        b = ref.support_resampling(gb[0], gb[1], cell, su, sv, sd, cl, cr, cfg)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_oracle_delaunay_order_equals_reference(orc, ref):
    rng = np.random.default_rng(3)
    for trial in range(300):
        n = int(rng.integers(3, 120))
        span = int(rng.choice([8, 30, 200]))
        u = rng.integers(0, span, n).astype(np.int32)
        v = rng.integers(0, span, n).astype(np.int32)
        assert np.array_equal(orc.delaunay(u, v), ref.delaunay(u, v))


def test_oracle_predicates(orc):
    # proj/tests/test_delaunay.cpp:26-36
    assert orc.orient2d((0, 0), (4, 0), (0, 4)) > 0
    assert orc.orient2d((0, 0), (0, 4), (4, 0)) < 0
    assert orc.orient2d((0, 0), (4, 4), (8, 8)) == 0
    assert orc.incircle_sign((0, 0), (4, 0), (0, 4), (1, 1)) > 0
    assert orc.incircle_sign((0, 0), (4, 0), (0, 4), (9, 9)) < 0
    assert orc.incircle_sign((0, 0), (4, 0), (0, 4), (4, 4)) == 0


def _wta_cases():
    import json
    import os

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "wta_cases.npz"))
    return {name: {k: z[f"{name}_{k}"] for k in ("left", "right", "mask", "nd", "disparity", "valid", "cost")}
            for name in json.loads(str(z["cases"]))}


def test_oracle_wta_matches_golden(orc):
    """wtaOracle restatement vs the reference's outputs (tests/golden/wta_cases.npz)."""
    for name, c in _wta_cases().items():
        d, ok, cost = orc.wta(c["left"], c["right"], c["mask"], int(c["nd"]))
        assert np.array_equal(ok, c["valid"]), name
        assert np.array_equal(d.view(np.uint32), c["disparity"].view(np.uint32)), name
        assert np.array_equal(cost.view(np.uint32), c["cost"].view(np.uint32)), name


def test_oracle_wta_equals_reference(orc, ref):
    rng = np.random.default_rng(33)
    for w, h, nd in [(64, 40, 24), (33, 17, 100), (80, 60, 0)]:
        L = rng.integers(0, 256, (h, w), dtype=np.uint8)
        R = np.roll(L, 3, axis=1)
        m = (rng.random((h, w)) < 0.5).astype(np.uint8)
        for a, b in zip(orc.wta(L, R, m, nd), ref.wta(L, R, m, nd)):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_oracle_encoders_reference_known_answers(orc):
    """The io.cpp encoder restatements against the reference's own known
    answers (proj/tests/test_io.cpp:144-312); io.cpp itself cannot be compiled
    here (it needs libpng), so these pin the restatement."""
    # KITTI: raw = lround(d * 256), big-endian, raw 0 reserved (test_io.cpp:179-200)
    d = np.zeros((16, 20), np.float32)
    ok = np.zeros((16, 20), np.uint8)
    for u, val in [(4, 2.0), (5, 0.5), (6, 63.75)]:
        d[4, u], ok[4, u] = val, 1
    raster, neg = orc.encode_kitti16(d, ok)
    assert neg == -1
    raw = raster[:, 0::2].astype(np.int32) << 8 | raster[:, 1::2]
    assert raw[4, 4] == 512 and raw[4, 5] == 128 and raw[4, 6] == 16320
    assert (raw > 0).sum() == 3
    # round trip within the codec precision (test_io.cpp:202-216), clamp at both ends
    rng = np.random.default_rng(31)
    d = rng.uniform(0.01, 127.0, (19, 25)).astype(np.float32)
    ok = (rng.random((19, 25)) < 0.75).astype(np.uint8)
    d[0, 0], ok[0, 0] = 0.0, 1      # raw 0 -> clamped to 1
    d[0, 1], ok[0, 1] = 300.0, 1    # raw 76800 -> clamped to 65535
    raster, neg = orc.encode_kitti16(d, ok)
    raw = raster[:, 0::2].astype(np.int32) << 8 | raster[:, 1::2]
    assert neg == -1 and ((raw > 0) == (ok == 1)).all()
    assert raw[0, 0] == 1 and raw[0, 1] == 65535
    m = (ok == 1)
    m[0, :2] = False
    assert (np.abs(raw[m] / 256.0 - d[m]) <= 1.0 / 256.0).all()
    # negative disparities cannot be encoded (test_io.cpp:218-224)
    d = np.zeros((16, 16), np.float32)
    ok = np.zeros((16, 16), np.uint8)
    d[3, 3], ok[3, 3] = -1.0, 1
    assert orc.encode_kitti16(d, ok)[1] == 3 * 16 + 3
    # PFM: bottom-up rows, invalid -1, bit-exact round trip (test_io.cpp:144-159)
    d = rng.uniform(0.01, 127.0, (17, 31)).astype(np.float32)
    ok = (rng.random((17, 31)) < 0.75).astype(np.uint8)
    pfm = orc.encode_pfm(d, ok)
    back = pfm[::-1]
    assert ((back > 0) == (ok == 1)).all() and np.array_equal(back[ok == 1], d[ok == 1])
    assert (back[ok == 0] == -1.0).all()
    # point cloud (test_io.cpp:232-274, 301-310)
    img = np.full((32, 32), 200, np.uint8)
    d = np.zeros((32, 32), np.float32)
    ok = np.zeros((32, 32), np.uint8)
    for (u, v, val) in [(16, 16, 25.0), (20, 16, 25.0), (4, 4, 0.2)]:
        d[v, u], ok[v, u] = val, 1
    xyz, inten = orc.point_cloud(d, ok, img, (100.0, 0.5, 16.0, 16.0))
    assert len(xyz) == 2 and (inten == 200).all()
    assert np.allclose(xyz[0], [0.0, 0.0, 2.0]) and np.allclose(xyz[1], [(20 - 16) * 2.0 / 100.0, 0.0, 2.0])
    assert len(orc.point_cloud(np.zeros((16, 16), np.float32), np.zeros((16, 16), np.uint8),
                               img[:16, :16], (100.0, 0.5, 8.0, 8.0))[0]) == 0
    assert orc.point_cloud(d, ok, img, (0.0, 0.5, 0.0, 0.0))[0] is None


def test_oracle_accuracy_equals_reference(orc, ref):
    """accuracy restatement vs the compiled reference (proj/src/eval.cpp:19-70),
    including the sequential binary64 error sum and NoOverlap."""
    rng = np.random.default_rng(41)
    for h, w in [(48, 64), (120, 160)]:
        p = rng.uniform(0, 60, (h, w)).astype(np.float32)
        pv = (rng.random((h, w)) < 0.8).astype(np.uint8)
        g = (p + rng.normal(0, 2, (h, w))).astype(np.float32)
        gv = (rng.random((h, w)) < 0.8).astype(np.uint8)
        m = (rng.random((h, w)) < 0.6).astype(np.uint8)
        for mm in (None, m):
            a = orc.accuracy(p, pv, g, gv, mm, [0.5, 1.0, 2.0, 3.0])
            b = ref.accuracy(p, pv, g, gv, mm, [0.5, 1.0, 2.0, 3.0])
            assert a[0] == b[0] == 0 and np.array_equal(a[1], b[1]) and a[2] == b[2] and a[3] == b[3]
    assert orc.accuracy(p, pv * 0, g, gv, None, [1.0])[0] == ref.accuracy(p, pv * 0, g, gv, None, [1.0])[0] == 13
