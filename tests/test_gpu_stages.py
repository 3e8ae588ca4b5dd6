"""GPU stage kernels through the C ABI vs the oracle and the reference's own
known-answer tests (proj/tests/test_core.cpp, test_sparse.cpp, test_mesh.cpp,
test_pipeline.cpp)."""
import numpy as np
import pytest

import paper_1511_00758_b200 as ps
from conftest import load_golden, random_image

pytestmark = pytest.mark.gpu


def rand_img(w, h, seed):
    return random_image(w, h, seed)  # the reference tests' own images (testutil.hpp:10-17)


# ------------------------------------------------------------- K1 census / mask
def test_census_known_answers(ctx):
    # test_core.cpp:77-123
    c = ctx.census(np.full((16, 16), 77, np.uint8))
    assert (c == 0).all()
    img = np.full((16, 16), 50, np.uint8)
    img[8, 8] = 100
    assert ctx.census(img)[8, 8] == 0x00FFFFFF
    ramp = np.tile((10 * (np.arange(16) + 1)).astype(np.uint8), (16, 1))
    word = ctx.census(ramp)[4, 4]
    assert bin(int(word)).count("1") == 10
    exp, bit = 0, 0
    for dv in range(-2, 3):
        for du in range(-2, 3):
            if dv == 0 and du == 0:
                continue
            if ramp[4 + dv, 4 + du] < ramp[4, 4]:
                exp |= 1 << bit
            bit += 1
    assert word == exp


def test_census_and_mask_equal_oracle(ctx, orc):
    g = load_golden("stages_random_64x48.npz")
    assert np.array_equal(ctx.census(g["image"]), g["census"])
    for t in (0, 10, 20, 35):
        m, n = ctx.gradient_mask(g["image"], t)
        assert np.array_equal(m, g[f"mask_t{t}"]) and n == int(g[f"mask_t{t}"].sum())
    for w, h in [(16, 16), (131, 77), (640, 480), (1242, 375)]:
        img = rand_img(w, h, w + h)
        assert np.array_equal(ctx.census(img), orc.census(img))
        m, n = ctx.gradient_mask(img, 20)
        mo, no = orc.gradient_mask(img, 20)
        assert np.array_equal(m, mo) and n == no


def test_mask_properties(ctx):
    # test_core.cpp:20-75
    assert ctx.gradient_mask(np.full((32, 32), 100, np.uint8), 1)[1] == 0
    assert ctx.gradient_mask(rand_img(20, 18, 99), 0)[1] == (20 - 4) * (18 - 4)
    step = np.full((16, 16), 50, np.uint8)
    step[:, 8:] = 150
    m, n = ctx.gradient_mask(step, 20)
    assert n == 24 and set(np.nonzero(m)[1]) == {7, 8}


# ------------------------------------------------------------- K2 corners
def test_corners_known_answers(ctx):
    cfg = ps.PipelineConfig()
    u, v, s = ctx.detect_candidates(np.full((48, 64), 120, np.uint8), cfg)
    assert len(u) == 0  # test_sparse.cpp:24-28
    dot = np.zeros((16, 16), np.uint8)
    dot[8, 8] = 255
    u, v, s = ctx.detect_candidates(dot, cfg)
    assert list(u) == [8] and list(v) == [8] and s[0] > 0  # :30-39


def test_corners_equal_oracle(ctx, orc):
    g = load_golden("stages_random_64x48.npz")
    u, v, s = ctx.detect_candidates(g["image"], ps.PipelineConfig())
    assert np.array_equal(u, g["cand_u"]) and np.array_equal(v, g["cand_v"])
    assert np.array_equal(s, g["cand_score"])
    rng = np.random.default_rng(1)
    for trial in range(10):
        w, h = int(rng.integers(20, 700)), int(rng.integers(20, 500))
        img = ps.synth_pair(max(w, 16), max(h, 16), 4, 32, False, 2.0, seed=trial)[0]
        cfg = ps.PipelineConfig(perBinCap=int(rng.choice([1, 3, 5, 8, 9, 20, 70])),
                                cornerThreshold=int(rng.integers(0, 40)))
        a = ctx.detect_candidates(img, cfg)
        b = orc.detect_candidates(img, cfg)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), (trial, cfg)


def test_checkerboard_cap(ctx):
    board = ((np.add.outer(np.arange(80) // 8, np.arange(96) // 8) % 2) * 255).astype(np.uint8)
    u, v, s = ctx.detect_candidates(board, ps.PipelineConfig(perBinCap=5))
    bins = {}
    for uu, vv in zip(u, v):
        key = (min(11, uu * 12 // 96), min(9, vv * 10 // 80))
        bins[key] = bins.get(key, 0) + 1
    assert all(c <= 5 for c in bins.values())


# ------------------------------------------------------------- K3 matching
def test_matching_known_answers(ctx, orc):
    cfg = ps.PipelineConfig()
    img = rand_img(80, 64, 12)
    c = ctx.census(img)
    u, v, s = ctx.detect_candidates(img, cfg)
    su, sv, sd = ctx.match_epipolar(c, c, u, v, cfg)
    assert len(su) > 0 and (sd == 0).all()  # test_sparse.cpp:84-92
    for seed in (21, 22, 23):  # :94-105
        left = rand_img(96, 64, seed)
        right = rand_img(96, 64, seed + 1000)
        right[:, : 96 - 7] = left[:, 7:]
        cl, cr = ctx.census(left), ctx.census(right)
        u, v, s = ctx.detect_candidates(left, cfg)
        su, sv, sd = ctx.match_epipolar(cl, cr, u, v, cfg)
        # The reference test claims d == 7 at EVERY accepted point; the
        # reference code itself accepts a few points near the left border
        # with d < 7 on these very images (oracle/_ref, same mt19937 bytes),
        # so parity with the reference is the check, plus the bulk property.
        ou, ov, od = orc.match_epipolar(cl, cr, u, v, cfg)
        assert np.array_equal(su, ou) and np.array_equal(sd, od)
        assert len(su) > 0 and np.mean(sd == 7.0) > 0.9
    left = rand_img(64, 48, 5)  # :107-117
    right = rand_img(64, 48, 77)
    right[:, : 64 - 9] = left[:, 9:]
    su, sv, sd = ctx.match_epipolar(ctx.census(left), ctx.census(right), [3, 3, 3], [20, 30, 40], cfg)
    assert (sd <= 1.0).all()
    c = ctx.census(rand_img(64, 48, 3))  # duplicates collapse (:146-156)
    su, sv, sd = ctx.match_epipolar(c, c, [20, 20, 30], [20, 20, 25], cfg)
    assert sum((su == 20) & (sv == 20)) <= 1


def test_matching_equals_oracle(ctx, orc):
    rng = np.random.default_rng(2)
    for trial in range(8):
        w, h = int(rng.integers(40, 400)), int(rng.integers(30, 200))
        L, R = ps.synth_pair(w, h, 5, 64, False, 2.0, seed=50 + trial)
        cl, cr = orc.census(L), orc.census(R)
        cu = rng.integers(-2, w + 2, 300).astype(np.int32)
        cv = rng.integers(-2, h + 2, 300).astype(np.int32)
        cu[100:110] = cu[5]
        cv[100:110] = cv[5]
        cfg = ps.PipelineConfig(maxDisparity=int(rng.integers(1, 100)),
                                uniquenessRatio=float(rng.choice([0.5, 0.9, 1.0])),
                                sparseAcceptCost=float(rng.choice([0.1, 0.25, 1.0])))
        a = ctx.match_epipolar(cl, cr, cu, cv, cfg)
        b = orc.match_epipolar(cl, cr, cu, cv, cfg)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), trial


# ------------------------------------------------------------- K5/K6 mesh
def test_mesh_equals_golden(ctx):
    g = load_golden("stages_random_64x48.npz")
    planes, lookup = ctx.mesh_build(g["pts_u"] + 2, g["pts_v"] + 2, g["pts_d"], g["pts_tris"], 64, 64)
    assert np.array_equal(planes.view(np.uint8), g["planes"].view(np.uint8))
    assert np.array_equal(lookup, g["lookup"])


def test_mesh_known_answers(ctx):
    # test_mesh.cpp:62-74 / 168-184 (fitPlane through a one-triangle mesh)
    pl, lk = ctx.mesh_build([0, 16, 0], [0, 0, 16], [0.0, 8.0, 0.0], [[0, 1, 2]], 32, 32)
    assert np.allclose(pl[0], [0.5, 0.0, 0.0])
    val, ok = ctx.interpolate(lk, pl, 128.0)
    assert ok[4, 8] and abs(val[4, 8] - 4.0) < 1e-9 and not ok[30, 30]
    val, ok = ctx.interpolate(lk, pl, 4.0)  # invalidated, not clamped (:225-230)
    assert not ok[2, 10] and ok[4, 4]
    with pytest.raises(ps.DegenerateTriangle):
        ctx.mesh_build([0, 8, 16], [0, 0, 0], [5.0, 5.0, 5.0], [[0, 1, 2]], 32, 32)


def test_mesh_lookup_equals_oracle_on_random_meshes(ctx, orc):
    rng = np.random.default_rng(4)
    for trial in range(12):
        w, h = int(rng.integers(20, 300)), int(rng.integers(20, 200))
        n = int(rng.integers(3, 400))
        u = rng.integers(0, w, n).astype(np.int32)
        v = rng.integers(0, h, n).astype(np.int32)
        d = (rng.integers(0, 200, n) / 4.0).astype(np.float64)
        keep = np.unique(v.astype(np.int64) * w + u, return_index=True)[1]
        u, v, d = u[np.sort(keep)], v[np.sort(keep)], d[np.sort(keep)]
        t = orc.delaunay(u, v)
        if len(t) == 0:
            continue
        p1, l1 = ctx.mesh_build(u, v, d, t, w, h)
        p2, l2 = orc.mesh_build(u, v, d, t, w, h)
        assert np.array_equal(p1.view(np.uint8), p2.view(np.uint8))
        assert np.array_equal(l1, l2)
        m = (rng.random((h, w)) < 0.8).astype(np.uint8)
        val, ok = ctx.interpolate(l1, p1, 40.0, mask=m)
        cov = (l1 >= 0) & (m == 1)
        want = np.zeros((h, w), np.float32)
        vv, uu = np.nonzero(cov)
        tt = l1[cov]
        want[cov] = (p1[tt, 0] * uu + p1[tt, 1] * vv + p1[tt, 2]).astype(np.float32)
        wok = cov & (want >= 0) & (want < 40.0)
        assert np.array_equal(ok.astype(bool), wok)
        assert np.array_equal(val[wok], want[wok])


# ------------------------------------------------------------- cost evaluation
def test_cost_evaluation_known_answers(ctx):
    # test_pipeline.cpp:28-73
    img = rand_img(64, 48, 4)
    m, _ = ctx.gradient_mask(img, 20)
    c = ctx.census(img)
    zero = np.zeros((48, 64), np.float32)
    ones = np.ones((48, 64), np.uint8)
    cost = ctx.cost_evaluation(c, c, zero, ones, m)
    assert (cost[m == 1] == 0).all()
    far = np.tile(np.arange(64, dtype=np.float32) + 5, (48, 1))
    assert (ctx.cost_evaluation(c, c, far, ones, m)[m == 1] == 1.0).all()
    assert (ctx.cost_evaluation(c, c, zero, np.zeros_like(ones), m)[m == 1] == 1.0).all()


def test_cost_evaluation_equals_oracle(ctx, orc):
    rng = np.random.default_rng(6)
    L, R = ps.synth_pair(200, 150, 6, 40, False, 2.0, seed=77)
    cl, cr = orc.census(L), orc.census(R)
    m, _ = orc.gradient_mask(L, 20)
    val = (rng.random((150, 200)) * 50 - 2).astype(np.float32)
    val[0, :8] = [0.5, 1.5, 2.5, -0.5, 63.5, 3.49999, 2.50001, 0]  # rounding ties (App. A.3)
    ok = (rng.random((150, 200)) < 0.9).astype(np.uint8)
    val = np.where(ok == 1, val, np.float32(0))
    assert np.array_equal(ctx.cost_evaluation(cl, cr, val, ok, m), orc.cost_evaluation(cl, cr, val, ok, m))


# ------------------------------------------------------------- refinement / resampling stages
def test_refinement_and_resampling_equal_oracle(ctx, orc):
    rng = np.random.default_rng(8)
    w, h = 90, 70
    img = rng.integers(0, 256, (h, w), dtype=np.uint8)
    img2 = rng.integers(0, 256, (h, w), dtype=np.uint8)
    cfg = ps.PipelineConfig()
    mask = (rng.random((h, w)) < 0.7).astype(np.uint8)
    ok = (rng.random((h, w)) < 0.9).astype(np.uint8)
    val = np.where(ok == 1, (rng.random((h, w)) * 30).astype(np.float32), np.float32(0))
    # arbitrary float costs (not only k/24), including exact ties
    cost = rng.choice(np.array([0.0, 0.05, 0.1, 0.1, 0.25, 0.3, 0.5, 0.8, 0.9, 1.0], np.float32),
                      size=(h, w)).astype(np.float32)
    cl, cr = orc.census(img), orc.census(img2)
    for cell in (1, 3, 8, 32):
        fd1 = np.zeros((h, w), np.float32); fv1 = np.zeros((h, w), np.uint8)
        fc1 = np.full((h, w), 0.5, np.float32)
        fd2, fv2, fc2 = fd1.copy(), fv1.copy(), fc1.copy()
        g1 = ctx.refinement(val, ok, cost, fd1, fv1, fc1, mask, cell, cfg)
        g2 = orc.refinement(val, ok, cost, fd2, fv2, fc2, mask, cell, cfg)
        assert np.array_equal(fd1, fd2) and np.array_equal(fv1, fv2) and np.array_equal(fc1, fc2)
        for a, b in zip(g1, g2):
            assert a.tobytes() == b.tobytes(), cell
        su = rng.integers(2, w - 2, 20).astype(np.int32)
        sv = rng.integers(2, h - 2, 20).astype(np.int32)
        sd = rng.integers(0, 20, 20).astype(np.float64)
        a = ctx.support_resampling(g1[0], g1[1], cell, su, sv, sd, cl, cr, cfg)
        b = orc.support_resampling(g2[0], g2[1], cell, su, sv, sd, cl, cr, cfg)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), cell


def _wta_cases():
    import json
    import os

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "wta_cases.npz"))
    return {name: {k: z[f"{name}_{k}"] for k in z.files if k.startswith(name + "_")
                   for k in [k[len(name) + 1:]]}
            for name in json.loads(str(z["cases"]))}


@pytest.mark.gpu
def test_wta_equals_reference_golden(ctx):
    """GPU wtaOracle vs the reference's own outputs, bit for bit."""
    for name, c in _wta_cases().items():
        d, ok, cost = ctx.wta_oracle(c["left"], c["right"], c["mask"], int(c["nd"]))
        assert np.array_equal(ok, c["valid"]), name
        assert np.array_equal(d.view(np.uint32), c["disparity"].view(np.uint32)), name
        assert np.array_equal(cost.view(np.uint32), c["cost"].view(np.uint32)), name


@pytest.mark.gpu
def test_wta_reference_behaviour(ctx):
    """proj/tests/test_synth.cpp:82-108: identical images give d = 0 and cost 0
    on every mask pixel; a rendered constant shift of 7 is recovered almost
    everywhere.  (The reference test asks for >= 99%; the compiled reference
    itself reaches 96.5% on this render — tests/golden/wta_cases.npz — so the
    bar here is the reference's own figure, which the GPU matches exactly.)"""
    c = _wta_cases()
    ident = c["identical"]
    d, ok, cost = ctx.wta_oracle(ident["left"], ident["right"], ident["mask"], 128)
    m = ident["mask"].astype(bool)
    assert ok[m].all() and (d[m] == 0).all() and (cost[m] == 0).all()
    s = c["shift7"]
    d, ok, cost = ctx.wta_oracle(s["left"], s["right"], s["mask"], 128)
    both = s["mask"].astype(bool) & (s["gt_valid"] == 1) & (ok == 1)
    assert both.sum() > 500
    ref_rate = (s["disparity"][both] == 7.0).mean()
    assert (d[both] == 7.0).mean() == ref_rate >= 0.95


@pytest.mark.gpu
def test_wta_batch_equals_oracle(ctx, orc):
    n, w, h = 5, 160, 120
    L, R = ps.synth_batch(n, w, h, 8, 64, False, 2.0, seed=61)
    for nd in (64, 255):
        d, ok, cost = ctx.wta_batch(L, R, 20, nd)
        for f in range(n):
            m, _ = orc.gradient_mask(L[f], 20)
            od, ook, oc = orc.wta(L[f], R[f], m, nd)
            assert np.array_equal(ok[f], ook)
            assert np.array_equal(d[f].view(np.uint32), od.view(np.uint32))
            assert np.array_equal(cost[f].view(np.uint32), oc.view(np.uint32))


@pytest.mark.gpu
def test_wta_vga_properties(ctx, orc):
    """Full VGA frame at config 2's ND: against the oracle and as the lower bound of
    the pipeline's final costs (proj/tests/test_pipeline.cpp:255-268)."""
    L, R = ps.synth_pair(640, 480, 40, 64, seed=5)
    cfg = ps.baseline_config(2)
    res = ctx.run(L, R, cfg, unchecked_cell=True)
    m, _ = ctx.gradient_mask(L, cfg.gradientThreshold)
    d, ok, cost = ctx.wta_oracle(L, R, m, cfg.maxDisparity)
    od, ook, oc = orc.wta(L, R, m, cfg.maxDisparity)
    assert np.array_equal(ok, ook) and np.array_equal(d, od) and np.array_equal(cost, oc)
    v = res.disparity_valid.astype(bool)
    assert (res.costs[v] >= cost[v]).all()
    assert ok[m.astype(bool)].all()
