"""GPU parity of the full pipeline (planestereo::run, proj/src/pipeline.cpp:131-203)
through the C ABI, against the golden fixtures (reference outputs) and the oracle.

Bar (BASELINE.json north_star): supports, costs and validity bit-exact;
disparities within 1e-3 px (in practice bit-exact: the plane arithmetic is
reproduced operation for operation); at most 0.1% validity differences and
only at exact threshold ties.  The tests below demand bit-exactness and fall
back to the tolerance only for D_f, where the tolerance is written.
"""
import numpy as np
import pytest

import paper_1511_00758_b200 as ps
from conftest import config_of, golden_names, load_golden

pytestmark = pytest.mark.gpu

D_TOL = 1e-3  # px, BASELINE.json north_star


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def assert_frame_parity(got, want, tag=""):
    """Every output map bit for bit (C_f, validity, D_f, dense and its
    validity): the mesh reproduces the reference's triangle set, the planes of
    its stored vertex rotations and its hull-vertex pins (frame_mesh.hpp), so
    no tolerance is needed; D_TOL is the north star's bound, never used."""
    assert np.array_equal(bits(got["costs"]), bits(want["costs"])), f"{tag} C_f bits"
    assert np.array_equal(got["disparity_valid"], want["disparity_valid"]), f"{tag} validity"
    assert np.array_equal(bits(got["disparity"]), bits(want["disparity"])), f"{tag} D_f bits"
    assert np.array_equal(got["dense_valid"], want["dense_valid"]), f"{tag} dense validity"
    assert np.array_equal(bits(got["dense"]), bits(want["dense"])), f"{tag} dense bits"


def result_dict(r):
    return dict(costs=r.costs, disparity_valid=r.disparity_valid, disparity=r.disparity,
                dense=r.dense, dense_valid=r.dense_valid)


@pytest.mark.parametrize("name", golden_names("pipe_"))
def test_golden_pipeline(ctx, name):
    g = load_golden(name)
    cfg = config_of(g["meta"])
    unchecked = g["meta"]["unchecked_cell"]
    if int(g["status"]) == 7:
        with pytest.raises(ps.SeedingFailed):
            ctx.run(g["left"], g["right"], cfg, unchecked_cell=unchecked)
        return
    r = ctx.run(g["left"], g["right"], cfg, unchecked_cell=unchecked)
    assert_frame_parity(result_dict(r), g, name)
    # bit-exact D_f too (plane evaluation reproduced exactly)
    assert np.array_equal(bits(r.disparity), bits(g["disparity"]))
    u, v, d = ctx.supports(0)
    assert np.array_equal(u, g["sup_u"]) and np.array_equal(v, g["sup_v"])
    assert np.array_equal(d, g["sup_d"])
    assert [t.supportCount for t in r.trace] == list(g["trace_support"])
    assert [t.triangleCount for t in r.trace] == list(g["trace_tri"])
    assert [t.occupancyCellSize for t in r.trace] == list(g["trace_cell"])
    assert [t.meanCost for t in r.trace] == list(g["trace_mean"])
    assert [t.validCount for t in r.trace] == list(g["trace_valid"])


@pytest.mark.parametrize("idx,seed", [(0, 1), (0, 2), (1, 1), (2, 3)])
def test_baseline_shapes_match_oracle(ctx, orc, idx, seed):
    c = ps.BASELINE_CONFIGS[idx]
    cfg = ps.baseline_config(idx)
    L, R = ps.synth_pair(c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                         c["sigma"], seed=seed)
    r = ctx.run(L, R, cfg, unchecked_cell=True)
    w = orc.run(L, R, cfg)
    assert_frame_parity(result_dict(r), w, f"cfg{idx}")
    u, v, d = ctx.supports(0)
    wu, wv, wd = w["supports"]
    assert np.array_equal(u, wu) and np.array_equal(v, wv) and np.array_equal(d, wd)
    assert [t.meanCost for t in r.trace] == [t["meanCost"] for t in w["trace"]]


def test_batch_equals_per_frame_oracle(ctx, orc):
    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    L, R = ps.synth_batch(12, c["width"], c["height"], c["n_planes"], c["max_disparity"],
                          c["ground"], c["sigma"], seed=500)
    res = ctx.run_batch(L, R, cfg, unchecked_cell=True)
    assert (res["status"] == 0).all()
    for f in range(12):
        w = orc.run(L[f], R[f], cfg)
        assert_frame_parity({k: res[k][f] for k in w if k in res}, w, f"frame {f}")
        assert [t.meanCost for t in res["trace"][f]] == [t["meanCost"] for t in w["trace"]]


def test_batch_with_a_failed_frame(ctx, orc):
    L, R = ps.synth_batch(3, 96, 72, 6, 32, False, 2.0, seed=9)
    L[1] = 128
    R[1] = 128
    cfg = ps.PipelineConfig(iterations=2, maxDisparity=32, occupancyCellSize=8)
    res = ctx.run_batch(L, R, cfg, raise_on_failure=False)
    assert list(res["status"]) == [0, 7, 0]
    for f in (0, 2):
        assert_frame_parity({k: res[k][f] for k in ["costs", "disparity_valid", "disparity", "dense", "dense_valid"]},
                            orc.run(L[f], R[f], cfg), f"frame {f}")
    assert res["disparity_valid"][1].sum() == 0


def test_streamed_download_into_page_locked_buffers(ctx):
    """ps_run_batch with page-locked outputs copies each frame group as it
    finishes (Engine::set_sink); the result equals the end-of-run download,
    including the zero/costHigh fill of a frame whose seeding failed."""
    import torch

    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    n = 40  # > 32 frames: several frame groups
    L, R = ps.synth_batch(n, c["width"], c["height"], c["n_planes"], c["max_disparity"],
                          c["ground"], c["sigma"], seed=77)
    L[5] = 128
    R[5] = 128
    shape = (n, c["height"], c["width"])
    out = {k: torch.full(shape, 3, dtype=dt, pin_memory=True).numpy()
           for k, dt in [("disparity", torch.float32), ("disparity_valid", torch.uint8),
                         ("costs", torch.float32), ("dense", torch.float32),
                         ("dense_valid", torch.uint8)]}
    streamed = ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False, out=out)
    plain = ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False)
    assert streamed["status"][5] == 7 and (np.delete(streamed["status"], 5) == 0).all()
    assert (streamed["status"] == plain["status"]).all()
    for k in out:
        assert np.array_equal(streamed[k].view(np.uint8), plain[k].view(np.uint8)), k
    assert streamed["costs"][5].min() == cfg.costHigh and streamed["disparity_valid"][5].sum() == 0


def test_schedules_agree(monkeypatch):
    """Frame groups seeded and refined one after another (the default event
    chain) or concurrently (PS_SERIAL_DEVICE=0), with 1 or 8 groups: the same
    bits — results do not depend on the device schedule."""
    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    n = 70  # three frame groups of uneven size
    L, R = ps.synth_batch(n, 160, 120, c["n_planes"], 40, False, 2.0, seed=31)
    cfg.maxDisparity = 40
    runs = []
    for serial, prio in (("1", "0"), ("0", "0"), ("0", "1")):
        monkeypatch.setenv("PS_SERIAL_DEVICE", serial)
        monkeypatch.setenv("PS_GROUP_PRIO", prio)
        with ps.Context(0) as cx:
            runs.append(cx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False))
            cx.set_max_groups(1)
            runs.append(cx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False))
    for r in runs[1:]:
        assert (r["status"] == runs[0]["status"]).all()
        for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
            assert np.array_equal(bits(r[k]), bits(runs[0][k])), k
        assert [[t.meanCost for t in tr] for tr in r["trace"]] == \
               [[t.meanCost for t in tr] for tr in runs[0]["trace"]]


def test_concurrent_batches_agree(ctx):
    """Two batches in flight on one GPU (two contexts, one host thread each,
    sharing the host worker pool and the device: bench.py --inflight 2) give
    the bits of each batch run alone -- the reference's threaded == sequential
    guard (proj/tests/test_pipeline.cpp:75-84,282-291) for the engine."""
    import threading

    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    batches = [ps.synth_batch(40, 320, 240, c["n_planes"], 48, False, 2.0, seed=s) for s in (71, 72)]
    cfg.maxDisparity = 48
    alone = [ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False) for L, R in batches]
    got = [None, None]
    with ps.Context(0) as c1, ps.Context(0) as c2:
        def work(i, cx):
            for _ in range(2):
                got[i] = cx.run_batch(*batches[i], cfg, unchecked_cell=True, raise_on_failure=False)

        ts = [threading.Thread(target=work, args=(0, c1)), threading.Thread(target=work, args=(1, c2))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    for a, g in zip(alone, got):
        assert (a["status"] == g["status"]).all()
        for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
            assert np.array_equal(bits(a[k]), bits(g[k])), k


def test_run_batch_multi_equals_single_context(ctx):
    """ps_run_batch_multi (frames sharded over contexts, one host thread each;
    SURVEY 8(e)) gives the single-context bits, with a failed frame in the
    second block.  Only one GPU is visible here, so both contexts sit on
    device 0 — the sharding and offsets are what is under test."""
    L, R = ps.synth_batch(11, 160, 120, 6, 40, False, 2.0, seed=61)
    L[8] = 128
    R[8] = 128
    cfg = ps.PipelineConfig(iterations=2, maxDisparity=40, occupancyCellSize=8)
    one = ctx.run_batch(L, R, cfg, raise_on_failure=False)
    with ps.Context(0) as c1, ps.Context(0) as c2:
        multi = ps.run_batch_multi([c1, c2], L, R, cfg, raise_on_failure=False)
        with pytest.raises(ps.SeedingFailed):
            ps.run_batch_multi([c1, c2], L, R, cfg)
        with pytest.raises(ps.Error):
            ps.run_batch_multi([c1, c1], L, R, cfg)
    assert list(multi["status"]) == list(one["status"]) and multi["status"][8] == 7
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert np.array_equal(bits(multi[k]), bits(one[k])), k
    assert [[t.meanCost for t in tr] for tr in multi["trace"]] == \
           [[t.meanCost for t in tr] for tr in one["trace"]]


@pytest.mark.parametrize("w,h", [(16, 16), (17, 19), (37, 23), (64, 16), (255, 17),
                                 (50, 48), (99, 64), (126, 96)])
def test_small_and_odd_sizes(ctx, orc, w, h):
    rng = np.random.default_rng(w * 100 + h)
    L = rng.integers(0, 256, (h, w), dtype=np.uint8)
    R = np.roll(L, -2, axis=1)
    cfg = ps.PipelineConfig(iterations=3, maxDisparity=8, occupancyCellSize=4, cornerThreshold=10)
    want = orc.run(L, R, cfg)
    if want["status"] == 7:
        with pytest.raises(ps.SeedingFailed):
            ctx.run(L, R, cfg)
        return
    assert_frame_parity(result_dict(ctx.run(L, R, cfg)), want)


@pytest.mark.parametrize("w,h,cell", [(254, 96, 5), (322, 120, 10), (333, 144, 2)])
def test_bulk_refine_row_wrap(ctx, orc, w, h, cell):
    """K7's bulk path when a lane's four pixels can cross a row end (W % 4 != 0,
    P % 16 == 0): the row-wrap variant of k_refine_bulk."""
    assert (w * h) % 16 == 0 and w % 4 != 0
    L, R = ps.synth_pair(w, h, 6, 32, False, 2.0, seed=w + h)
    cfg = ps.PipelineConfig(iterations=3, maxDisparity=32, occupancyCellSize=cell)
    want = orc.run(L, R, cfg)
    assert want["status"] == 0
    r = ctx.run(L, R, cfg, unchecked_cell=True)
    assert_frame_parity(result_dict(r), want)
    assert [t.meanCost for t in r.trace] == [t["meanCost"] for t in want["trace"]]


def test_random_configs_match_oracle(ctx, orc):
    rng = np.random.default_rng(42)
    for trial in range(8):
        w, h = int(rng.integers(48, 260)), int(rng.integers(40, 200))
        nd = int(rng.integers(8, 80))
        L, R = ps.synth_pair(w, h, int(rng.integers(2, 12)), nd, bool(rng.integers(0, 2)),
                             float(rng.choice([0.0, 2.0, 4.0])), seed=1000 + trial)
        low = float(rng.choice([0.15, 0.2, 0.25, 0.3]))
        cfg = ps.PipelineConfig(iterations=int(rng.integers(1, 6)), maxDisparity=nd,
                                occupancyCellSize=int(rng.integers(1, 20)), costLow=low,
                                costHigh=float(low + rng.choice([0.1, 0.2, 0.3])),
                                gradientThreshold=int(rng.integers(0, 40)),
                                cornerThreshold=int(rng.integers(5, 30)),
                                perBinCap=int(rng.integers(1, 14)),
                                sparseAcceptCost=float(rng.choice([0.2, 0.25, 0.4])),
                                uniquenessRatio=float(rng.choice([0.7, 0.8, 0.9, 1.0])))
        want = orc.run(L, R, cfg)
        if want["status"] != 0:
            with pytest.raises(ps.SeedingFailed):
                ctx.run(L, R, cfg, unchecked_cell=True)
            continue
        r = ctx.run(L, R, cfg, unchecked_cell=True)
        assert_frame_parity(result_dict(r), want, f"trial {trial}")
        assert [t.meanCost for t in r.trace] == [t["meanCost"] for t in want["trace"]]


# ------------------------------------------------ reference test_pipeline.cpp behaviour

def test_errors_and_precedence(ctx):
    # test_pipeline.cpp:292-310
    a = np.zeros((48, 64), np.uint8)
    b = np.zeros((64, 48), np.uint8)
    with pytest.raises(ps.DimensionMismatch):
        ctx.run(a, b, ps.PipelineConfig())
    with pytest.raises(ps.InvalidConfig):
        ctx.run(a, b, ps.PipelineConfig(iterations=0))
    flat = np.full((48, 64), 128, np.uint8)
    with pytest.raises(ps.SeedingFailed):
        ctx.run(flat, flat, ps.PipelineConfig())
    with pytest.raises(ps.DimensionTooSmall):
        ctx.run(np.zeros((15, 64), np.uint8), np.zeros((15, 64), np.uint8), ps.PipelineConfig())
    with pytest.raises(ps.InvalidConfig):
        ctx.run(flat, flat, ps.PipelineConfig(occupancyCellSize=10))


def test_flat_scene_accuracy_and_schedule(ctx):
    g = load_golden("pipe_render_flat20_160x120.npz")
    r = ctx.run(g["left"], g["right"], ps.PipelineConfig())
    m = r.disparity_valid.astype(bool) & g["gt_valid"].astype(bool)
    mask, _ = ctx.gradient_mask(g["left"], 20)
    m &= mask.astype(bool)
    assert m.sum() > 1000
    # test_pipeline.cpp:177-197 claims >= 99% within 1 px; the reference code itself
    # reaches 73.5% on this exact scene (tests/golden, generated by the compiled
    # reference), so the check here is equality with the reference's accuracy.
    acc = np.mean(np.abs(r.disparity[m] - 20.0) < 1.0)
    gm = g["disparity_valid"].astype(bool) & g["gt_valid"].astype(bool) & mask.astype(bool)
    assert acc == np.mean(np.abs(g["disparity"][gm] - 20.0) < 1.0)
    g7 = load_golden("pipe_render_flat10_128x96_i7.npz")
    r7 = ctx.run(g7["left"], g7["right"], ps.PipelineConfig(iterations=7))
    assert [t.occupancyCellSize for t in r7.trace] == [32, 16, 8, 4, 2, 1, 1]


def test_observer_costs_monotone_and_valid_iff_below_threshold(ctx):
    g = load_golden("pipe_render_steps_96x80_i4.npz")
    hist = []
    r = ctx.run(g["left"], g["right"], ps.PipelineConfig(iterations=4),
                observer=lambda it, d, v, c: hist.append(c))
    assert len(hist) == 4
    for a, b in zip(hist, hist[1:]):
        assert (b <= a).all()  # test_pipeline.cpp:211-230
    assert np.array_equal(hist[-1], r.costs)
    assert np.array_equal(r.disparity_valid.astype(bool), r.costs < 0.5)  # :243-253
    tr = r.trace
    for a, b in zip(tr, tr[1:]):
        assert b.supportCount >= a.supportCount and b.meanCost <= a.meanCost + 1e-9


def test_final_cost_bounded_by_wta(ctx):
    g = load_golden("pipe_render_flat11_64x64_i3.npz")
    r = ctx.run(g["left"], g["right"], ps.PipelineConfig(iterations=3))
    v = r.disparity_valid.astype(bool) & g["mask"].astype(bool)
    assert (r.costs[v] >= g["wta_cost"][v]).all()  # test_pipeline.cpp:255-268


def test_deterministic(ctx):
    g = load_golden("pipe_render_steps_96x80_i4.npz")
    a = ctx.run(g["left"], g["right"], ps.PipelineConfig(iterations=3))
    b = ctx.run(g["left"], g["right"], ps.PipelineConfig(iterations=3))
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert np.array_equal(bits(getattr(a, k)), bits(getattr(b, k)))


def test_full_size_properties_1080p(ctx):
    """cfg3 at full size: size-independent invariants (the oracle takes ~10 s here)."""
    c = ps.BASELINE_CONFIGS[3]
    cfg = ps.baseline_config(3)
    L, R = ps.synth_pair(c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                         c["sigma"], seed=3)
    hist = []
    r = ctx.run(L, R, cfg, observer=lambda it, d, v, cc: hist.append(cc))
    k = np.round(r.costs * 24)
    on_grid = (np.abs(r.costs - (k / 24).astype(np.float32)) == 0) | (r.costs == np.float32(0.5))
    assert on_grid.all()
    assert np.array_equal(r.disparity_valid.astype(bool), r.costs < cfg.costHigh)
    for a, b in zip(hist, hist[1:]):
        assert (b <= a).all()
    ok = r.disparity_valid.astype(bool)
    assert (r.disparity[ok] >= 0).all() and (r.disparity[ok] < cfg.maxDisparity).all()
    r2 = ctx.run(L, R, cfg)
    assert np.array_equal(bits(r.costs), bits(r2.costs))


def test_4k_frame_bit_exact(ctx, orc):
    """Maximum-size frame (BASELINE config 4: 3840x2160, ND 256, grid 6) for two
    iterations, bit for bit against the restatement: every output map and the
    final support list (the restatement takes a few seconds here)."""
    c = ps.BASELINE_CONFIGS[4]
    cfg = ps.baseline_config(4)
    cfg.iterations = 2
    L, R = ps.synth_pair(c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                         c["sigma"], seed=44)
    r = ctx.run(L, R, cfg, unchecked_cell=True)
    w = orc.run(L, R, cfg)  # validate() skipped: grid 6 is BASELINE's, not a power of two
    assert w["status"] == 0
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert np.array_equal(bits(getattr(r, k)), bits(w[k])), k
    u, v, d = ctx.supports(0)
    su, sv, sd = w["supports"]
    assert np.array_equal(u, su) and np.array_equal(v, sv) and np.array_equal(bits(d), bits(sd))
    assert [t.meanCost for t in r.trace] == [t["meanCost"] for t in w["trace"]]
