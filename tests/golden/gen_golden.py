"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/gen_golden.py
It needs oracle/_ref/libps_ref.so (``make -C oracle ref``), i.e. the unmodified
reference sources compiled in place.  The fixtures store the seeded inputs
and the reference's outputs, so the GPU box (which has no /root/reference)
can check both the C restatement and the CUDA product against them.

Scenes: the BASELINE-style generator of the product (ps_synth_pair, a
seeded fixture) at small sizes, and the reference's own
renderScene scenes used by proj/tests/test_pipeline.cpp (flat / steps /
slanted), plus per-stage known-answer inputs.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1511_00758_b200 as ps  # noqa: E402


def cfg_dict(cfg: ps.PipelineConfig) -> dict:
    return {f: getattr(cfg, f) for f in cfg.__dataclass_fields__}


def render(ref, kind, p, w, h, seed=1234, max_disp=128.0):
    L = np.zeros((h, w), np.uint8)
    R = np.zeros((h, w), np.uint8)
    gt = np.zeros((h, w), np.float32)
    gv = np.zeros((h, w), np.uint8)
    fn = ref.lib.ref_render_scene
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_uint32,
                   C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    st = fn(kind, *(list(p) + [0.0] * (3 - len(p))), w, h, seed, max_disp,
            L.ctypes.data_as(C.c_void_p), R.ctypes.data_as(C.c_void_p),
            gt.ctypes.data_as(C.c_void_p), gv.ctypes.data_as(C.c_void_p))
    assert st == 0
    return L, R, gt, gv


def wta(ref, L, R, mask, nd):
    h, w = L.shape
    fn = ref.lib.ref_wta
    fn.restype = None
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                   C.c_void_p, C.c_void_p]
    d = np.zeros((h, w), np.float32)
    v = np.zeros((h, w), np.uint8)
    c = np.zeros((h, w), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    fn(p(L), p(R), w, h, p(np.ascontiguousarray(mask, np.uint8)), nd, p(d), p(v), p(c))
    return d, v, c


def save_pipeline(ref, name, L, R, cfg, validate=0, extra=None):
    out = ref.run(L, R, cfg, validate=validate)
    if validate == 0 and all((cfg.occupancyCellSize & (cfg.occupancyCellSize - 1)) == 0 for _ in [0]):
        # the staged loop must equal planestereo::run itself (pipeline.cpp:131-203)
        direct = ref.run(L, R, cfg, validate=2)
        if out["status"] == 0:
            for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
                assert np.array_equal(out[k].view(np.uint8), direct[k].view(np.uint8)), (name, k)
    arrays = dict(left=L, right=R, status=np.int32(out["status"]))
    if out["status"] == 0:
        su, sv, sd = out["supports"]
        tr = out["trace"]
        arrays.update(
            disparity=out["disparity"], disparity_valid=out["disparity_valid"],
            costs=out["costs"], dense=out["dense"], dense_valid=out["dense_valid"],
            sup_u=su, sup_v=sv, sup_d=sd,
            trace_support=np.array([t["supportCount"] for t in tr], np.int32),
            trace_tri=np.array([t["triangleCount"] for t in tr], np.int32),
            trace_cell=np.array([t["occupancyCellSize"] for t in tr], np.int32),
            trace_mean=np.array([t["meanCost"] for t in tr], np.float64),
            trace_valid=np.array([t["validCount"] for t in tr], np.int32))
    if extra:
        arrays.update(extra)
    meta = dict(kind="pipeline", config=cfg_dict(cfg),
                unchecked_cell=bool(cfg.occupancyCellSize & (cfg.occupancyCellSize - 1)))
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    print(name, "status", out["status"], "valid", int(out["disparity_valid"].sum()))


def main():
    ref = oracle.load_ref()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"

    # BASELINE-style synthetic scenes at fixture size.
    L, R = ps.synth_pair(96, 72, 6, 32, False, 2.0, seed=11)
    save_pipeline(ref, "pipe_synth_96x72_c8_i3",
                  L, R, ps.PipelineConfig(iterations=3, maxDisparity=32, occupancyCellSize=8))
    L, R = ps.synth_pair(128, 96, 8, 48, True, 2.0, seed=12)
    save_pipeline(ref, "pipe_synth_128x96_c10_i4_ground",
                  L, R, ps.PipelineConfig(iterations=4, maxDisparity=48, occupancyCellSize=10))
    L, R = ps.synth_pair(99, 67, 5, 24, False, 4.0, seed=13)  # P odd: scalar kernel paths
    save_pipeline(ref, "pipe_synth_99x67_c6_i5_odd",
                  L, R, ps.PipelineConfig(iterations=5, maxDisparity=24, occupancyCellSize=6))
    L, R = ps.synth_pair(160, 120, 10, 64, False, 2.0, seed=14)
    save_pipeline(ref, "pipe_synth_160x120_cap12",
                  L, R, ps.PipelineConfig(iterations=3, maxDisparity=64, occupancyCellSize=16,
                                          perBinCap=12, cornerThreshold=15))
    L, R = ps.synth_pair(120, 90, 6, 40, False, 2.0, seed=15)
    save_pipeline(ref, "pipe_synth_120x90_thresholds",
                  L, R, ps.PipelineConfig(iterations=3, maxDisparity=40, occupancyCellSize=8,
                                          costLow=0.3, costHigh=0.45, gradientThreshold=12,
                                          sparseAcceptCost=0.3, uniquenessRatio=0.8))

    # The reference's own rendered scenes (proj/tests/test_pipeline.cpp).
    L, R, gt, gv = render(ref, 0, [20.0], 160, 120)
    save_pipeline(ref, "pipe_render_flat20_160x120", L, R, ps.PipelineConfig(),
                  extra=dict(gt=gt, gt_valid=gv))
    L, R, gt, gv = render(ref, 0, [10.0], 128, 96)
    save_pipeline(ref, "pipe_render_flat10_128x96_i7", L, R, ps.PipelineConfig(iterations=7))
    L, R, gt, gv = render(ref, 2, [5.0, 17.0], 96, 80, seed=100)
    save_pipeline(ref, "pipe_render_steps_96x80_i4", L, R, ps.PipelineConfig(iterations=4))
    L, R, gt, gv = render(ref, 1, [0.08, 0.02, 6.0], 128, 96)
    save_pipeline(ref, "pipe_render_slanted_128x96_i5", L, R, ps.PipelineConfig(iterations=5))
    L, R, gt, gv = render(ref, 0, [11.0], 64, 64)
    m, _ = ref.gradient_mask(L, 20)
    wd, wv, wc = wta(ref, L, R, m, 128)
    save_pipeline(ref, "pipe_render_flat11_64x64_i3", L, R, ps.PipelineConfig(iterations=3),
                  extra=dict(wta_cost=wc, mask=m))
    flat = np.full((48, 64), 128, np.uint8)
    save_pipeline(ref, "pipe_textureless_64x48", flat, flat.copy(), ps.PipelineConfig())

    # Stage known answers.
    rng = np.random.default_rng(2024)
    img = rng.integers(0, 256, (48, 64), dtype=np.uint8)
    img2 = rng.integers(0, 256, (48, 64), dtype=np.uint8)
    cfg = ps.PipelineConfig()
    cu, cv, cs = ref.detect_candidates(img, cfg)
    cl, cr = ref.census(img), ref.census(img2)
    mu, mv, md = ref.match_epipolar(cl, cl, cu, cv, cfg)
    sh = np.roll(img, -7, axis=1)
    csh = ref.census(sh)
    su7, sv7, sd7 = ref.match_epipolar(cl, csh, cu, cv, cfg)
    masks = {f"mask_t{t}": ref.gradient_mask(img, t)[0] for t in (0, 10, 20, 35)}
    grid_u, grid_v = np.meshgrid(np.arange(7) * 4, np.arange(7) * 4)
    lat_u, lat_v = grid_u.ravel().astype(np.int32), grid_v.ravel().astype(np.int32)
    lat_t = ref.delaunay(lat_u, lat_v)
    pts_u = rng.integers(0, 60, 45).astype(np.int32)
    pts_v = rng.integers(0, 60, 45).astype(np.int32)
    pts_t = ref.delaunay(pts_u, pts_v)
    sup_d = (rng.integers(0, 200, 45) / 2.0).astype(np.float64)
    planes, lookup = ref.mesh_build(pts_u + 2, pts_v + 2, sup_d, pts_t, 64, 64)
    np.savez_compressed(
        os.path.join(HERE, "stages_random_64x48.npz"), image=img, image2=img2, census=cl,
        census2=cr, cand_u=cu, cand_v=cv, cand_score=cs, self_u=mu, self_v=mv, self_d=md,
        shift_image=sh, shift_u=su7, shift_v=sv7, shift_d=sd7, lattice_u=lat_u, lattice_v=lat_v,
        lattice_tris=lat_t, pts_u=pts_u, pts_v=pts_v, pts_tris=pts_t, pts_d=sup_d, planes=planes,
        lookup=lookup, meta=np.array(json.dumps(dict(kind="stages", config=cfg_dict(cfg)))),
        **masks)
    print("stages_random_64x48 ok")


def gen_wta(ref):
    """wtaOracle known answers (proj/src/synth.cpp:171-198), the reference's
    own cases (proj/tests/test_synth.cpp:82-108) plus ND edge cases."""
    cases = {}
    L, R, gt, gv = render(ref, 0, [7.0], 96, 64)  # rendered constant shift
    m, _ = ref.gradient_mask(L, 20)
    cases["shift7"] = (L, R, m, 128, dict(gt=gt, gt_valid=gv))
    L0, _, _, _ = render(ref, 0, [0.0], 64, 48)  # identical images
    m0, _ = ref.gradient_mask(L0, 20)
    cases["identical"] = (L0, L0.copy(), m0, 128, {})
    Ls, Rs = ps.synth_pair(120, 90, 6, 40, False, 2.0, seed=21)
    ms, _ = ref.gradient_mask(Ls, 12)
    cases["synth_nd40"] = (Ls, Rs, ms, 40, {})
    cases["synth_nd200"] = (Ls, Rs, ms, 200, {})  # > width: bounded by u - 2
    cases["synth_nd0"] = (Ls, Rs, ms, 0, {})
    rng = np.random.default_rng(5)
    mr = (rng.random((90, 120)) < 0.3).astype(np.uint8)  # arbitrary mask, border pixels too
    cases["synth_randmask_nd9"] = (Ls, Rs, mr, 9, {})
    arrays = {}
    for name, (L, R, m, nd, extra) in cases.items():
        d, v, c = wta(ref, L, R, m, nd)
        arrays.update({f"{name}_left": L, f"{name}_right": R, f"{name}_mask": m,
                       f"{name}_nd": np.int32(nd), f"{name}_disparity": d, f"{name}_valid": v,
                       f"{name}_cost": c})
        arrays.update({f"{name}_{k}": x for k, x in extra.items()})
    arrays["cases"] = np.array(json.dumps(sorted(cases)))
    np.savez_compressed(os.path.join(HERE, "wta_cases.npz"), **arrays)
    print("wta_cases ok")


def gen_render(ref):
    """renderScene known answers (proj/src/synth.cpp:88-169) over region lists,
    with the occlusion map and the reference's error statuses."""
    fn = ref.lib.ref_render_regions
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_int, C.c_float, C.c_uint32, C.c_void_p, C.c_void_p, C.c_int,
                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    cases = {
        "flat7_96x64": (96, 64, 128.0, 1234, [(0, 0, 96, 64, 0.0, 0.0, 7.0)]),
        "slanted_128x96": (128, 96, 128.0, 1234, [(0, 0, 128, 96, 0.08, 0.02, 6.0)]),
        "steps_97x61": (97, 61, 64.0, 77, [(0, 0, 48, 61, 0.0, 0.0, 5.0), (48, 0, 97, 61, 0.0, 0.0, 17.0)]),
        "quad_160x120": (160, 120, 96.0, 9, [(0, 0, 70, 50, 0.01, -0.02, 20.0),
                                             (70, 0, 160, 50, -0.05, 0.0, 30.5),
                                             (0, 50, 90, 120, 0.0, 0.1, 3.25),
                                             (90, 50, 160, 120, 0.0, 0.0, 0.0)]),
        "err_plane": (64, 48, 16.0, 1, [(0, 0, 64, 48, 0.3, 0.0, 0.5)]),
        "err_overlap": (64, 48, 128.0, 1, [(0, 0, 40, 48, 0, 0, 3), (30, 0, 64, 48, 0, 0, 3)]),
        "err_cover": (64, 48, 128.0, 1, [(0, 0, 40, 48, 0, 0, 3)]),
        "err_bounds": (64, 48, 128.0, 1, [(0, 0, 65, 48, 0, 0, 3)]),
    }
    arrays = {}
    for name, (w, h, md, seed, regs) in cases.items():
        box = np.array([r[:4] for r in regs], np.int32)
        pl = np.array([r[4:] for r in regs], np.float64)
        L = np.zeros((h, w), np.uint8)
        R = np.zeros((h, w), np.uint8)
        g = np.zeros((h, w), np.float32)
        gv = np.zeros((h, w), np.uint8)
        oc = np.zeros((h, w), np.uint8)
        st = fn(w, h, md, seed, p(box), p(pl), len(regs), p(L), p(R), p(g), p(gv), p(oc))
        arrays.update({f"{name}_box": box, f"{name}_plane": pl, f"{name}_status": np.int32(st),
                       f"{name}_geom": np.array([w, h, seed], np.int64), f"{name}_maxd": np.float32(md)})
        if st == 0:
            arrays.update({f"{name}_left": L, f"{name}_right": R, f"{name}_gt": g,
                           f"{name}_gt_valid": gv, f"{name}_occluded": oc})
        print(name, "status", st)
    arrays["cases"] = np.array(json.dumps(sorted(cases)))
    np.savez_compressed(os.path.join(HERE, "render_cases.npz"), **arrays)


if __name__ == "__main__":
    if sys.argv[1:] in (["wta"], ["render"]):
        ref = oracle.load_ref()
        assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
        (gen_wta if sys.argv[1] == "wta" else gen_render)(ref)
    else:
        main()
        gen_wta(oracle.load_ref())
        gen_render(oracle.load_ref())
