"""On-device scene generation (kernels/synth.cu): the BASELINE generator gives
the host generator's bytes, and renderScene gives the compiled reference's
images, ground truth and occlusion (tests/golden/render_cases.npz)."""
import json
import os

import numpy as np
import pytest

import paper_1511_00758_b200 as ps

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "render_cases.npz")


@pytest.mark.parametrize("w,h,planes,nd,ground,sigma,n", [
    (640, 480, 40, 64, False, 2.0, 3),     # BASELINE config 2 frames
    (1242, 375, 24, 128, True, 2.0, 2),    # config 1 (ground plane)
    (99, 67, 5, 24, False, 4.0, 4),        # odd sizes, sigma 4
    (64, 48, 0, 16, False, 0.0, 2),        # no planes, no noise
])
def test_device_generator_equals_host(ctx, w, h, planes, nd, ground, sigma, n):
    L, R = ps.synth_batch(n, w, h, planes, nd, ground, sigma, seed=1000)
    gL, gR, ggt = ctx.synth_batch(n, w, h, planes, nd, ground, sigma, seed=1000, with_gt=True)
    assert np.array_equal(gL, L)
    assert np.array_equal(gR, R)
    for f in range(n):
        _, _, gt = ps.synth_pair(w, h, planes, nd, ground, sigma, seed=1000 + f, with_gt=True)
        assert np.array_equal(ggt[f], gt)


def test_resident_generation_runs_like_uploaded_inputs(ctx):
    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    n = 6
    L, R = ps.synth_batch(n, c["width"], c["height"], c["n_planes"], c["max_disparity"],
                          c["ground"], c["sigma"], seed=55)
    ref = ctx.run_batch(L, R, cfg, unchecked_cell=True)
    ctx.synth_resident(n, c["width"], c["height"], c["n_planes"], c["max_disparity"],
                       c["ground"], c["sigma"], seed=55)
    assert ctx.run_resident(cfg, unchecked_cell=True) == 0
    out = {k: np.zeros_like(ref[k]) for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]}
    lib = ps._native.load()
    import ctypes as C

    st = np.zeros(n, np.int32)
    ps._check(lib.ps_download_batch(ctx._h, *[C.c_void_p(out[k].ctypes.data) for k in
                                               ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]],
                                    None, C.c_void_p(st.ctypes.data)))
    for k in out:
        assert np.array_equal(out[k].view(np.uint8), ref[k].view(np.uint8)), k


def _cases():
    z = np.load(GOLDEN)
    for name in json.loads(str(z["cases"])):
        yield name, {k[len(name) + 1:]: z[k] for k in z.files if k.startswith(name + "_")}


def test_render_scene_equals_reference(ctx):
    for name, c in _cases():
        w, h, seed = (int(x) for x in c["geom"])
        regions = [tuple(b) + tuple(p) for b, p in zip(c["box"].tolist(), c["plane"].tolist())]
        st = int(c["status"])
        if st != 0:
            with pytest.raises(ps.Error) as e:
                ctx.render_scene(w, h, regions, float(c["maxd"]), seed)
            assert ps._STATUS[st] is type(e.value), name
            if st == 14:
                assert "outside [0, 16.000000)" in str(e.value) and "plane value" in str(e.value)
            continue
        out = ctx.render_scene(w, h, regions, float(c["maxd"]), seed)
        for k in ["left", "right", "gt_valid", "occluded"]:
            assert np.array_equal(out[k], c[k]), (name, k)
        assert np.array_equal(out["gt"].view(np.uint32), c["gt"].view(np.uint32)), name


def test_rendered_scene_through_the_pipeline(ctx, orc):
    """A device-rendered scene is a valid pipeline input (the reference's
    flat-shift scene): run it and compare with the restatement."""
    out = ctx.render_scene(160, 120, [(0, 0, 160, 120, 0.0, 0.0, 20.0)], 128.0, 1234)
    cfg = ps.PipelineConfig()
    got = ctx.run(out["left"], out["right"], cfg)
    want = orc.run(out["left"], out["right"], cfg)
    for k in ["disparity_valid", "disparity", "costs"]:
        assert np.array_equal(np.asarray(getattr(got, k)).view(np.uint8), want[k].view(np.uint8)), k
