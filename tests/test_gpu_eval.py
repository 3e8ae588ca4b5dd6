"""On-device accuracy (accuracy.cu, proj/src/eval.cpp:19-70) against the C
restatement (pinned to the compiled reference in tests/test_oracle.py): the
counts, the fractions and the sequential binary64 meanAbsError, bit for bit."""
import numpy as np
import pytest

import paper_1511_00758_b200 as ps
from conftest import load_golden

pytestmark = pytest.mark.gpu

TH = [0.25, 0.5, 1.0, 2.0, 3.0, 5.0]


def maps(rng, h, w):
    p = rng.uniform(0, 60, (h, w)).astype(np.float32)
    pv = (rng.random((h, w)) < 0.8).astype(np.uint8)
    g = (p + rng.normal(0, 2, (h, w))).astype(np.float32)
    gv = (rng.random((h, w)) < 0.8).astype(np.uint8)
    return p, pv, g, gv


def test_accuracy_equals_oracle(ctx, orc):
    rng = np.random.default_rng(3)
    for h, w in [(48, 64), (37, 91), (480, 640)]:
        p, pv, g, gv = maps(rng, h, w)
        m = (rng.random((h, w)) < 0.6).astype(np.uint8)
        for mm in (None, m):
            fr, ev, mae = ctx.accuracy(p, pv, g, gv, mm, TH)
            st, ofr, oev, omae = orc.accuracy(p, pv, g, gv, mm, TH)
            assert st == 0 and ev == oev and np.array_equal(fr, ofr)
            assert mae == omae  # the reference's row-major sum, not a reassociated one


def test_accuracy_batch_and_no_overlap(ctx, orc):
    rng = np.random.default_rng(4)
    P, PV, G, GV = zip(*[maps(rng, 60, 80) for _ in range(5)])
    P, PV, G, GV = map(np.stack, (P, PV, G, GV))
    fr, ev, mae = ctx.accuracy(P, PV, G, GV, None, TH)
    for f in range(5):
        st, ofr, oev, omae = orc.accuracy(P[f], PV[f], G[f], GV[f], None, TH)
        assert ev[f] == oev and np.array_equal(fr[f], ofr) and mae[f] == omae
    PV[2] = 0
    with pytest.raises(ps.NoOverlap):
        ctx.accuracy(P, PV, G, GV, None, TH)


def test_accuracy_of_pipeline_results(ctx, orc):
    """Rendered flat scene with ground truth (golden fixture of the reference):
    the pipeline result's accuracy over the gradient mask, host-side and
    device-resident, equals the restatement's on the same maps."""
    gl = load_golden("pipe_render_flat20_160x120.npz")
    cfg = ps.PipelineConfig()
    L, R = gl["left"], gl["right"]
    res = ctx.run_batch(L[None], R[None], cfg)
    m, _ = orc.gradient_mask(L, cfg.gradientThreshold)
    st, ofr, oev, omae = orc.accuracy(res["disparity"][0], res["disparity_valid"][0], gl["gt"],
                                      gl["gt_valid"], m, TH)
    assert st == 0
    fr, ev, mae = ctx.download_accuracy(gl["gt"][None], gl["gt_valid"][None], True, TH)
    assert ev[0] == oev and np.array_equal(fr[0], ofr) and mae[0] == omae
    fr1, ev1, mae1 = ctx.accuracy(res["disparity"][0], res["disparity_valid"][0], gl["gt"],
                                  gl["gt_valid"], m, TH)
    assert ev1 == oev and np.array_equal(fr1, ofr) and mae1 == omae
    # the golden result (the reference's own run) scores identically
    st, gfr, gev, gmae = orc.accuracy(gl["disparity"], gl["disparity_valid"], gl["gt"],
                                      gl["gt_valid"], m, TH)
    assert gev == ev1 and np.array_equal(gfr, fr1) and gmae == mae1
