"""BASELINE configs 3 (1920x1080, 4 iterations) and 4 (3840x2160, 6
iterations) at their full iteration counts, bit for bit against digests of the
compiled reference's own outputs (tests/golden/digests_large.json, written by
tests/golden/gen_digests.py from oracle/_ref: the unmodified reference sources
driven by the staged run() loop, proj/src/pipeline.cpp:131-203).

The cfg4 schedule 6 -> 3 -> 1 -> 1 -> 1 -> 1 reaches s = 1 on a 4K frame, where
~28% of the triangles lie in cocircular cells and the mesh
holds ~5.6 M supports: the hardest case for the triangle-set tie rule, the
reference sweep's rotations and the hull-vertex pins.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1511_00758_b200 as ps

HERE = os.path.dirname(os.path.abspath(__file__))
DIGESTS = os.path.join(HERE, "golden", "digests_large.json")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_digest(trace) -> str:
    rows = [(t.iteration, t.supportCount, t.triangleCount, t.occupancyCellSize,
             float(t.meanCost).hex(), t.validCount) for t in trace]
    return hashlib.sha256(json.dumps(rows).encode()).hexdigest()


def cases():
    with open(DIGESTS) as f:
        db = json.load(f)
    return [pytest.param(db[k], id=k) for k in sorted(db)]


@pytest.mark.gpu
@pytest.mark.parametrize("rec", cases())
def test_large_config_digests(ctx, rec):
    L, R = ps.synth_pair(rec["width"], rec["height"], rec["planes"], rec["max_disparity"],
                         rec["ground"], rec["sigma"], seed=rec["seed"])
    assert sha(L) == rec["left"] and sha(R) == rec["right"], "inputs differ from the digested ones"
    cfg = ps.PipelineConfig(iterations=rec["iterations"], maxDisparity=rec["max_disparity"],
                            occupancyCellSize=rec["cell"])
    r = ctx.run(L, R, cfg, unchecked_cell=True)
    u, v, d = ctx.supports(0)
    rows = [dict(supportCount=t.supportCount, triangleCount=t.triangleCount,
                 occupancyCellSize=t.occupancyCellSize, meanCost=float(t.meanCost).hex(),
                 validCount=t.validCount) for t in r.trace]
    assert rows == rec["trace_rows"]
    assert len(u) == rec["support_count"]
    sup = np.concatenate([u.astype(np.int32).view(np.uint8), v.astype(np.int32).view(np.uint8),
                          d.astype(np.float64).view(np.uint8)])
    assert sha(sup) == rec["supports"], "support list"
    for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
        assert sha(getattr(r, k)) == rec[k], k
    assert trace_digest(r.trace) == rec["trace"]
