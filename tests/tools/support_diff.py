"""Find frames whose final support list differs between GPU and oracle; print details."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1511_00758_b200 as ps
import oracle
orc = oracle.load_oracle()
c = ps.BASELINE_CONFIGS[2]; cfg = ps.baseline_config(2)
n = 48
L, R = ps.synth_batch(n, 640, 480, 12, 64, False, 2.0, seed=7000 + 2 * 1000)
with ps.Context(0) as ctx:
    res = ctx.run_batch(L, R, cfg, unchecked_cell=True)
    for f in range(n):
        u, v, d = ctx.supports(f)
        w = orc.run(L[f], R[f], cfg)
        wu, wv, wd = w["supports"]
        if len(u) == len(wu) and np.array_equal(u, wu) and np.array_equal(v, wv) and np.array_equal(d, wd):
            continue
        print("frame", f, "len", len(u), len(wu), "trace gpu", [t.supportCount for t in res["trace"][f]], "orc", [t["supportCount"] for t in w["trace"]])
        m = min(len(u), len(wu))
        bad = np.nonzero((u[:m] != wu[:m]) | (v[:m] != wv[:m]) | (d[:m] != wd[:m]))[0]
        print("  first diffs", bad[:10])
        for i in bad[:5]:
            print("   ", i, (u[i], v[i], repr(d[i])), (wu[i], wv[i], repr(wd[i])))
