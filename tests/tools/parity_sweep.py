"""GPU vs oracle over many BASELINE-style frames: counts every kind of difference."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1511_00758_b200 as ps
import oracle

orc = oracle.load_oracle()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
summary = {}
with ps.Context(0) as ctx:
    for idx in (2, 0, 1):
        c = ps.BASELINE_CONFIGS[idx]; cfg = ps.baseline_config(idx)
        frames = n if idx != 1 else max(4, n // 8)
        L, R = ps.synth_batch(frames, c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"], c["sigma"], seed=7000 + idx * 1000)
        res = ctx.run_batch(L, R, cfg, unchecked_cell=True)
        bad = dict(frames=frames, cost=0, valid=0, dmax=0.0, sup=0, dense_tie_px=0, dense_other=0)
        for f in range(frames):
            w = orc.run(L[f], R[f], cfg)
            cb = int(np.sum(res["costs"][f].view(np.uint32) != w["costs"].view(np.uint32)))
            vb = int(np.sum(res["disparity_valid"][f] != w["disparity_valid"]))
            bad["cost"] += cb > 0; bad["valid"] += vb > 0
            bad["dmax"] = max(bad["dmax"], float(np.max(np.abs(res["disparity"][f] - w["disparity"]))))
            u, v, d = ctx.supports(f); wu, wv, wd = w["supports"]
            bad["sup"] += not (len(u) == len(wu) and np.array_equal(u, wu) and np.array_equal(v, wv) and np.array_equal(d, wd))
            dd = res["dense_valid"][f] != w["dense_valid"]
            tiny = (np.abs(res["dense"][f]) <= 1e-9) & (np.abs(w["dense"]) <= 1e-9)
            bad["dense_tie_px"] += int(np.sum(dd & tiny)); bad["dense_other"] += int(np.sum(dd & ~tiny))
        print(f"cfg{idx}", bad, flush=True)
