"""Ad-hoc GPU parity probe: CUDA pipeline vs oracle on a few BASELINE shapes (prints diffs)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1511_00758_b200 as ps
import oracle

orc = oracle.load_oracle()

def cmp(tag, got, want, gsup=None):
    d = dict(
        cost_bits=int(np.sum(got["costs"].view(np.uint32) != want["costs"].view(np.uint32))),
        valid=int(np.sum(got["disparity_valid"] != want["disparity_valid"])),
        dmax=float(np.max(np.abs(got["disparity"] - want["disparity"]))),
        dbits=int(np.sum(got["disparity"].view(np.uint32) != want["disparity"].view(np.uint32))),
        dense=float(np.max(np.abs(got["dense"] - want["dense"]))),
        dense_valid=int(np.sum(got["dense_valid"] != want["dense_valid"])),
    )
    print(tag, d, flush=True)
    return d

with ps.Context(0) as ctx:
    for idx, seeds in [(0, [1, 2, 3]), (1, [1]), (2, [5])]:
        c = ps.BASELINE_CONFIGS[idx]
        cfg = ps.baseline_config(idx)
        for s in seeds:
            L, R = ps.synth_pair(c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"], c["sigma"], seed=s)
            t = time.time(); r = ctx.run(L, R, cfg, unchecked_cell=True); tg = time.time() - t
            t = time.time(); w = orc.run(L, R, cfg); to = time.time() - t
            got = dict(costs=r.costs, disparity_valid=r.disparity_valid, disparity=r.disparity, dense=r.dense, dense_valid=r.dense_valid)
            cmp(f"cfg{idx} seed{s} gpu {tg*1e3:.1f}ms orc {to*1e3:.1f}ms", got, w)
            u, v, d = ctx.supports(0)
            wu, wv, wd = w["supports"]
            print("  supports", len(u), len(wu), np.array_equal(u, wu) and np.array_equal(v, wv) and np.array_equal(d, wd))
            print("  trace gpu", [(t.supportCount, t.triangleCount, t.meanCost, t.validCount) for t in r.trace])
            print("  trace orc", [(t['supportCount'], t['triangleCount'], t['meanCost'], t['validCount']) for t in w['trace']])
    # batch
    c = ps.BASELINE_CONFIGS[2]; cfg = ps.baseline_config(2)
    L, R = ps.synth_batch(32, 640, 480, 12, 64, False, 2.0, seed=100)
    t = time.time(); res = ctx.run_batch(L, R, cfg, unchecked_cell=True); print("batch32 first", time.time() - t)
    t = time.time(); res = ctx.run_batch(L, R, cfg, unchecked_cell=True); print("batch32 second", time.time() - t)
    bad = 0
    for f in [0, 7, 31]:
        w = orc.run(L[f], R[f], cfg)
        got = {k: res[k][f] for k in ["costs", "disparity_valid", "disparity", "dense", "dense_valid"]}
        d = cmp(f"batch f{f}", got, w)
    ctx.set_profiling(True)
    res = ctx.run_batch(L, R, cfg, unchecked_cell=True)
    for k, v in ctx.kernel_stats().items():
        gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else 0
        print(f"  {k:16s} launches={v['launches']:4d} ms={v['ms']:.3f} GB/s={gbs:.0f}")
