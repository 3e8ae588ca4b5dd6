"""Randomised parity sweep: N random frame sizes and configurations through
the GPU pipeline (batched, several frames per run) against the C restatement,
bit for bit on every output map, the support list and the trace.

  python tests/tools/fuzz_parity.py [N] [seed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import paper_1511_00758_b200 as ps  # noqa: E402
from oracle import load_oracle  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    orc = load_oracle()
    ctx = ps.Context(0)
    bad = 0
    checked = 0
    for trial in range(n):
        w, h = int(rng.integers(32, 400)), int(rng.integers(24, 300))
        frames = int(rng.integers(1, 5))
        nd = int(rng.integers(4, 160))
        low = float(rng.choice([0.1, 0.15, 0.2, 0.25, 0.3]))
        cfg = ps.PipelineConfig(iterations=int(rng.integers(1, 7)), maxDisparity=nd,
                                occupancyCellSize=int(rng.integers(1, 24)), costLow=low,
                                costHigh=float(low + rng.choice([0.05, 0.1, 0.2, 0.3, 0.45])),
                                gradientThreshold=int(rng.integers(0, 50)),
                                cornerThreshold=int(rng.integers(3, 40)),
                                perBinCap=int(rng.integers(1, 20)),
                                sparseAcceptCost=float(rng.choice([0.15, 0.2, 0.25, 0.4, 0.6])),
                                uniquenessRatio=float(rng.choice([0.5, 0.7, 0.8, 0.9, 1.0])))
        L, R = ps.synth_batch(frames, w, h, int(rng.integers(0, 16)), max(1, nd - 1),
                              bool(rng.integers(0, 2)), float(rng.choice([0.0, 1.0, 2.0, 4.0])),
                              seed=int(rng.integers(0, 1 << 30)))
        res = ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False)
        for f in range(frames):
            want = orc.run(L[f], R[f], cfg)
            checked += 1
            if want["status"] != 0:
                if res["status"][f] != want["status"]:
                    bad += 1
                    print("status mismatch", trial, f, res["status"][f], want["status"])
                continue
            ok = res["status"][f] == 0
            for k in ["disparity", "disparity_valid", "costs", "dense", "dense_valid"]:
                ok = ok and np.array_equal(bits(res[k][f]), bits(want[k]))
            ok = ok and [t.meanCost for t in res["trace"][f]] == [t["meanCost"] for t in want["trace"]]
            if not ok:
                bad += 1
                print("MISMATCH trial", trial, "frame", f, w, h, cfg)
    print(f"fuzz: {checked} frames, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
