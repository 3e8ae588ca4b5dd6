"""Per-stage device/host times of one pipelined pass (the engine's CUDA-event
profiling), for the BASELINE cfg2 batch and for a single 32-frame group.

  python scripts/kernel_profile.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1511_00758_b200 as ps  # noqa: E402


def show(stats, keys=None):
    for k, v in stats.items():
        if keys and not any(k.startswith(x) for x in keys):
            continue
        gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 and v["bytes"] > 0 else 0
        print(f"{k:16s} launches {v['launches']:4d}  ms {v['ms']:8.3f}  "
              f"ms/launch {v['ms'] / max(1, v['launches']):7.4f}  GB/s {gbs:8.1f}")


def main():
    c = ps.BASELINE_CONFIGS[2]
    cfg = ps.baseline_config(2)
    L, R = ps.synth_batch(256, c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                          c["sigma"], seed=5)
    ctx = ps.Context(0)
    ctx.upload(L, R)
    ctx.run_resident(cfg, unchecked_cell=True)
    ctx.set_profiling(True)
    ctx.reset_kernel_stats()
    ctx.run_resident(cfg, unchecked_cell=True)
    print("---- 256 frames, 8 groups (pipelined)")
    show(ctx.kernel_stats())
    ctx.set_max_groups(1)
    ctx.upload(L[:32].copy(), R[:32].copy())
    ctx.run_resident(cfg, unchecked_cell=True)
    ctx.reset_kernel_stats()
    ctx.run_resident(cfg, unchecked_cell=True)
    print("---- 32 frames, one group")
    show(ctx.kernel_stats(), ["mesh", "refine", "h2d"])
    ctx.close()


if __name__ == "__main__":
    main()
