"""Probe of the device mesh (kernels/star.cu): one batch of BASELINE config 2
frames through ps_run_batch, for ncu captures of k_star / k_tri_check."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1511_00758_b200 as ps  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
c = ps.BASELINE_CONFIGS[2]
cfg = ps.baseline_config(2)
L, R = ps.synth_batch(n, c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                      c["sigma"], seed=1000)
with ps.Context(0) as ctx:
    ctx.set_max_groups(1)
    ctx.set_profiling(True)
    for _ in range(2):
        ctx.reset_kernel_stats()
        t0 = time.perf_counter()
        ctx.run_batch(L, R, cfg, unchecked_cell=True)
        dt = time.perf_counter() - t0
    print(f"{n} frames: {dt * 1e3:.1f} ms")
    for k, v in ctx.kernel_stats().items():
        print(f"  {k}: {v['launches']} launches, {v['ms']:.3f} ms")
