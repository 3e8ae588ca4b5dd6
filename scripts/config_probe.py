"""Probe one BASELINE config: a batch through ps_run_batch with engine profiling,
printing the wall time and the host-mesh statistics (replays by cause, order
queries, rotations).  `python scripts/config_probe.py CONFIG FRAMES [REPEATS]`"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1511_00758_b200 as ps  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = ps.BASELINE_CONFIGS[k]
cfg = ps.baseline_config(k)
L, R = ps.synth_batch(n, c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                      c["sigma"], seed=4000 + k)
with ps.Context(0) as ctx:
    ctx.set_profiling(True)
    for r in range(reps):
        ctx.reset_kernel_stats()
        t0 = time.perf_counter()
        res = ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False)
        dt = time.perf_counter() - t0
        print(f"cfg{k} {n} frames: {dt * 1e3:.1f} ms ({n / dt:.3f} frames/s), status {list(res['status'])}",
              flush=True)
    for name, v in ctx.kernel_stats().items():
        if v["launches"] or v["ms"]:
            print(f"  {name}: {v['launches']} launches, {v['ms']:.3f} ms")
