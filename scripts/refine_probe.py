"""Isolated-pass probe for ncu: one warm pass, then one pass with the frame
groups serialised (set_max_groups(1)), over BASELINE config 2 (256 VGA frames).
Prints the per-kernel CUDA-event times of the second pass.

  ncu --set full -k regex:k_refine_bulk -s 3 -c 3 python scripts/refine_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1511_00758_b200 as ps  # noqa: E402

cfgd = ps.BASELINE_CONFIGS[2]
cfg = ps.baseline_config(2)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else cfgd["frames"]
H, W = cfgd["height"], cfgd["width"]
L = np.empty((frames, H, W), np.uint8)
R = np.empty((frames, H, W), np.uint8)
ps.synth_batch(frames, W, H, cfgd["n_planes"], cfgd["max_disparity"], cfgd["ground"], cfgd["sigma"],
               seed=0, threads=os.cpu_count() or 8, left=L, right=R)
ctx = ps.Context(0)
ctx.upload_ptr(frames, L.ctypes.data, R.ctypes.data, W, H)
ctx.set_max_groups(1)
ctx.run_resident(cfg, unchecked_cell=True)
ctx.set_profiling(True)
ctx.reset_kernel_stats()
ctx.run_resident(cfg, unchecked_cell=True)
for name, k in ctx.kernel_stats().items():
    print(f"{name:16s} launches {k['launches']:4d}  ms {k['ms']:8.3f}")
