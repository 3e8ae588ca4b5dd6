"""Group milestones of three pipelined passes of the cfg2 batch (engine
PS_DEBUG_TIMELINE output on stderr).

  PS_DEBUG_TIMELINE=1 python scripts/timeline.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1511_00758_b200 as ps  # noqa: E402

c = ps.BASELINE_CONFIGS[2]
cfg = ps.baseline_config(2)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 256
L, R = ps.synth_batch(frames, c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                      c["sigma"], seed=5)
ctx = ps.Context(0)
ctx.upload(L, R)
for i in range(3):
    print("run", i, file=sys.stderr, flush=True)
    ctx.run_resident(cfg, unchecked_cell=True)
ctx.close()
