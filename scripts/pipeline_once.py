"""One warm 256-frame BASELINE config 2 batch through run_resident with the
default frame groups (for ncu launch lists of the pipeline as it runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1511_00758_b200 as ps  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = ps.BASELINE_CONFIGS[2]
cfg = ps.baseline_config(2)
L, R = ps.synth_batch(n, c["width"], c["height"], c["n_planes"], c["max_disparity"], c["ground"],
                      c["sigma"], seed=5)
with ps.Context(0) as ctx:
    ctx.upload(L, R)
    for _ in range(runs):
        ctx.run_resident(cfg, unchecked_cell=True)
print("ok")
