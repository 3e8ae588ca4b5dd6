"""Small pipeline batches for compute-sanitizer (racecheck / synccheck / memcheck / initcheck)
or for the bounds-checked build (PS_LIB_PATH=.../libplanestereo_b200_checked.so).

Runs every device stage of the pipeline (K1 front end, K2 corners + sort, K3
match + compaction, the device mesh of kernels/star.cu, the raster, K7 bulk
refine in both variants, K8 resampling) plus the stage API's separate kernels
on small frames, and checks the result against the C restatement so a
sanitizer-perturbed schedule that changes the output also fails.  This stands
in for the reference's threaded-equals-sequential guard
(proj/tests/test_pipeline.cpp:75-84,282-291).

  compute-sanitizer --tool racecheck --error-exitcode 9 python tests/tools/sanitize_run.py [small|tiny]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import oracle
import paper_1511_00758_b200 as ps


def main(mode: str) -> int:
    if mode == "tiny":
        shapes = [(64, 48, 1, 16, 4, 2)]
    elif mode == "baseline":
        # BASELINE config 2 geometry (VGA, ND 64, grid 10, 3 iterations), a
        # 70-frame batch (two frame groups), and cfg1's KITTI shape
        shapes = [(640, 480, 70, 64, 10, 3), (1242, 375, 3, 128, 8, 4)]
    else:
        # (W, H, frames, ND, cell, iterations): a multi-group batch is not
        # needed for the kernels' own races; 8 frames exercise the grid loops
        shapes = [(160, 120, 8, 32, 8, 3), (97, 61, 3, 24, 5, 4)]
    orc = oracle.load_oracle()
    bad = 0
    with ps.Context(0) as ctx:
        for (w, h, n, nd, cell, iters) in shapes:
            L, R = ps.synth_batch(n, w, h, 6, nd, False, 2.0, seed=w * 31 + h)
            cfg = ps.PipelineConfig(iterations=iters, maxDisparity=nd, occupancyCellSize=cell)
            res = ctx.run_batch(L, R, cfg, unchecked_cell=True)
            for f in range(n):
                want = orc.run(L[f], R[f], cfg)
                if not (np.array_equal(res["costs"][f].view(np.uint32), want["costs"].view(np.uint32))
                        and np.array_equal(res["disparity_valid"][f], want["disparity_valid"])):
                    bad += 1
            # stage API kernels (census, cost evaluation, interpolation, WTA)
            cen = ctx.census(L[0])
            assert np.array_equal(cen, orc.census(L[0]))
            m, _ = orc.gradient_mask(L[0], cfg.gradientThreshold)
            wta = ctx.wta_oracle(L[0], R[0], m, nd)
            assert np.array_equal(wta[1], orc.wta(L[0], R[0], m, nd)[1])
            print(f"{w}x{h} x{n}, {iters} it.: {n} frames, mismatches so far {bad}", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1] if len(sys.argv) > 1 else "small"))
