"""The bounds-checked build (libplanestereo_b200_checked.so: kernels/common.cuh
PS_CHECK on the stage buffers of K7, the raster's pixel writes, the support
and re-match compactions, the device mesh's grid and triangle emission) over
every device stage, each run checked bit for bit against the C restatement.

compute-sanitizer is not allowed on this GPU pool; a failing
check prints its site and traps, so the run would fail here.  This stands in
for the reference's threaded == sequential guard
(proj/tests/test_pipeline.cpp:75-84,282-291) together with
test_gpu_pipeline.py::test_concurrent_batches_agree.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1511_00758_b200", "libplanestereo_b200_checked.so")
SCRIPT = os.path.join(ROOT, "tests", "tools", "sanitize_run.py")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["small", "baseline"])
def test_checked_build(mode):
    if not os.path.exists(LIB):
        pytest.fail("checked build missing: run __graft_entry__.build()")
    env = dict(os.environ, PS_LIB_PATH=LIB)
    r = subprocess.run([sys.executable, SCRIPT, mode], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    out = r.stdout + r.stderr
    assert "PS_CHECK failed" not in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
