"""C-ABI boundary tests that need no GPU: the library loads, exports exactly what
include/planestereo_c.h declares, validates configs like
PipelineConfig::validate, and the synthetic generator is deterministic."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1511_00758_b200 as ps
from paper_1511_00758_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "planestereo_c.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)) - {"ps_observer_fn"})


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ps_[a-z0-9_]+)", out))
    for name in declared_symbols():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_struct_layouts_match_reference():
    # PipelineConfig is 11 x 4 B (config.hpp:8-34); IterationStats 40 B (pipeline.hpp:50-58)
    assert C.sizeof(_native.PsConfig) == 44
    assert C.sizeof(_native.PsIterStats) == 40


def test_config_defaults_and_validation():
    c = _native.PsConfig()
    _native.load().ps_config_default(C.byref(c))
    d = ps.PipelineConfig()
    assert (c.iterations, c.max_disparity, c.occupancy_cell_size, c.per_bin_cap) == (
        d.iterations, d.maxDisparity, d.occupancyCellSize, d.perBinCap)
    d.validate()
    # proj/tests/test_core.cpp:188-207
    for bad in [dict(iterations=0), dict(costLow=0.6), dict(occupancyCellSize=24),
                dict(maxDisparity=0), dict(perBinCap=0), dict(threads=0),
                dict(sparseAcceptCost=0.0), dict(uniquenessRatio=1.5), dict(costHigh=1.5),
                dict(gradientThreshold=-1), dict(cornerThreshold=-1)]:
        with pytest.raises(ps.InvalidConfig):
            ps.PipelineConfig(**bad).validate()
    # BASELINE grids 10 / 6 need the explicit opt-in
    with pytest.raises(ps.InvalidConfig):
        ps.PipelineConfig(occupancyCellSize=10).validate()
    ps.PipelineConfig(occupancyCellSize=10).validate(unchecked_cell=True)
    with pytest.raises(ps.InvalidConfig):
        ps.PipelineConfig(occupancyCellSize=0).validate(unchecked_cell=True)


def test_context_without_device_fails_loudly():
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises((ps.NoDevice, ps.CudaError)):
        ps.Context(0)


def test_synth_is_deterministic_and_shaped():
    a = ps.synth_pair(128, 96, 8, 48, True, 2.0, seed=5, with_gt=True)
    b = ps.synth_pair(128, 96, 8, 48, True, 2.0, seed=5, with_gt=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    L, R, gt = a
    assert gt.min() >= 0 and gt.max() <= 47
    c = ps.synth_pair(128, 96, 8, 48, True, 2.0, seed=6)
    assert not np.array_equal(L, c[0])
    bl, br = ps.synth_batch(3, 128, 96, 8, 48, True, 2.0, seed=5, threads=2)
    assert np.array_equal(bl[0], L) and np.array_equal(br[0], R)
    assert np.array_equal(bl[1], c[0])


def test_synth_statistics_match_survey(orc):
    """M/P ~ 0.85 and a saturated corner cap at VGA (SURVEY 8(d) expectations)."""
    L, R = ps.synth_pair(640, 480, 12, 64, False, 2.0, seed=1)
    _, m = orc.gradient_mask(L, 20)
    assert 0.80 < m / (640 * 480) < 0.90
    u, v, s = orc.detect_candidates(L, ps.PipelineConfig())
    assert len(u) == 600
