"""ctypes binding of the C ABI (include/planestereo_c.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``paper_1511_00758_b200/libplanestereo_b200.so``).  There is no fallback: if
the library is missing or no sm_100 device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PS_LIB_PATH: an instrumented build of the same sources (profiling probes)
LIB_PATH = os.environ.get("PS_LIB_PATH") or os.path.join(_HERE, "libplanestereo_b200.so")


class PsConfig(C.Structure):
    """Field-for-field planestereo::PipelineConfig (proj/include/planestereo/config.hpp:8-34)."""

    _fields_ = [
        ("iterations", C.c_int),
        ("max_disparity", C.c_int),
        ("cost_low", C.c_float),
        ("cost_high", C.c_float),
        ("gradient_threshold", C.c_int),
        ("occupancy_cell_size", C.c_int),
        ("corner_threshold", C.c_int),
        ("per_bin_cap", C.c_int),
        ("sparse_accept_cost", C.c_float),
        ("uniqueness_ratio", C.c_float),
        ("threads", C.c_int),
    ]


class PsIterStats(C.Structure):
    """planestereo::IterationStats (proj/include/planestereo/pipeline.hpp:50-58)."""

    _fields_ = [
        ("iteration", C.c_int),
        ("support_count", C.c_int),
        ("triangle_count", C.c_int),
        ("occupancy_cell_size", C.c_int),
        ("mean_cost", C.c_double),
        ("valid_count", C.c_int),
        ("millis", C.c_double),
    ]


class PsKernelStat(C.Structure):
    _fields_ = [
        ("name", C.c_char * 32),
        ("launches", C.c_int),
        ("total_ms", C.c_double),
        ("algorithmic_bytes", C.c_double),
    ]


class PsSynthParams(C.Structure):
    _fields_ = [
        ("width", C.c_int),
        ("height", C.c_int),
        ("n_planes", C.c_int),
        ("max_disparity", C.c_int),
        ("ground", C.c_int),
        ("noise_sigma", C.c_float),
        ("seed", C.c_uint32),
    ]


class PsCell(C.Structure):
    _fields_ = [
        ("u", C.c_int),
        ("v", C.c_int),
        ("disparity", C.c_float),
        ("cost", C.c_float),
        ("occupied", C.c_int),
    ]


class PsSceneRegion(C.Structure):
    """SceneRegion (proj/include/planestereo/synth.hpp:13-20)."""

    _fields_ = [("u0", C.c_int), ("v0", C.c_int), ("u1", C.c_int), ("v1", C.c_int),
                ("a", C.c_double), ("b", C.c_double), ("c", C.c_double)]


class PsCalib(C.Structure):
    """CameraCalib (proj/include/planestereo/io.hpp:17-24)."""

    _fields_ = [("focal", C.c_double), ("baseline", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double)]


OBSERVER = C.CFUNCTYPE(None, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                       C.c_void_p)

P = C.c_void_p
I = C.c_int
F = C.c_float

# name -> (restype, argtypes); exactly the symbols include/planestereo_c.h declares.
SIGNATURES = {
    "ps_version": (C.c_char_p, []),
    "ps_ctx_create": (I, [I, P]),
    "ps_ctx_destroy": (None, [P]),
    "ps_last_error": (C.c_char_p, [P]),
    "ps_config_default": (None, [P]),
    "ps_config_validate": (I, [P, C.c_uint]),
    "ps_run": (I, [P, P, P, I, I, P, C.c_uint, P, P, P, P, P, P, OBSERVER, P]),
    "ps_run_batch": (I, [P, I, P, P, I, I, P, C.c_uint, P, P, P, P, P, P, P]),
    "ps_run_batch_multi": (I, [P, I, I, P, P, I, I, P, C.c_uint, P, P, P, P, P, P, P]),
    "ps_upload_batch": (I, [P, I, P, P, I, I]),
    "ps_run_resident": (I, [P, P, C.c_uint]),
    "ps_download_batch": (I, [P, P, P, P, P, P, P, P]),
    "ps_get_supports": (I, [P, I, P, P, P, I, P]),
    "ps_set_profiling": (I, [P, I]),
    "ps_set_max_groups": (I, [P, I]),
    "ps_get_host_threads": (I, [P, P]),
    "ps_reset_kernel_stats": (I, [P]),
    "ps_get_kernel_stats": (I, [P, P, I, P]),
    "ps_launch_count": (C.c_longlong, [P]),
    "ps_ctx_stream": (C.c_void_p, [P]),
    "ps_gradient_mask": (I, [P, P, I, I, I, P, P]),
    "ps_census": (I, [P, P, I, I, P]),
    "ps_detect_candidates": (I, [P, P, I, I, P, P, P, P, I, P]),
    "ps_match_epipolar": (I, [P, P, P, I, I, P, P, I, P, P, P, P, I, P]),
    "ps_delaunay": (I, [P, P, I, P, I, P]),
    "ps_delaunay_fast": (I, [P, P, I, P, I, P]),
    "ps_mesh_build": (I, [P, P, P, P, I, P, I, I, I, P, P]),
    "ps_interpolate": (I, [P, P, P, I, I, I, P, F, P, P]),
    "ps_cost_evaluation": (I, [P, P, P, I, I, P, P, P, P]),
    "ps_refinement": (I, [P, P, P, P, P, P, P, P, I, I, I, P, P, P]),
    "ps_support_resampling": (I, [P, P, P, I, P, P, P, I, P, P, I, I, P, P, P, P, I, P]),
    "ps_wta_oracle": (I, [P, P, P, I, I, P, I, P, P, P]),
    "ps_wta_batch": (I, [P, I, P, P, I, I, I, I, P, P, P]),
    "ps_encode_kitti16": (I, [P, P, P, I, I, I, P]),
    "ps_encode_pfm": (I, [P, P, P, I, I, I, P]),
    "ps_point_cloud": (I, [P, P, P, P, I, I, P, C.c_double, P, P, I, P]),
    "ps_download_kitti16": (I, [P, I, P]),
    "ps_download_pfm": (I, [P, I, P]),
    "ps_download_point_cloud": (I, [P, I, I, P, C.c_double, P, P, I, P]),
    "ps_accuracy": (I, [P, I, P, P, P, P, P, I, I, P, I, P, P, P]),
    "ps_download_accuracy": (I, [P, I, P, P, I, P, I, P, P, P]),
    "ps_synth_pair": (I, [P, P, P, P]),
    "ps_synth_batch": (I, [P, I, I, P, P]),
    "ps_synth_batch_gpu": (I, [P, P, I, P, P, P]),
    "ps_synth_resident": (I, [P, P, I]),
    "ps_render_scene": (I, [P, I, I, F, C.c_uint32, P, I, P, P, P, P, P]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libplanestereo_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc sm_100a) first; "
            "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
