"""paper_1511_00758_b200 — B200-native hot path of the iterative piecewise-planar
stereo method of arXiv 1511.00758 (reference: ``planestereo``, /root/reference/proj).

Python host mirror of the reference's C++ API, over the C ABI of
``libplanestereo_b200.so`` (sm_100a kernels + C++ engine):

    PipelineConfig        planestereo::PipelineConfig   (config.hpp:8-34)
    Context.run           planestereo::run              (pipeline.cpp:131-203)
    Context.run_batch     batched run over many frames on one GPU
    Context.<stage>       the public stage functions (gradientMask, censusTransform,
                          detectCandidates, matchEpipolar, mesh, interpolate,
                          costEvaluation)
    delaunay_triangulate  planestereo::delaunayTriangulate (delaunay.cpp:288-325)

Errors are raised as the Python mirror of the reference's exception classes
(error.hpp:9-72).  Nothing here falls back to a CPU implementation.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from typing import Callable, List, Optional

import numpy as np

from . import _native
from ._native import PsConfig, PsIterStats

PS_RUN_UNCHECKED_CELL = 0x1


# ---------------------------------------------------------------- errors (error.hpp)
class Error(RuntimeError):
    """planestereo::Error"""


class InvalidConfig(Error):
    pass


class DimensionTooSmall(Error):
    pass


class DimensionMismatch(Error):
    pass


class FewerThanThreePoints(Error):
    pass


class DegenerateTriangle(Error):
    pass


class SeedingFailed(Error):
    pass


class NegativeDisparity(Error):
    pass


class EmptyCloud(Error):
    pass


class NoOverlap(Error):
    pass


class InvalidPlane(Error):
    pass


class CudaError(Error):
    pass


class NoDevice(Error):
    pass


_STATUS = {
    1: Error, 2: InvalidConfig, 3: DimensionTooSmall, 4: DimensionMismatch,
    5: FewerThanThreePoints, 6: DegenerateTriangle, 7: SeedingFailed, 8: CudaError,
    9: NoDevice, 10: Error, 11: NegativeDisparity, 12: EmptyCloud, 13: NoOverlap,
    14: InvalidPlane,
}


def _maps(disparity, valid):
    d = np.ascontiguousarray(disparity, dtype=np.float32)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    if d.shape != v.shape or d.ndim < 2:
        raise DimensionMismatch("disparity and validity must be equal arrays of >= 2 dims")
    return d, v


def _check(status: int) -> None:
    if status != 0:
        msg = _native.load().ps_last_error(None)
        raise _STATUS.get(status, Error)(msg.decode() if msg else f"status {status}")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- config
@dataclass
class PipelineConfig:
    """planestereo::PipelineConfig, same field names and defaults (config.hpp:10-30)."""

    iterations: int = 1
    maxDisparity: int = 128
    costLow: float = 0.25
    costHigh: float = 0.5
    gradientThreshold: int = 20
    occupancyCellSize: int = 32
    cornerThreshold: int = 20
    perBinCap: int = 5
    sparseAcceptCost: float = 0.25
    uniquenessRatio: float = 0.9
    threads: int = 1

    def to_c(self) -> PsConfig:
        return PsConfig(self.iterations, self.maxDisparity, self.costLow, self.costHigh,
                        self.gradientThreshold, self.occupancyCellSize, self.cornerThreshold,
                        self.perBinCap, self.sparseAcceptCost, self.uniquenessRatio, self.threads)

    def validate(self, unchecked_cell: bool = False) -> None:
        """PipelineConfig::validate (config.cpp:17-49); raises InvalidConfig."""
        c = self.to_c()
        _check(_native.load().ps_config_validate(C.byref(c), PS_RUN_UNCHECKED_CELL if unchecked_cell else 0))


@dataclass
class IterationStats:
    iteration: int
    supportCount: int
    triangleCount: int
    occupancyCellSize: int
    meanCost: float
    validCount: int
    millis: float


@dataclass
class StereoResult:
    """planestereo::StereoResult (pipeline.hpp:62-67) as numpy arrays (H x W)."""

    disparity: np.ndarray
    disparity_valid: np.ndarray
    costs: np.ndarray
    dense: np.ndarray
    dense_valid: np.ndarray
    trace: List[IterationStats] = field(default_factory=list)


def _stats(s: PsIterStats) -> IterationStats:
    return IterationStats(s.iteration, s.support_count, s.triangle_count, s.occupancy_cell_size,
                          s.mean_cost, s.valid_count, s.millis)


def _u8(img) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 2:
        raise DimensionMismatch("expected a 2-D uint8 image")
    return a


class Context:
    """One GPU context (ps_ctx): device memory, a stream, host worker pool."""

    def __init__(self, device: int = 0):
        self._lib = _native.load()
        h = C.c_void_p()
        _check(self._lib.ps_ctx_create(device, C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.ps_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------ pipeline
    def run(self, left, right, config: PipelineConfig, unchecked_cell: bool = False,
            observer: Optional[Callable] = None) -> StereoResult:
        """planestereo::run.  observer(iteration, final_disparity, final_valid, final_cost)."""
        L, R = _u8(left), _u8(right)
        if L.shape != R.shape:
            config.validate(unchecked_cell)  # InvalidConfig takes precedence (pipeline.cpp:133-136)
            raise DimensionMismatch("stereo pair dimensions differ")
        h, w = L.shape
        cfg = config.to_c()
        out = StereoResult(np.zeros((h, w), np.float32), np.zeros((h, w), np.uint8),
                           np.zeros((h, w), np.float32), np.zeros((h, w), np.float32),
                           np.zeros((h, w), np.uint8))
        trace = (PsIterStats * max(1, config.iterations))()
        cb = _native.OBSERVER(0)
        if observer is not None:
            def _obs(it, fd, fv, fc, ww, hh, user):
                n = ww * hh
                d = np.ctypeslib.as_array((C.c_float * n).from_address(fd)).reshape(hh, ww).copy()
                v = np.ctypeslib.as_array((C.c_uint8 * n).from_address(fv)).reshape(hh, ww).copy()
                c = np.ctypeslib.as_array((C.c_float * n).from_address(fc)).reshape(hh, ww).copy()
                observer(it, d, v, c)
            cb = _native.OBSERVER(_obs)
        flags = PS_RUN_UNCHECKED_CELL if unchecked_cell else 0
        self._shape = (1, h, w)
        _check(self._lib.ps_run(self._h, _ptr(L), _ptr(R), w, h, C.byref(cfg), flags,
                                _ptr(out.disparity), _ptr(out.disparity_valid), _ptr(out.costs),
                                _ptr(out.dense), _ptr(out.dense_valid), trace, cb, None))
        out.trace = [_stats(trace[i]) for i in range(config.iterations)]
        return out

    def run_batch(self, left: np.ndarray, right: np.ndarray, config: PipelineConfig,
                  unchecked_cell: bool = False, raise_on_failure: bool = True,
                  out: Optional[dict] = None) -> dict:
        """Batched run over frames stacked as (F, H, W) uint8 arrays.

        `out` may supply the five output arrays (keys disparity,
        disparity_valid, costs, dense, dense_valid; C-contiguous, right dtype
        and shape); page-locked ones are filled group by group during the run
        (streamed D2H, Engine::set_sink)."""
        L = np.ascontiguousarray(left, dtype=np.uint8)
        R = np.ascontiguousarray(right, dtype=np.uint8)
        if L.ndim != 3 or L.shape != R.shape:
            raise DimensionMismatch("expected two (F, H, W) uint8 stacks of equal shape")
        n, h, w = L.shape
        cfg = config.to_c()
        spec = {"disparity": np.float32, "disparity_valid": np.uint8, "costs": np.float32,
                "dense": np.float32, "dense_valid": np.uint8}
        res = {}
        for key, dt in spec.items():
            a = (out or {}).get(key)
            if a is None:
                a = np.zeros((n, h, w), dt)
            elif a.dtype != dt or a.shape != (n, h, w) or not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"out[{key!r}] must be a C-contiguous {np.dtype(dt).name} array of shape {(n, h, w)}")
            res[key] = a
        res["status"] = np.zeros(n, np.int32)
        self._shape = (n, h, w)
        trace = (PsIterStats * (n * config.iterations))()
        st = self._lib.ps_run_batch(self._h, n, _ptr(L), _ptr(R), w, h, C.byref(cfg),
                                    PS_RUN_UNCHECKED_CELL if unchecked_cell else 0,
                                    _ptr(res["disparity"]), _ptr(res["disparity_valid"]),
                                    _ptr(res["costs"]), _ptr(res["dense"]),
                                    _ptr(res["dense_valid"]), trace, _ptr(res["status"]))
        return _finish_batch(res, st, trace, n, config, raise_on_failure)

    def upload(self, left: np.ndarray, right: np.ndarray) -> None:
        n, h, w = left.shape
        _check(self._lib.ps_upload_batch(self._h, n, _ptr(left), _ptr(right), w, h))
        self._shape = (n, h, w)

    def upload_ptr(self, n: int, left_ptr: int, right_ptr: int, w: int, h: int) -> None:
        _check(self._lib.ps_upload_batch(self._h, n, C.c_void_p(left_ptr), C.c_void_p(right_ptr), w, h))
        self._shape = (n, h, w)

    def run_resident(self, config: PipelineConfig, unchecked_cell: bool = False) -> int:
        cfg = config.to_c()
        return self._lib.ps_run_resident(self._h, C.byref(cfg),
                                         PS_RUN_UNCHECKED_CELL if unchecked_cell else 0)

    def download_ptr(self, disparity=0, disparity_valid=0, costs=0, dense=0, dense_valid=0) -> None:
        p = lambda x: C.c_void_p(x) if x else None
        _check(self._lib.ps_download_batch(self._h, p(disparity), p(disparity_valid), p(costs),
                                           p(dense), p(dense_valid), None, None))

    def supports(self, frame: int = 0):
        n = C.c_int()
        self._lib.ps_get_supports(self._h, frame, None, None, None, 0, C.byref(n))
        u = np.zeros(n.value, np.int32)
        v = np.zeros(n.value, np.int32)
        d = np.zeros(n.value, np.float64)
        _check(self._lib.ps_get_supports(self._h, frame, _ptr(u), _ptr(v), _ptr(d), n.value, C.byref(n)))
        return u, v, d

    def set_profiling(self, on: bool) -> None:
        _check(self._lib.ps_set_profiling(self._h, 1 if on else 0))

    def set_max_groups(self, groups: int) -> None:
        _check(self._lib.ps_set_max_groups(self._h, groups))

    def host_threads(self) -> int:
        n = C.c_int()
        _check(self._lib.ps_get_host_threads(self._h, C.byref(n)))
        return n.value

    def reset_kernel_stats(self) -> None:
        _check(self._lib.ps_reset_kernel_stats(self._h))

    def kernel_stats(self) -> dict:
        arr = (_native.PsKernelStat * 64)()
        n = C.c_int()
        _check(self._lib.ps_get_kernel_stats(self._h, arr, 64, C.byref(n)))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].total_ms,
                                       "bytes": arr[i].algorithmic_bytes}
                for i in range(min(64, n.value))}

    def launch_count(self) -> int:
        return int(self._lib.ps_launch_count(self._h))

    def stream_handle(self) -> int:
        """cudaStream_t of this context (for torch.cuda.ExternalStream)."""
        return int(self._lib.ps_ctx_stream(self._h) or 0)

    # ------------------------------------------------------------ stages
    def gradient_mask(self, image, threshold: int):
        img = _u8(image)
        h, w = img.shape
        m = np.zeros((h, w), np.uint8)
        n = C.c_int()
        _check(self._lib.ps_gradient_mask(self._h, _ptr(img), w, h, threshold, _ptr(m), C.byref(n)))
        return m, n.value

    def census(self, image) -> np.ndarray:
        img = _u8(image)
        h, w = img.shape
        out = np.zeros((h, w), np.uint32)
        _check(self._lib.ps_census(self._h, _ptr(img), w, h, _ptr(out)))
        return out

    def detect_candidates(self, image, config: PipelineConfig):
        img = _u8(image)
        h, w = img.shape
        cap = 120 * config.perBinCap
        u = np.zeros(cap, np.int32)
        v = np.zeros(cap, np.int32)
        s = np.zeros(cap, np.float32)
        n = C.c_int()
        cfg = config.to_c()
        _check(self._lib.ps_detect_candidates(self._h, _ptr(img), w, h, C.byref(cfg), _ptr(u),
                                              _ptr(v), _ptr(s), cap, C.byref(n)))
        return u[:n.value], v[:n.value], s[:n.value]

    def match_epipolar(self, census_left, census_right, cand_u, cand_v, config: PipelineConfig):
        cl = np.ascontiguousarray(census_left, dtype=np.uint32)
        cr = np.ascontiguousarray(census_right, dtype=np.uint32)
        h, w = cl.shape
        cu = np.ascontiguousarray(cand_u, dtype=np.int32)
        cv = np.ascontiguousarray(cand_v, dtype=np.int32)
        n = len(cu)
        u = np.zeros(max(1, n), np.int32)
        v = np.zeros(max(1, n), np.int32)
        d = np.zeros(max(1, n), np.float64)
        cnt = C.c_int()
        cfg = config.to_c()
        _check(self._lib.ps_match_epipolar(self._h, _ptr(cl), _ptr(cr), w, h, _ptr(cu), _ptr(cv), n,
                                           C.byref(cfg), _ptr(u), _ptr(v), _ptr(d), max(1, n),
                                           C.byref(cnt)))
        k = cnt.value
        return u[:k], v[:k], d[:k]

    def mesh_build(self, u, v, d, tris, width: int, height: int):
        u = np.ascontiguousarray(u, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.int32)
        d = np.ascontiguousarray(d, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
        planes = np.zeros((max(1, len(t)), 3), np.float64)
        lookup = np.zeros((height, width), np.int32)
        _check(self._lib.ps_mesh_build(self._h, _ptr(u), _ptr(v), _ptr(d), len(u), _ptr(t), len(t),
                                       width, height, _ptr(planes), _ptr(lookup)))
        return planes[:len(t)], lookup

    def interpolate(self, lookup, planes, max_disparity: float, mask=None):
        lk = np.ascontiguousarray(lookup, dtype=np.int32)
        pl = np.ascontiguousarray(planes, dtype=np.float64).reshape(-1, 3)
        h, w = lk.shape
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        val = np.zeros((h, w), np.float32)
        ok = np.zeros((h, w), np.uint8)
        _check(self._lib.ps_interpolate(self._h, _ptr(lk), _ptr(pl), len(pl), w, h, _ptr(m),
                                        C.c_float(max_disparity), _ptr(val), _ptr(ok)))
        return val, ok

    def refinement(self, interp, interp_valid, cost, final_disparity, final_valid, final_cost,
                   mask, cell_size: int, config: PipelineConfig):
        """disparityRefinement: updates the final_* arrays in place, returns the
        (confident, invalid) grids as structured arrays (u, v, disparity, cost, occupied)."""
        h, w = np.asarray(interp).shape
        cells = (-(-w // cell_size)) * (-(-h // cell_size))
        dt = np.dtype([("u", np.int32), ("v", np.int32), ("disparity", np.float32),
                       ("cost", np.float32), ("occupied", np.int32)])
        conf = np.zeros(cells, dt)
        inv = np.zeros(cells, dt)
        cfg = config.to_c()
        for a, t in ((final_disparity, np.float32), (final_valid, np.uint8), (final_cost, np.float32)):
            if not (isinstance(a, np.ndarray) and a.dtype == t and a.flags.c_contiguous):
                raise Error("final_* must be C-contiguous arrays of the reference types")
        _check(self._lib.ps_refinement(
            self._h, _ptr(np.ascontiguousarray(interp, np.float32)),
            _ptr(np.ascontiguousarray(interp_valid, np.uint8)),
            _ptr(np.ascontiguousarray(cost, np.float32)), _ptr(final_disparity), _ptr(final_valid),
            _ptr(final_cost), _ptr(np.ascontiguousarray(mask, np.uint8)), w, h, cell_size,
            C.byref(cfg), _ptr(conf), _ptr(inv)))
        return conf, inv

    def support_resampling(self, confident, invalid, cell_size: int, sup_u, sup_v, sup_d,
                           census_left, census_right, config: PipelineConfig):
        """supportResampling over structured cell arrays (as returned by refinement)."""
        cl = np.ascontiguousarray(census_left, np.uint32)
        h, w = cl.shape
        su = np.ascontiguousarray(sup_u, np.int32)
        sv = np.ascontiguousarray(sup_v, np.int32)
        sd = np.ascontiguousarray(sup_d, np.float64)
        cap = len(su) + 2 * len(confident) + 1
        u = np.zeros(cap, np.int32)
        v = np.zeros(cap, np.int32)
        d = np.zeros(cap, np.float64)
        n = C.c_int()
        cfg = config.to_c()
        _check(self._lib.ps_support_resampling(
            self._h, _ptr(np.ascontiguousarray(confident)), _ptr(np.ascontiguousarray(invalid)),
            cell_size, _ptr(su), _ptr(sv), _ptr(sd), len(su), _ptr(cl),
            _ptr(np.ascontiguousarray(census_right, np.uint32)), w, h, C.byref(cfg), _ptr(u),
            _ptr(v), _ptr(d), cap, C.byref(n)))
        return u[:n.value], v[:n.value], d[:n.value]

    def wta_oracle(self, left, right, mask, max_disparity: int):
        """wtaOracle (proj/src/synth.cpp:171-198) on the device:
        (disparity, valid, cost), cost 1.0 off the mask."""
        L = np.ascontiguousarray(left, dtype=np.uint8)
        R = np.ascontiguousarray(right, dtype=np.uint8)
        M = np.ascontiguousarray(mask, dtype=np.uint8)
        if L.shape != R.shape or L.shape != M.shape or L.ndim != 2:
            raise DimensionMismatch("left, right and mask must be equal 2-D arrays")
        h, w = L.shape
        d = np.zeros((h, w), np.float32)
        ok = np.zeros((h, w), np.uint8)
        c = np.zeros((h, w), np.float32)
        _check(self._lib.ps_wta_oracle(self._h, _ptr(L), _ptr(R), w, h, _ptr(M), max_disparity,
                                       _ptr(d), _ptr(ok), _ptr(c)))
        return d, ok, c

    def wta_batch(self, left, right, gradient_threshold: int, max_disparity: int):
        """Dense WTA baseline of an (F, H, W) batch, mask = gradientMask(left, t)."""
        L = np.ascontiguousarray(left, dtype=np.uint8)
        R = np.ascontiguousarray(right, dtype=np.uint8)
        if L.ndim != 3 or L.shape != R.shape:
            raise DimensionMismatch("expected two (F, H, W) uint8 stacks of equal shape")
        n, h, w = L.shape
        d = np.zeros((n, h, w), np.float32)
        ok = np.zeros((n, h, w), np.uint8)
        c = np.zeros((n, h, w), np.float32)
        _check(self._lib.ps_wta_batch(self._h, n, _ptr(L), _ptr(R), w, h, gradient_threshold,
                                      max_disparity, _ptr(d), _ptr(ok), _ptr(c)))
        return d, ok, c

    # ------------------------------------------------------------ encoders
    def encode_kitti16(self, disparity, valid) -> np.ndarray:
        """writeKittiPng's raster (proj/src/io.cpp:349-368): (..., H, 2W) uint8,
        the PNG row bytes (big-endian raw = clamp(lround(d*256), 1, 65535), 0 invalid)."""
        d, v = _maps(disparity, valid)
        *lead, h, w = d.shape
        n = int(np.prod(lead)) if lead else 1
        out = np.zeros(tuple(lead) + (h, 2 * w), np.uint8)
        _check(self._lib.ps_encode_kitti16(self._h, _ptr(d), _ptr(v), w, h, n, _ptr(out)))
        return out

    def encode_pfm(self, disparity, valid) -> np.ndarray:
        """writePfm's raster (proj/src/io.cpp:311-329): rows bottom-up, invalid -1.0."""
        d, v = _maps(disparity, valid)
        *lead, h, w = d.shape
        n = int(np.prod(lead)) if lead else 1
        out = np.zeros(d.shape, np.float32)
        _check(self._lib.ps_encode_pfm(self._h, _ptr(d), _ptr(v), w, h, n, _ptr(out)))
        return out

    def point_cloud(self, disparity, valid, image, calib, min_disparity: float = 0.5):
        """exportPointCloud's vertices (proj/src/io.cpp:395-454): (xyz (N, 3) float32,
        intensity (N,) uint8), row-major; calib = (focal, baseline, cx, cy)."""
        d, v = _maps(disparity, valid)
        img = _u8(image)
        h, w = d.shape
        c = _native.PsCalib(*[float(x) for x in calib])
        cap = int(v.sum()) + 1
        xyz = np.zeros((cap, 3), np.float32)
        inten = np.zeros(cap, np.uint8)
        n = C.c_int()
        _check(self._lib.ps_point_cloud(self._h, _ptr(d), _ptr(v), _ptr(img), w, h, C.byref(c),
                                        C.c_double(min_disparity), _ptr(xyz), _ptr(inten), cap,
                                        C.byref(n)))
        return xyz[:n.value], inten[:n.value]

    def download_kitti16(self, which: int = 0) -> np.ndarray:
        """KITTI raster of the last run's maps, encoded on the device (F, H, 2W)."""
        f, h, w = self._resident_shape()
        out = np.zeros((f, h, 2 * w), np.uint8)
        _check(self._lib.ps_download_kitti16(self._h, which, _ptr(out)))
        return out

    def download_pfm(self, which: int = 0) -> np.ndarray:
        f, h, w = self._resident_shape()
        out = np.zeros((f, h, w), np.float32)
        _check(self._lib.ps_download_pfm(self._h, which, _ptr(out)))
        return out

    def download_point_cloud(self, frame: int, calib, min_disparity: float = 0.5, which: int = 0):
        f, h, w = self._resident_shape()
        c = _native.PsCalib(*[float(x) for x in calib])
        cap = h * w
        xyz = np.zeros((cap, 3), np.float32)
        inten = np.zeros(cap, np.uint8)
        n = C.c_int()
        _check(self._lib.ps_download_point_cloud(self._h, frame, which, C.byref(c),
                                                 C.c_double(min_disparity), _ptr(xyz), _ptr(inten),
                                                 cap, C.byref(n)))
        return xyz[:n.value], inten[:n.value]

    # ---------------------------------------------------------- evaluation
    def accuracy(self, prediction, prediction_valid, ground_truth, ground_truth_valid,
                 mask=None, thresholds=(1.0, 2.0, 3.0)):
        """planestereo::accuracy (proj/src/eval.cpp:19-70) on the device.
        2-D maps -> (fractions, evaluated, meanAbsError); (F, H, W) stacks ->
        arrays (F, T), (F,), (F,).  NoOverlap when a frame has no jointly valid pixel."""
        d, v = _maps(prediction, prediction_valid)
        g, gv = _maps(ground_truth, ground_truth_valid)
        if g.shape != d.shape:
            raise DimensionMismatch("prediction and ground truth dimensions differ")
        m = None
        if mask is not None:
            m = np.ascontiguousarray(mask, np.uint8)
            if m.shape != d.shape:
                raise DimensionMismatch("mask dimensions differ from the disparity maps")
        single = d.ndim == 2
        *lead, h, w = d.shape
        n = int(np.prod(lead)) if lead else 1
        th = np.ascontiguousarray(thresholds, np.float64)
        fr = np.zeros((n, len(th)), np.float64)
        ev = np.zeros(n, np.int64)
        mae = np.zeros(n, np.float64)
        _check(self._lib.ps_accuracy(self._h, n, _ptr(d), _ptr(v), _ptr(g), _ptr(gv),
                                     None if m is None else _ptr(m), w, h, _ptr(th), len(th),
                                     _ptr(fr), _ptr(ev), _ptr(mae)))
        return (fr[0], int(ev[0]), float(mae[0])) if single else (fr, ev, mae)

    def download_accuracy(self, ground_truth, ground_truth_valid, use_mask: bool = True,
                          thresholds=(1.0, 2.0, 3.0), which: int = 0):
        """accuracy of the last run's maps (device-resident) against (F, H, W) ground truth."""
        f, h, w = self._resident_shape()
        g, gv = _maps(ground_truth, ground_truth_valid)
        if g.shape != (f, h, w):
            raise DimensionMismatch("ground truth must be (F, H, W) of the last batch")
        th = np.ascontiguousarray(thresholds, np.float64)
        fr = np.zeros((f, len(th)), np.float64)
        ev = np.zeros(f, np.int64)
        mae = np.zeros(f, np.float64)
        _check(self._lib.ps_download_accuracy(self._h, which, _ptr(g), _ptr(gv), int(use_mask),
                                              _ptr(th), len(th), _ptr(fr), _ptr(ev), _ptr(mae)))
        return fr, ev, mae

    # ------------------------------------------------ on-device generation
    def synth_batch(self, n: int, width: int, height: int, n_planes: int, max_disparity: int,
                    ground: bool = False, noise_sigma: float = 2.0, seed: int = 0,
                    with_gt: bool = False):
        """The BASELINE generator (synth_batch) run on the GPU: same bytes."""
        p = _native.PsSynthParams(width, height, n_planes, max_disparity, 1 if ground else 0,
                                  noise_sigma, seed)
        L = np.zeros((n, height, width), np.uint8)
        R = np.zeros((n, height, width), np.uint8)
        gt = np.zeros((n, height, width), np.float32) if with_gt else None
        _check(self._lib.ps_synth_batch_gpu(self._h, C.byref(p), n, _ptr(L), _ptr(R), _ptr(gt)))
        return (L, R, gt) if with_gt else (L, R)

    def synth_resident(self, n: int, width: int, height: int, n_planes: int, max_disparity: int,
                       ground: bool = False, noise_sigma: float = 2.0, seed: int = 0) -> None:
        """Generate the batch straight into the device input buffers (then run_resident)."""
        p = _native.PsSynthParams(width, height, n_planes, max_disparity, 1 if ground else 0,
                                  noise_sigma, seed)
        _check(self._lib.ps_synth_resident(self._h, C.byref(p), n))
        self._shape = (n, height, width)

    def render_scene(self, width: int, height: int, regions, max_disparity: float = 128.0,
                     seed: int = 1234):
        """renderScene (proj/src/synth.cpp:88-169) on the GPU.  regions: sequence
        of (u0, v0, u1, v1, a, b, c).  -> dict(left, right, gt, gt_valid, occluded)."""
        regs = (_native.PsSceneRegion * max(1, len(regions)))()
        for k, r in enumerate(regions):
            regs[k] = _native.PsSceneRegion(int(r[0]), int(r[1]), int(r[2]), int(r[3]),
                                            float(r[4]), float(r[5]), float(r[6]))
        out = {k: np.zeros((height, width), dt) for k, dt in
               [("left", np.uint8), ("right", np.uint8), ("gt", np.float32),
                ("gt_valid", np.uint8), ("occluded", np.uint8)]}
        _check(self._lib.ps_render_scene(self._h, width, height, float(max_disparity), seed, regs,
                                         len(regions), _ptr(out["left"]), _ptr(out["right"]),
                                         _ptr(out["gt"]), _ptr(out["gt_valid"]),
                                         _ptr(out["occluded"])))
        return out

    def _resident_shape(self):
        if not getattr(self, "_shape", None):
            raise Error("no batch uploaded through this Context")
        return self._shape

    def cost_evaluation(self, census_left, census_right, interp, interp_valid, mask):
        cl = np.ascontiguousarray(census_left, dtype=np.uint32)
        cr = np.ascontiguousarray(census_right, dtype=np.uint32)
        h, w = cl.shape
        iv = np.ascontiguousarray(interp, dtype=np.float32)
        ok = np.ascontiguousarray(interp_valid, dtype=np.uint8)
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        cost = np.zeros((h, w), np.float32)
        _check(self._lib.ps_cost_evaluation(self._h, _ptr(cl), _ptr(cr), w, h, _ptr(iv), _ptr(ok),
                                            _ptr(m), _ptr(cost)))
        return cost


def delaunay_triangulate(u, v, fast: bool = False) -> np.ndarray:
    """planestereo::delaunayTriangulate: (T, 3) index triples (host C++, exact).
    fast=True returns the same set in the engine's radial-sweep order."""
    lib = _native.load()
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    n = len(u)
    cap = max(1, 2 * n)
    tris = np.zeros((cap, 3), np.int32)
    nt = C.c_int()
    fn = lib.ps_delaunay_fast if fast else lib.ps_delaunay
    _check(fn(_ptr(u), _ptr(v), n, _ptr(tris), cap, C.byref(nt)))
    return tris[:nt.value]


def synth_pair(width: int, height: int, n_planes: int, max_disparity: int, ground: bool = False,
               noise_sigma: float = 2.0, seed: int = 0, with_gt: bool = False):
    """Seeded BASELINE-style stereo pair; returns (left, right[, gt])."""
    lib = _native.load()
    p = _native.PsSynthParams(width, height, n_planes, max_disparity, 1 if ground else 0,
                              noise_sigma, seed)
    L = np.zeros((height, width), np.uint8)
    R = np.zeros((height, width), np.uint8)
    gt = np.zeros((height, width), np.float32) if with_gt else None
    _check(lib.ps_synth_pair(C.byref(p), _ptr(L), _ptr(R), _ptr(gt)))
    return (L, R, gt) if with_gt else (L, R)


def _finish_batch(res, st, trace, n, config, raise_on_failure):
    if st != 0 and (raise_on_failure or st != 7):
        _check(st)
    res["trace"] = [[_stats(trace[f * config.iterations + i]) for i in range(config.iterations)]
                    for f in range(n)]
    return res


def run_batch_multi(contexts, left: np.ndarray, right: np.ndarray, config: PipelineConfig,
                    unchecked_cell: bool = False, raise_on_failure: bool = True) -> dict:
    """One (F, H, W) batch sharded over several contexts (one per GPU) from
    this process: ps_run_batch_multi — contiguous frame blocks, one host
    thread per context, no collective.  Same result dict as
    Context.run_batch."""
    L = np.ascontiguousarray(left, dtype=np.uint8)
    R = np.ascontiguousarray(right, dtype=np.uint8)
    if L.ndim != 3 or L.shape != R.shape:
        raise DimensionMismatch("expected two (F, H, W) uint8 stacks of equal shape")
    if not contexts:
        raise ValueError("no contexts")
    n, h, w = L.shape
    cfg = config.to_c()
    res = {"disparity": np.zeros((n, h, w), np.float32), "disparity_valid": np.zeros((n, h, w), np.uint8),
           "costs": np.zeros((n, h, w), np.float32), "dense": np.zeros((n, h, w), np.float32),
           "dense_valid": np.zeros((n, h, w), np.uint8), "status": np.zeros(n, np.int32)}
    handles = (C.c_void_p * len(contexts))(*[cx._h for cx in contexts])
    trace = (PsIterStats * (n * config.iterations))()
    lib = contexts[0]._lib
    st = lib.ps_run_batch_multi(handles, len(contexts), n, _ptr(L), _ptr(R), w, h, C.byref(cfg),
                                PS_RUN_UNCHECKED_CELL if unchecked_cell else 0,
                                _ptr(res["disparity"]), _ptr(res["disparity_valid"]), _ptr(res["costs"]),
                                _ptr(res["dense"]), _ptr(res["dense_valid"]), trace, _ptr(res["status"]))
    per = (n + len(contexts) - 1) // len(contexts)
    for i, cx in enumerate(contexts):  # each context holds its own block
        k = min(n, (i + 1) * per) - min(n, i * per)
        cx._shape = (k, h, w) if k > 0 else None
    return _finish_batch(res, st, trace, n, config, raise_on_failure)


def synth_batch(n_frames: int, width: int, height: int, n_planes: int, max_disparity: int,
                ground: bool = False, noise_sigma: float = 2.0, seed: int = 0, threads: int = 8,
                left: Optional[np.ndarray] = None, right: Optional[np.ndarray] = None):
    """n_frames pairs with seeds seed+i, generated on host threads."""
    lib = _native.load()
    p = _native.PsSynthParams(width, height, n_planes, max_disparity, 1 if ground else 0,
                              noise_sigma, seed)
    L = left if left is not None else np.zeros((n_frames, height, width), np.uint8)
    R = right if right is not None else np.zeros((n_frames, height, width), np.uint8)
    _check(lib.ps_synth_batch(C.byref(p), n_frames, threads, _ptr(L), _ptr(R)))
    return L, R


# BASELINE.json configs.  grid 10 and 6 need the
# unchecked-cell opt-in (they fail the power-of-two rule of validate()).
BASELINE_CONFIGS = {
    0: dict(width=640, height=480, frames=1, n_planes=12, max_disparity=64, ground=False,
            sigma=2.0, iterations=2, cell=10),
    1: dict(width=1242, height=375, frames=1, n_planes=24, max_disparity=128, ground=True,
            sigma=2.0, iterations=4, cell=8),
    2: dict(width=640, height=480, frames=256, n_planes=12, max_disparity=64, ground=False,
            sigma=2.0, iterations=3, cell=10),
    3: dict(width=1920, height=1080, frames=1, n_planes=40, max_disparity=256, ground=False,
            sigma=4.0, iterations=4, cell=8),
    4: dict(width=3840, height=2160, frames=64, n_planes=60, max_disparity=256, ground=False,
            sigma=2.0, iterations=6, cell=6),
}


def baseline_config(idx: int) -> PipelineConfig:
    c = BASELINE_CONFIGS[idx]
    return PipelineConfig(iterations=c["iterations"], maxDisparity=c["max_disparity"],
                          occupancyCellSize=c["cell"])


__all__ = [
    "Error", "InvalidConfig", "DimensionTooSmall", "DimensionMismatch", "FewerThanThreePoints",
    "DegenerateTriangle", "SeedingFailed", "NegativeDisparity", "EmptyCloud", "NoOverlap",
    "InvalidPlane",
    "CudaError", "NoDevice", "PipelineConfig",
    "IterationStats", "StereoResult", "Context", "delaunay_triangulate", "synth_pair",
    "synth_batch", "BASELINE_CONFIGS", "baseline_config", "PS_RUN_UNCHECKED_CELL",
]
