"""TEST INFRASTRUCTURE ONLY — CPU parity checkers for the planestereo hot path.

Two checkers with one Python interface:

* ``load_oracle()`` — ``oracle/_build/libps_oracle.so``, the plain-C
  restatement of the reference algorithm (``oracle/ps_oracle.c``);
* ``load_ref()``    — ``oracle/_ref/libps_ref.so``, the reference's own
  sources compiled in place from /root/reference/proj (``oracle/Makefile``),
  available wherever that build has been run (it is git-ignored but travels
  to the GPU box with the working tree).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package.  The product (``paper_1511_00758_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libps_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libps_ref.so")


class _Cfg(C.Structure):
    _fields_ = [("iterations", C.c_int), ("max_disparity", C.c_int), ("cost_low", C.c_float),
                ("cost_high", C.c_float), ("gradient_threshold", C.c_int),
                ("occupancy_cell_size", C.c_int), ("corner_threshold", C.c_int),
                ("per_bin_cap", C.c_int), ("sparse_accept_cost", C.c_float),
                ("uniqueness_ratio", C.c_float), ("threads", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("iteration", C.c_int), ("support_count", C.c_int), ("triangle_count", C.c_int),
                ("occupancy_cell_size", C.c_int), ("mean_cost", C.c_double),
                ("valid_count", C.c_int), ("millis", C.c_double)]


class _Cell(C.Structure):
    _fields_ = [("u", C.c_int), ("v", C.c_int), ("disparity", C.c_float), ("cost", C.c_float),
                ("occupied", C.c_int)]


CELL_DTYPE = np.dtype([("u", np.int32), ("v", np.int32), ("disparity", np.float32),
                       ("cost", np.float32), ("occupied", np.int32)])

P = C.c_void_p
I = C.c_int


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def to_cfg(cfg) -> _Cfg:
    """Accepts a paper_1511_00758_b200.PipelineConfig-like object or a dict."""
    g = (lambda k: cfg[k]) if isinstance(cfg, dict) else (lambda k: getattr(cfg, k))
    return _Cfg(g("iterations"), g("maxDisparity"), g("costLow"), g("costHigh"),
                g("gradientThreshold"), g("occupancyCellSize"), g("cornerThreshold"),
                g("perBinCap"), g("sparseAcceptCost"), g("uniquenessRatio"), g("threads"))


class _Calib(C.Structure):
    """ps_calib = CameraCalib (proj/include/planestereo/io.hpp:17-24)."""

    _fields_ = [("focal", C.c_double), ("baseline", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double)]


class CpuChecker:
    """numpy interface over a C library exporting <prefix>_* entry points."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        sig = {
            "gradient_mask": (I, [P, I, I, I, P]),
            "census": (None, [P, I, I, P]),
            "detect_candidates": (I, [P, I, I, P, P, P, P, I]),
            "match_epipolar": (I, [P, P, I, I, P, P, I, P, P, P, P]),
            "orient2d": (C.c_longlong, [I] * 6),
            "incircle_sign": (I, [I] * 8),
            "delaunay": (I, [P, P, I, P]),
            "fit_plane": (I, [I, I, C.c_double, I, I, C.c_double, I, I, C.c_double, P]),
            "mesh_build": (I, [P, P, P, P, I, I, I, P, P]),
            "cost_evaluation": (None, [P, P, I, I, P, P, P, P]),
            "wta": (None, [P, P, I, I, P, I, P, P, P]),
            "accuracy": (I, [P, P, P, P, P, I, I, P, I, P, P, P]),
            "refinement": (None, [P, P, P, P, P, P, P, I, I, I, P, P, P]),
            "support_resampling": (I, [P, P, I, P, P, P, I, P, P, I, I, P, P, P, P, I]),
            "run": (I, [P, P, I, I, P, I, P, P, P, P, P, P, P, P, P, I, P]),
            "run_batch": (I, [I, P, P, I, I, P, I, P, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, f"{prefix}_{name}")
            fn.restype = res
            fn.argtypes = args
        if prefix == "orc":
            self.lib.orc_encode_kitti16.restype = C.c_longlong
            self.lib.orc_encode_kitti16.argtypes = [P, P, I, I, P]
            self.lib.orc_encode_pfm.restype = None
            self.lib.orc_encode_pfm.argtypes = [P, P, I, I, P]
            self.lib.orc_point_cloud.restype = I
            self.lib.orc_point_cloud.argtypes = [P, P, P, I, I, P, C.c_double, P, P]
            self.lib.orc_interpolate.restype = None
            self.lib.orc_interpolate.argtypes = [P, P, I, I, P, C.c_float, P, P]
        if prefix == "ref":
            self.lib.ref_interpolate_mesh.restype = None
            self.lib.ref_interpolate_mesh.argtypes = [P, P, P, I, P, I, I, I, P, C.c_float, P, P]
            self.lib.ref_triangulate.restype = I
            self.lib.ref_triangulate.argtypes = [P, P, P, I, I, I, P, P, P]
            self.lib.ref_benchmark_run.restype = C.c_double
            self.lib.ref_benchmark_run.argtypes = [P, P, I, I, P, I]

    def f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    # -- stages
    def gradient_mask(self, img, thr):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        m = np.zeros((h, w), np.uint8)
        n = self.f("gradient_mask")(_p(img), w, h, thr, _p(m))
        return m, n

    def census(self, img):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        out = np.zeros((h, w), np.uint32)
        self.f("census")(_p(img), w, h, _p(out))
        return out

    def detect_candidates(self, img, cfg):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        cap = 120 * cfg.perBinCap
        u = np.zeros(cap, np.int32)
        v = np.zeros(cap, np.int32)
        s = np.zeros(cap, np.float32)
        c = to_cfg(cfg)
        n = self.f("detect_candidates")(_p(img), w, h, C.byref(c), _p(u), _p(v), _p(s), cap)
        return u[:n], v[:n], s[:n]

    def match_epipolar(self, cl, cr, cu, cv, cfg):
        cl = np.ascontiguousarray(cl, np.uint32)
        cr = np.ascontiguousarray(cr, np.uint32)
        h, w = cl.shape
        cu = np.ascontiguousarray(cu, np.int32)
        cv = np.ascontiguousarray(cv, np.int32)
        n = len(cu)
        u = np.zeros(max(1, n), np.int32)
        v = np.zeros(max(1, n), np.int32)
        d = np.zeros(max(1, n), np.float64)
        c = to_cfg(cfg)
        k = self.f("match_epipolar")(_p(cl), _p(cr), w, h, _p(cu), _p(cv), n, C.byref(c), _p(u),
                                     _p(v), _p(d))
        return u[:k], v[:k], d[:k]

    def orient2d(self, a, b, c):
        return self.f("orient2d")(a[0], a[1], b[0], b[1], c[0], c[1])

    def incircle_sign(self, a, b, c, d):
        return self.f("incircle_sign")(a[0], a[1], b[0], b[1], c[0], c[1], d[0], d[1])

    def delaunay(self, u, v):
        u = np.ascontiguousarray(u, np.int32)
        v = np.ascontiguousarray(v, np.int32)
        n = len(u)
        tris = np.zeros((max(1, 2 * n), 3), np.int32)
        t = self.f("delaunay")(_p(u), _p(v), n, _p(tris))
        if t < 0:
            raise ValueError("coordinates out of range")
        return tris[:t]

    def fit_plane(self, p1, p2, p3):
        out = np.zeros(3, np.float64)
        r = self.f("fit_plane")(p1[0], p1[1], p1[2], p2[0], p2[1], p2[2], p3[0], p3[1], p3[2], _p(out))
        if r != 0:
            raise ValueError("degenerate triangle")
        return out

    def mesh_build(self, u, v, d, tris, w, h):
        u = np.ascontiguousarray(u, np.int32)
        v = np.ascontiguousarray(v, np.int32)
        d = np.ascontiguousarray(d, np.float64)
        t = np.ascontiguousarray(tris, np.int32).reshape(-1, 3)
        planes = np.zeros((max(1, len(t)), 3), np.float64)
        lookup = np.zeros((h, w), np.int32)
        r = self.f("mesh_build")(_p(u), _p(v), _p(d), _p(t), len(t), w, h, _p(planes), _p(lookup))
        if r != 0:
            raise ValueError("degenerate triangle")
        return planes[:len(t)], lookup

    def cost_evaluation(self, cl, cr, val, ok, mask):
        cl = np.ascontiguousarray(cl, np.uint32)
        cr = np.ascontiguousarray(cr, np.uint32)
        h, w = cl.shape
        cost = np.zeros((h, w), np.float32)
        self.f("cost_evaluation")(_p(cl), _p(cr), w, h, _p(np.ascontiguousarray(val, np.float32)),
                                  _p(np.ascontiguousarray(ok, np.uint8)),
                                  _p(np.ascontiguousarray(mask, np.uint8)), _p(cost))
        return cost

    # -- io.cpp encoders (restatement only: io.cpp needs libpng, absent here)
    def encode_kitti16(self, d, valid):
        d = np.ascontiguousarray(d, np.float32)
        h, w = d.shape
        out = np.zeros((h, 2 * w), np.uint8)
        neg = self.lib.orc_encode_kitti16(_p(d), _p(np.ascontiguousarray(valid, np.uint8)), w, h, _p(out))
        return out, int(neg)

    def encode_pfm(self, d, valid):
        d = np.ascontiguousarray(d, np.float32)
        h, w = d.shape
        out = np.zeros((h, w), np.float32)
        self.lib.orc_encode_pfm(_p(d), _p(np.ascontiguousarray(valid, np.uint8)), w, h, _p(out))
        return out

    def point_cloud(self, d, valid, image, calib, min_disparity=0.5):
        d = np.ascontiguousarray(d, np.float32)
        h, w = d.shape
        xyz = np.zeros((h * w, 3), np.float32)
        inten = np.zeros(h * w, np.uint8)
        c = _Calib(*[float(x) for x in calib])
        n = self.lib.orc_point_cloud(_p(d), _p(np.ascontiguousarray(valid, np.uint8)),
                                     _p(np.ascontiguousarray(image, np.uint8)), w, h, C.byref(c),
                                     float(min_disparity), _p(xyz), _p(inten))
        return (None, None) if n < 0 else (xyz[:n], inten[:n])

    def accuracy(self, pred, pred_valid, gt, gt_valid, mask, thresholds):
        """accuracy (proj/src/eval.cpp:19-70) -> (status, fractions, evaluated, meanAbsError)."""
        pred = np.ascontiguousarray(pred, np.float32)
        h, w = pred.shape
        th = np.ascontiguousarray(thresholds, np.float64)
        fr = np.zeros(len(th), np.float64)
        ev = C.c_longlong()
        mae = C.c_double()
        st = self.f("accuracy")(_p(pred), _p(np.ascontiguousarray(pred_valid, np.uint8)),
                                _p(np.ascontiguousarray(gt, np.float32)),
                                _p(np.ascontiguousarray(gt_valid, np.uint8)),
                                None if mask is None else _p(np.ascontiguousarray(mask, np.uint8)),
                                w, h, _p(th), len(th), _p(fr), C.byref(ev), C.byref(mae))
        return st, fr, ev.value, mae.value

    def wta(self, left, right, mask, nd):
        """wtaOracle (proj/src/synth.cpp:171-198) -> (disparity, valid, cost)."""
        L = np.ascontiguousarray(left, np.uint8)
        R = np.ascontiguousarray(right, np.uint8)
        h, w = L.shape
        d = np.zeros((h, w), np.float32)
        ok = np.zeros((h, w), np.uint8)
        c = np.zeros((h, w), np.float32)
        self.f("wta")(_p(L), _p(R), w, h, _p(np.ascontiguousarray(mask, np.uint8)), nd, _p(d), _p(ok),
                      _p(c))
        return d, ok, c

    def refinement(self, val, ok, cost, fd, fv, fc, mask, cell, cfg):
        h, w = val.shape
        cols, rows = -(-w // cell), -(-h // cell)
        gc = np.zeros(cols * rows, CELL_DTYPE)
        gi = np.zeros(cols * rows, CELL_DTYPE)
        c = to_cfg(cfg)
        self.f("refinement")(_p(np.ascontiguousarray(val, np.float32)),
                             _p(np.ascontiguousarray(ok, np.uint8)),
                             _p(np.ascontiguousarray(cost, np.float32)), _p(fd), _p(fv), _p(fc),
                             _p(np.ascontiguousarray(mask, np.uint8)), w, h, cell, C.byref(c),
                             _p(gc), _p(gi))
        return gc, gi

    def support_resampling(self, gc, gi, cell, su, sv, sd, cl, cr, cfg):
        h, w = cl.shape
        cap = len(su) + 2 * len(gc) + 16
        ou = np.zeros(cap, np.int32)
        ov = np.zeros(cap, np.int32)
        od = np.zeros(cap, np.float64)
        c = to_cfg(cfg)
        n = self.f("support_resampling")(_p(gc), _p(gi), cell,
                                         _p(np.ascontiguousarray(su, np.int32)),
                                         _p(np.ascontiguousarray(sv, np.int32)),
                                         _p(np.ascontiguousarray(sd, np.float64)), len(su),
                                         _p(np.ascontiguousarray(cl, np.uint32)),
                                         _p(np.ascontiguousarray(cr, np.uint32)), w, h, C.byref(c),
                                         _p(ou), _p(ov), _p(od), cap)
        return ou[:n], ov[:n], od[:n]

    def run(self, left, right, cfg, validate: int = 0) -> dict:
        L = np.ascontiguousarray(left, np.uint8)
        R = np.ascontiguousarray(right, np.uint8)
        h, w = L.shape
        P_ = w * h
        out = {
            "disparity": np.zeros((h, w), np.float32),
            "disparity_valid": np.zeros((h, w), np.uint8),
            "costs": np.zeros((h, w), np.float32),
            "dense": np.zeros((h, w), np.float32),
            "dense_valid": np.zeros((h, w), np.uint8),
        }
        trace = (_Stats * max(1, cfg.iterations))()
        su = np.zeros(P_ + 16, np.int32)
        sv = np.zeros(P_ + 16, np.int32)
        sd = np.zeros(P_ + 16, np.float64)
        ns = C.c_int(0)
        c = to_cfg(cfg)
        st = self.f("run")(_p(L), _p(R), w, h, C.byref(c), validate, _p(out["disparity"]),
                           _p(out["disparity_valid"]), _p(out["costs"]), _p(out["dense"]),
                           _p(out["dense_valid"]), trace, _p(su), _p(sv), _p(sd), P_ + 16,
                           C.byref(ns))
        out["status"] = st
        out["supports"] = (su[:ns.value].copy(), sv[:ns.value].copy(), sd[:ns.value].copy())
        out["trace"] = [dict(iteration=t.iteration, supportCount=t.support_count,
                             triangleCount=t.triangle_count,
                             occupancyCellSize=t.occupancy_cell_size, meanCost=t.mean_cost,
                             validCount=t.valid_count, millis=t.millis)
                        for t in list(trace)[:cfg.iterations]]
        return out

    def run_batch(self, left, right, cfg, threads: int, outputs: bool = False):
        L = np.ascontiguousarray(left, np.uint8)
        R = np.ascontiguousarray(right, np.uint8)
        n, h, w = L.shape
        c = to_cfg(cfg)
        status = np.zeros(n, np.int32)
        if outputs:
            d = np.zeros((n, h, w), np.float32)
            dv = np.zeros((n, h, w), np.uint8)
            co = np.zeros((n, h, w), np.float32)
            de = np.zeros((n, h, w), np.float32)
            dev = np.zeros((n, h, w), np.uint8)
        else:
            d = dv = co = de = dev = None
        self.f("run_batch")(n, _p(L), _p(R), w, h, C.byref(c), threads, _p(d), _p(dv), _p(co),
                            _p(de), _p(dev), _p(status))
        return dict(status=status, disparity=d, disparity_valid=dv, costs=co, dense=de,
                    dense_valid=dev)


def load_oracle() -> CpuChecker:
    return CpuChecker(ORACLE_SO, "orc")


def load_ref() -> Optional[CpuChecker]:
    """The compiled reference, or None when oracle/_ref was not built."""
    if not os.path.exists(REF_SO):
        return None
    return CpuChecker(REF_SO, "ref")


def build(reference_root: str = "/root/reference/proj") -> None:
    """Builds the C restatement, and the reference checker when its sources exist."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if os.path.isdir(reference_root):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={reference_root}"], check=True)
