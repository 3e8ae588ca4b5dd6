#!/usr/bin/env python
"""Benchmark of the B200 planestereo hot path (BASELINE.json metric:
"stereo frames/sec & Mpix/s at VGA, N iterations; achieved HBM GB/s vs peak").

Workload (default): BASELINE config 2 — a batch of 256 seeded synthetic VGA
pairs per GPU, 3 iterations, support grid 10 px, max disparity 64 (the
BASELINE generator stand-in of SURVEY 8(d); no dataset exists offline).  A
"step" is one full pipeline pass (planestereo::run semantics, including the
host Delaunay of every iteration) over the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by torchrun (one rank per GPU); frames are independent, so
each rank processes its own batch with no data-path collective ("weak"
scaling); NCCL is used only for the barrier and the max-over-ranks timing.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref, the unmodified reference sources; the C restatement if that
build is absent) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stereo frames/sec & Mpix/s at VGA, N iterations; achieved HBM GB/s vs peak"
UNIT = "frames/s"


# BASELINE.json configs (SURVEY 8(d) mapping); the same table as
# paper_1511_00758_b200.BASELINE_CONFIGS (checked in the ours arm), repeated
# here so the reference arm never imports the product package.
CONFIGS = {
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


def config_fields(k: int) -> dict:
    """PipelineConfig field dict (proj/include/planestereo/config.hpp:8-34 defaults)."""
    c = CONFIGS[k]
    return dict(iterations=c["iterations"], maxDisparity=c["max_disparity"], costLow=0.25,
                costHigh=0.5, gradientThreshold=20, occupancyCellSize=c["cell"], cornerThreshold=20,
                perBinCap=5, sparseAcceptCost=0.25, uniquenessRatio=0.9, threads=1)


def config_line(args, frames: int, world: int) -> dict:
    """The `config` object of both arms' JSON lines (identical by construction)."""
    c = CONFIGS[args.config]
    return {"workload": f"BASELINE config {args.config}: {frames} x {c['width']}x{c['height']} pairs per GPU, "
                        f"{c['iterations']} iterations, grid {c['cell']}, ND {c['max_disparity']}",
            "frames_per_gpu": frames, "parallelism": f"frame-sharded x{world} (no collective)",
            "l2": "working set (census+state ~2.9 GB/batch) far larger than L2; no flush needed"}


def host_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": os.cpu_count() or 1, "usable_cpus": usable}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2, help="BASELINE.json config index")
    p.add_argument("--frames", type=int, default=0, help="frames per GPU (default: the config's)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--inflight", type=int, default=0,
                   help="batches in flight per GPU: that many contexts on the GPU, one host thread "
                        "each, steps dealt round-robin (double buffering: one batch's host tail and "
                        "output copies overlap the next batch's device work)")
    p.add_argument("--cpu-sample-frames", type=int, default=128)
    p.add_argument("--ref-all", action="store_true",
                   help="with --configs: also time the reference throughput leg of cfg4 "
                        "(one frame per host thread, ~20 min)")
    p.add_argument("--configs", default="",
                   help="comma list of BASELINE configs: print a markdown table of ours (ps_run_batch, "
                        "pinned buffers, wall clock) vs the reference CPU arm instead of the JSON line")
    return p.parse_args()


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class NvmlClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 200 ms during the
    timed region, in process through NVML: the nvidia-smi polling process it
    replaces competed for the host cores the Delaunay workers run on."""

    BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
        self.samples = []
        self.stop_ev = threading.Event()

    def start(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, smax, rs))
            except Exception:
                pass
            self.stop_ev.wait(0.2)

    def stop(self):
        self.stop_ev.set()
        self.thread.join(timeout=5)
        sm = [x[0] for x in self.samples]
        reasons = sorted({n for _, _, r in self.samples for n, b in self.BITS.items() if r & b})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(x[1] for x in self.samples) if sm else None,
                "reasons": reasons, "samples": len(sm), "via": "nvml"}


def clock_sampler(gpu: int):
    """NVML in process when available (PS_CLOCKS=smi forces the nvidia-smi poller)."""
    if os.environ.get("PS_CLOCKS") != "smi":
        try:
            return NvmlClockSampler(gpu)
        except Exception:
            pass
    return ClockSampler(gpu)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def traffic_from_profiles(kernel: str):
    """dram__bytes_read+write per launch of `kernel` from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def cpu_checker():
    import oracle

    ref = oracle.load_ref()
    if ref is not None:
        return ref, "reference"
    return oracle.load_oracle(), "port"


def rank_seed(rank: int, frames: int) -> int:
    """First generator seed of a rank's batch: ranks get disjoint frame sets
    (frames never interact, so sharding needs no collective)."""
    return 1000 + rank * frames


def whole_job_value(frames_per_rank: int, world: int, steps: int, max_ms: float) -> float:
    """Aggregate frames/s over all ranks from the slowest rank's time."""
    return frames_per_rank * world * steps / (max_ms / 1e3)


def make_inputs(ps, cfgd, frames, seed, pinned):
    import numpy as np

    h, w = cfgd["height"], cfgd["width"]
    if pinned:
        import torch

        tl = torch.empty((frames, h, w), dtype=torch.uint8, pin_memory=True)
        tr = torch.empty((frames, h, w), dtype=torch.uint8, pin_memory=True)
        L, R = tl.numpy(), tr.numpy()
    else:
        tl = tr = None
        L = np.empty((frames, h, w), np.uint8)
        R = np.empty((frames, h, w), np.uint8)
    ps.synth_batch(frames, w, h, cfgd["n_planes"], cfgd["max_disparity"], cfgd["ground"],
                   cfgd["sigma"], seed=seed, threads=os.cpu_count() or 8, left=L, right=R)
    return L, R, (tl, tr)


def reference_inputs(ref, k: int, frames: int, seed: int):
    """The seeded pairs, generated inside oracle/_ref (ref_synth_batch: the
    repo's generator compiled into the checker), byte-identical to the ones
    the ours arm generates through the product."""
    import numpy as np

    c = CONFIGS[k]
    L = np.empty((frames, c["height"], c["width"]), np.uint8)
    R = np.empty_like(L)
    fn = ref.lib.ref_synth_batch
    fn.restype = C.c_int
    fn.argtypes = [C.c_int] * 4 + [C.c_int, C.c_float, C.c_uint, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    st = fn(c["width"], c["height"], c["n_planes"], c["max_disparity"], int(c["ground"]), c["sigma"],
            seed, frames, os.cpu_count() or 8, L.ctypes.data, R.ctypes.data)
    if st != 0:
        raise RuntimeError(f"ref_synth_batch failed: {st}")
    return L, R


def reference_latency(ref, L, R, cfgd, repeats=5):
    """The reference's own harness, benchmark(fn, repeats, pinToCore=true)
    (proj/src/eval.cpp:144-177, via ref_benchmark_run): median ms, one thread."""
    import oracle

    fn = ref.lib.ref_benchmark_run
    c = oracle.to_cfg(cfgd)
    h, w = L.shape
    return float(fn(L.ctypes.data, R.ctypes.data, w, h, C.byref(c), repeats))


def run_reference_arm(args, rank, world):
    """The reference's CPU path: oracle/_ref (the unmodified reference
    sources compiled in place, driven by the staged run() loop) on all host
    threads, one frame per thread.  Only oracle/_ref is loaded in this process."""
    if rank != 0:
        return
    import oracle

    ref = oracle.load_ref()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    cfgd = config_fields(args.config)
    c = CONFIGS[args.config]
    frames = args.frames or c["frames"]
    cores = os.cpu_count() or 1
    L, R = reference_inputs(ref, args.config, frames, rank_seed(0, frames))
    for _ in range(args.warmup):
        ref.run_batch(L, R, cfgd, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        st = ref.run_batch(L, R, cfgd, cores)["status"]
    dt = time.perf_counter() - t0
    value = frames * args.steps / dt
    P = c["width"] * c["height"]
    lat = reference_latency(ref, L[0], R[0], cfgd) if c["width"] * c["height"] <= 2_100_000 else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32/f32/f64",
        "data": "synthetic (seeded BASELINE-style generator, SURVEY 8(d)); host memory",
        "config": config_line(args, frames, world),
        "mpix_per_s": value * P / 1e6,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"all {frames} frames per step, one frame per host thread on {cores} "
                                   f"threads, oracle/_ref (reference sources, staged run())",
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "latency": {"reference_ms_median": lat,
                    "what": "one frame, benchmark(fn, 5, pinToCore=true) (eval.cpp:144-177)"},
        "failed_frames": int((st != 0).sum()),
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1511_00758_b200 as ps

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfgd = ps.BASELINE_CONFIGS[args.config]
    assert cfgd == CONFIGS[args.config], "bench.CONFIGS out of sync with the package"
    cfg = ps.baseline_config(args.config)
    assert {f: getattr(cfg, f) for f in cfg.__dataclass_fields__} == config_fields(args.config)
    frames = args.frames or cfgd["frames"]
    H, W = cfgd["height"], cfgd["width"]
    P = W * H
    L, R, keep = make_inputs(ps, cfgd, frames, rank_seed(rank, frames), pinned=True)
    inflight = args.inflight if args.inflight > 0 else (3 if world < 4 else 2)
    ctxs = [ps.Context(local_rank) for _ in range(inflight)]
    ctx = ctxs[0]
    stream = torch.cuda.current_stream()
    lib = ps._native.load()

    def run_steps(fn):
        """Steps dealt round-robin to the contexts, one host thread each (the
        C calls release the GIL); returns when every step has finished."""
        if inflight == 1:
            for k in range(args.steps):
                fn(0, k)
            return
        errs = []

        def worker(i):
            try:
                for k in range(i, args.steps, inflight):
                    fn(i, k)
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        ts = [threading.Thread(target=worker, args=(i,)) for i in range(inflight)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]

    def merged_stats():
        out = {}
        for c in ctxs:
            for k, v in c.kernel_stats().items():
                o = out.setdefault(k, {"launches": 0, "ms": 0.0, "bytes": 0.0})
                o["launches"] += v["launches"]
                o["ms"] += v["ms"]
                o["bytes"] += v.get("bytes", 0.0)
        return out

    # ---------------- value: inputs resident in HBM, full pipeline per step
    for c in ctxs:
        c.upload_ptr(frames, L.ctypes.data, R.ctypes.data, W, H)
        for _ in range(max(3, args.warmup)):
            st = c.run_resident(cfg, unchecked_cell=True)
            if st not in (0, 7):
                raise RuntimeError(f"pipeline failed: {lib.ps_last_error(None)}")
    sampler = clock_sampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    l0 = sum(c.launch_count() for c in ctxs)
    # per-kernel CUDA events, recorded by the engine on the stream each kernel
    # is launched on, live over the timed region (the roofline below)
    for c in ctxs:
        c.set_profiling(True)
        c.reset_kernel_stats()
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    w0 = time.perf_counter()
    run_steps(lambda i, k: ctxs[i].run_resident(cfg, unchecked_cell=True))
    torch.cuda.synchronize()  # every context's streams (device-wide)
    e1.record(stream)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3
    barrier()
    clocks = sampler.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = sum(c.launch_count() for c in ctxs) - l0
    kstats_timed = merged_stats()
    for c in ctxs:
        c.set_profiling(False)
    # Also one extra pass (outside the timed region) with the frame groups
    # serialised on one stream: each kernel's event time is then its isolated
    # launch duration (in the timed pass kernels of different groups overlap).
    ctx.set_profiling(True)
    ctx.set_max_groups(1)
    ctx.reset_kernel_stats()
    ctx.run_resident(cfg, unchecked_cell=True)
    kstats = ctx.kernel_stats()
    ctx.set_profiling(False)
    ctx.set_max_groups(int(os.environ.get("PS_MAX_GROUPS", "8")))
    status = np.zeros(frames, np.int32)
    lib.ps_download_batch(ctx._h, None, None, None, None, None, None, status.ctypes.data_as(C.c_void_p))
    value = whole_job_value(frames, world, args.steps, ms)

    # ---------------- e2e: public C-ABI call with host buffers (pinned), copies inside
    def out_set():
        return [torch.empty(frames * P * 4, dtype=torch.uint8, pin_memory=True),
                torch.empty(frames * P, dtype=torch.uint8, pin_memory=True),
                torch.empty(frames * P * 4, dtype=torch.uint8, pin_memory=True),
                torch.empty(frames * P * 4, dtype=torch.uint8, pin_memory=True),
                torch.empty(frames * P, dtype=torch.uint8, pin_memory=True)]

    outs = [out_set() for _ in ctxs]
    traces = [(ps._native.PsIterStats * (frames * cfg.iterations))() for _ in ctxs]
    trace = traces[0]
    cfgc = cfg.to_c()
    st_arrs = [np.zeros(frames, np.int32) for _ in ctxs]

    def e2e_call(i, k=0):
        return lib.ps_run_batch(ctxs[i]._h, frames, C.c_void_p(L.ctypes.data), C.c_void_p(R.ctypes.data),
                                W, H, C.byref(cfgc), ps.PS_RUN_UNCHECKED_CELL,
                                *[C.c_void_p(o.data_ptr()) for o in outs[i]], traces[i],
                                st_arrs[i].ctypes.data_as(C.c_void_p))

    for i in range(inflight):
        e2e_call(i)
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    run_steps(e2e_call)
    torch.cuda.synchronize()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    e2e_value = whole_job_value(frames, world, args.steps, e2e_ms)
    h2d = 2 * frames * P
    # D_f 4 B + dense 4 B + dense validity 1 B per pixel, and C_f / validity as
    # one code byte (expanded on the host: engine wire_codes; PS_WIRE_CODES=0: 5 B)
    wire = os.environ.get("PS_WIRE_CODES", "1") != "0"
    d2h = frames * P * (4 + 4 + 1 + (1 if wire else 5)) + frames * cfg.iterations * C.sizeof(ps._native.PsIterStats)

    # ---------------- single-frame latency through ps_run, wall clock
    lat = []
    for _ in range(5):
        t0 = time.perf_counter()
        ctx.run(L[0], R[0], cfg, unchecked_cell=True)
        lat.append((time.perf_counter() - t0) * 1e3)
    lat.sort()

    # ---------------- Delaunay throughput (K4 is host work: points/s)
    points_per_pass = sum(int(t.support_count) for t in trace)  # the e2e batch's trace
    sweep = kstats_timed.get("host_mesh", {"ms": 0.0})
    mesh_events = {k: kstats_timed.get(k, {}).get("launches", 0) // args.steps
                   for k in ("host_replay", "host_order", "host_check")}

    # ---------------- roofline of the dominant graded kernel (K7 refine)
    peak, peak_src = measured_peak()

    def per_launch(stats):
        k = stats.get("refine", {"launches": 0, "ms": 0.0, "bytes": 0.0})
        b = k["bytes"] / max(1, k["launches"])
        t = k["ms"] / max(1, k["launches"])
        return b, t, (b / (t * 1e-3) / 1e9 if t > 0 else 0.0)

    # live over the timed region (frame groups overlapping on the device)
    per_launch_bytes, per_launch_ms, achieved = per_launch(kstats_timed)
    iso_bytes, iso_ms, iso_achieved = per_launch(kstats)
    kernels = {k: {"launches": v["launches"], "ms_per_pass": v["ms"],
                   "gbs": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] > 0 and v["bytes"] > 0 else None}
               for k, v in kstats.items()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32/f32/f64",
        "data": "synthetic (seeded BASELINE-style generator, SURVEY 8(d)); inputs resident in HBM",
        "config": config_line(args, frames, world),
        "host": {**host_info(), "workers_per_rank": ctx.host_threads()},
        "mpix_per_s": value * P / 1e6,
        "wall_ms_per_step": wall_ms / args.steps,
        "gpu_launches": int(launches),
        "roofline": {"kernel": "k_refine (K7 interpolate+cost+refine, fused K9 on the last iteration)",
                     "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "peak_source": peak_src,
                     "frac_of_spec_8tbs": achieved / 8000.0,
                     "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "launches_timed": kstats_timed.get("refine", {}).get("launches", 0),
                     "measured": "CUDA events on each launch's own stream, live over the timed region",
                     "isolated": {"achieved": iso_achieved, "frac": iso_achieved / peak if peak else None,
                                  "bytes_per_launch": iso_bytes, "ms_per_launch": iso_ms,
                                  "note": "one extra pass with the frame groups serialised (no overlap)"},
                     "traffic": traffic_from_profiles("k_refine")},
        "kernels_isolated_pass": kernels,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "ps_run_batch (C ABI) with pinned host buffers",
                "inflight": inflight},
        "inflight": {"batches": inflight,
                     "how": "one context per in-flight batch on the same GPU, one host thread each, steps "
                            "dealt round-robin; the timed region runs from before the first step to "
                            "after the last step of every context (device-wide synchronize)"},
        "clocks": clocks,
        "failed_frames": int((status != 0).sum()),
        "delaunay": {"points_per_pass": points_per_pass,
                     "points_per_s": points_per_pass / (ms / args.steps / 1e3),
                     "sweep_ms_per_pass_per_worker": sweep["ms"] / args.steps,
                     "sweep_ms_per_frame_iteration":
                         sweep["ms"] / args.steps * ctx.host_threads() / (frames * cfg.iterations),
                     "workers": ctx.host_threads(),
                     "replayed_frame_iterations_per_pass": mesh_events["host_replay"],
                     "order_queries_per_pass": mesh_events["host_order"],
                     "planes_fitted_three_ways_per_pass": mesh_events["host_check"],
                     "frame_iterations_per_pass": frames * cfg.iterations,
                     "note": "host mesh per frame and iteration: incremental exact Delaunay (previous "
                             "iteration + new supports), reference sweep order/rotation recovered only "
                             "where the output depends on it (frame_mesh.hpp); replay = delaunay_lex"},
        "host_pipeline_ms_per_step": {k: v["ms"] / args.steps for k, v in kstats_timed.items()
                                      if k.startswith("host_")},
        "latency": {"ours_ms_min": lat[0], "ours_ms_median": lat[len(lat) // 2],
                    "what": "one frame of the workload through ps_run (host buffers in and out), wall clock"},
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        checker, kind = cpu_checker()
        n = min(args.cpu_sample_frames, frames)
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        checker.run_batch(L[:n], R[:n], cfg, cores)
        dt = time.perf_counter() - t0
        if kind == "reference":
            line["latency"]["reference_ms_median"] = reference_latency(
                checker, np.ascontiguousarray(L[0]), np.ascontiguousarray(R[0]), config_fields(args.config))
            line["latency"]["reference_what"] = "benchmark(fn, 5, pinToCore=true) (eval.cpp:144-177), median"
        line["cpu_baseline"] = {
            "value": n / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{n} of the {frames} frames, one frame per host thread on {cores} threads "
                      f"({'oracle/_ref: reference sources' if kind == 'reference' else 'oracle/ps_oracle.c'})",
            **host_info()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for c in ctxs:
        c.close()
    if dist is not None:
        dist.destroy_process_group()
    del keep


CONFIG_FRAMES = {0: 64, 1: 64, 2: 256, 3: 16, 4: 16}
CONFIG_REF = {0: True, 1: True, 2: True, 3: True, 4: False}


def run_configs_table(args):
    """SURVEY 8(d) for every BASELINE config: ours (one batch through ps_run_batch with
    pinned buffers, copies included; one frame through ps_run) beside the
    reference CPU arm (one frame per host thread on all threads; one frame on
    one thread).  Wall clock: the whole call is the unit of work; the device-
    timed headline is the JSON line.  The reference legs are skipped where one
    frame takes minutes (cfg4)."""
    import numpy as np
    import torch

    import paper_1511_00758_b200 as ps

    cfgs = [int(c) for c in args.configs.split(",")]
    ctx = ps.Context(0)
    threads = ctx.host_threads()
    ref, _ = cpu_checker()
    print("| config | shape | iterations | frames | ours frames/s (e2e) | ours Mpix/s | ours 1-frame ms "
          "| reference frames/s (%d threads) | reference 1-frame ms | speed-up (throughput) |" % threads)
    print("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|")
    for k in cfgs:
        c = ps.BASELINE_CONFIGS[k]
        cfg = ps.baseline_config(k)
        n = CONFIG_FRAMES[k]
        w, h = c["width"], c["height"]
        L = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True).numpy()
        R = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True).numpy()
        ps.synth_batch(n, w, h, c["n_planes"], c["max_disparity"], c["ground"], c["sigma"], seed=4000 + k,
                       left=L, right=R)
        out = {key: torch.empty((n, h, w), dtype=dt, pin_memory=True).numpy()
               for key, dt in [("disparity", torch.float32), ("disparity_valid", torch.uint8),
                               ("costs", torch.float32), ("dense", torch.float32),
                               ("dense_valid", torch.uint8)]}
        ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False, out=out)  # warm-up
        t0 = time.perf_counter()
        res = ctx.run_batch(L, R, cfg, unchecked_cell=True, raise_on_failure=False, out=out)
        dt = time.perf_counter() - t0
        ours = n / dt
        lat = []
        for _ in range(1 if k == 4 else 3):
            t0 = time.perf_counter()
            ctx.run(L[0], R[0], cfg, unchecked_cell=True)
            lat.append((time.perf_counter() - t0) * 1e3)
        rfps = rlat = None
        if ref is not None and (CONFIG_REF[k] or args.ref_all):
            m = min(n, threads)
            t0 = time.perf_counter()
            ref.run_batch(L[:m], R[:m], cfg, threads)
            rfps = m / (time.perf_counter() - t0)
            if CONFIG_REF[k]:  # cfg4: one frame alone would take another ~18 min
                t0 = time.perf_counter()
                ref.run(L[0], R[0], cfg)
                rlat = (time.perf_counter() - t0) * 1e3
        failed = int((np.asarray(res["status"]) != 0).sum())
        print(f"| cfg{k} | {w}x{h}, ND {c['max_disparity']}, grid {c['cell']} | {c['iterations']} | {n}"
              f"{' (' + str(failed) + ' failed)' if failed else ''} | {ours:.1f} | {ours * w * h / 1e6:.1f} "
              f"| {min(lat):.1f} | {'%.2f' % rfps if rfps else 'not run'} | {'%.0f' % rlat if rlat else 'not run'} "
              f"| {'%.1fx' % (ours / rfps) if rfps else '-'} |", flush=True)
    ctx.close()



def relaunch_under_torchrun(n: int) -> None:
    """`python bench.py --gpus N` without a launcher: re-exec as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.configs:
        relaunch_under_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.configs:
        run_configs_table(args)
    elif args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
