import os, sys, time, threading, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1511_00758_b200 as ps
c = ps.BASELINE_CONFIGS[2]; cfg = ps.baseline_config(2); F = 256; W, H = c["width"], c["height"]; P = W * H
L = torch.empty((F, H, W), dtype=torch.uint8).pin_memory().numpy(); R = torch.empty((F, H, W), dtype=torch.uint8).pin_memory().numpy()
ps.synth_batch(F, W, H, c["n_planes"], c["max_disparity"], c["ground"], c["sigma"], seed=1, left=L, right=R)
lib = ps._native.load(); cfgc = cfg.to_c()
for inflight in (1, 2):
    ctxs = [ps.Context(0) for _ in range(inflight)]
    for mode in ("all", "disp", "none"):
        outs = []
        for i in range(inflight):
            o = [torch.empty(F * P * 4, dtype=torch.uint8).pin_memory(), torch.empty(F * P, dtype=torch.uint8).pin_memory(),
                 torch.empty(F * P * 4, dtype=torch.uint8).pin_memory(), torch.empty(F * P * 4, dtype=torch.uint8).pin_memory(),
                 torch.empty(F * P, dtype=torch.uint8).pin_memory()]
            ptrs = [C.c_void_p(x.data_ptr()) for x in o]
            if mode == "disp": ptrs = ptrs[:2] + [None, None, None]
            if mode == "none": ptrs = [None] * 5
            outs.append((o, ptrs))
        tr = [(ps._native.PsIterStats * (F * cfg.iterations))() for _ in range(inflight)]
        st = [np.zeros(F, np.int32) for _ in range(inflight)]
        def call(i):
            return lib.ps_run_batch(ctxs[i]._h, F, C.c_void_p(L.ctypes.data), C.c_void_p(R.ctypes.data), W, H, C.byref(cfgc), ps.PS_RUN_UNCHECKED_CELL, *outs[i][1], tr[i], st[i].ctypes.data_as(C.c_void_p))
        for i in range(inflight): call(i)
        steps = 8
        torch.cuda.synchronize(); t0 = time.perf_counter()
        def worker(i):
            for k in range(i, steps, inflight): call(i)
        ts = [threading.Thread(target=worker, args=(i,)) for i in range(inflight)]
        [t.start() for t in ts]; [t.join() for t in ts]
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"inflight {inflight} outputs {mode}: {steps * F / dt:.0f} frames/s, {dt / steps * 1e3:.1f} ms/step", flush=True)
    for cx in ctxs: cx.close()
