"""Diagnostic: host enqueue time and single-stream step time of skei_pass_host at cfg3, for
the y_S transfer variants (strided copies per run of angles vs host gather + one copy)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05771_b200 as sk  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
x1, y = synth.make_workload(cfg, 0)
hx1, hy = torch.from_numpy(x1).pin_memory(), torch.from_numpy(y).pin_memory()
d = sk.alloc_pass_outputs(plan, cfg.B, cfg.m, "cuda")
d.update(x1=torch.empty(x1.shape, device="cuda"), y=torch.empty(y.shape, device="cuda"),
         g=torch.empty(1, dtype=torch.int32, device="cuda"),
         idx=torch.empty(1, cfg.m, dtype=torch.int32, device="cuda"))
ws = plan.workspace(cfg.B, cfg.m)
hmc, hei = torch.empty(cfg.B).pin_memory(), torch.empty(cfg.B).pin_memory()
ys = torch.empty(cfg.B, cfg.m, cfg.n_det).pin_memory()
for mode in (sk.MODE_UNIFORM, sk.MODE_INTERLEAVED):
    g, idx = sk.draw(0, 0, sk.SHARED_IMAGE, cfg.n_full, cfg.m, mode)
    hg = torch.tensor([g], dtype=torch.int32).pin_memory()
    hidx = torch.tensor([idx], dtype=torch.int32).pin_memory()
    runs = 1 + int(np.sum(np.diff(idx) != 1))
    for stage in (None, ys):
        call = lambda: sk.sketched_pass_host(plan, hx1, hy, hg, hidx, d, hmc, hei, ws, d["x2"],  # noqa: E731
                                             h_ystage=stage)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            call()
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / 50
        print(f"mode {mode} runs {runs} {'staged' if stage is not None else 'strided'}: "
              f"enqueue {np.median(ts) * 1e3:.3f} ms, single-stream step {el * 1e3:.3f} ms")
