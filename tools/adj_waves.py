"""Diagnostic: stage times of the pass vs batch size at cfg3 geometry (wave quantization of the
backprojector: 32 x 32 tiles x groups of 4 images, 3 CTAs per SM).  python tools/adj_waves.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2411_05771_b200 as sk  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for B in (4, 8, 12, 16, 20, 24, 28, 32):
    x1 = torch.from_numpy(synth.rand_images(B, cfg.N, 1)).cuda()
    y = torch.from_numpy(synth.rand_sinograms(B, cfg.n_full, cfg.n_det, 2)).cuda()
    out = sk.alloc_pass_outputs(plan, B, cfg.m, "cuda")
    ws = plan.workspace(B, cfg.m)
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    ts = []
    for it in range(25):
        flush.zero_()
        evs = [mk() for _ in range(6)]
        sk.sketched_pass_profiled(plan, x1, y, g, idx, evs, out, ws)
        torch.cuda.synchronize()
        if it >= 5:
            ts.append([evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(4)])
    t = np.median(np.array(ts), 0)
    print(f"B={B:3d} rot {t[0]:6.1f} fwd {t[1]:6.1f} ramp {t[2]:5.1f} adj {t[3]:6.1f} us   "
          f"adj/img {t[3] / B:5.2f}  fwd/img {t[1] / B:5.2f}")
