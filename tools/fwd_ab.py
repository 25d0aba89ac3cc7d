"""Diagnostic: forward-launch duration via in-pass events, (a) direct launches with a fixed
draw, (b) direct launches with a fresh draw per iteration, (c) CUDA-graph replays (as
bench.py).  python tools/fwd_ab.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2411_05771_b200 as sk  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["cfg3"]
plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
x1, y = synth.make_workload(cfg, 0)
x1 = torch.from_numpy(x1).cuda()
y = torch.from_numpy(y).cuda()
out = sk.alloc_pass_outputs(plan, cfg.B, cfg.m, "cuda")
ws = plan.workspace(cfg.B, cfg.m)
g = torch.empty(1, dtype=torch.int32, device="cuda")
idx = torch.empty(1, cfg.m, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(it, evs):
    sk.draw_device(0, it, 0, 1, True, cfg.n_full, cfg.m, g=g, idx=idx)
    sk.sketched_pass_profiled(plan, x1, y, g, idx, evs, out, ws)


def direct(fresh):
    ts = []
    for i in range(30):
        flush.zero_()
        evs = [None, mk(), mk(), None, None, None]
        run(i if fresh else 0, evs)
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(evs[1].elapsed_time(evs[2]))
    return np.mean(ts), np.min(ts), np.max(ts)


print("direct fixed draw  mean/min/max ms", direct(False))
print("direct fresh draws mean/min/max ms", direct(True))
evs_all = []
graphs = []
cap = torch.cuda.Stream()
for i in range(30):
    evs = [None, mk(), mk(), None, None, None]
    for e in evs:
        if e is not None:
            e.record()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cap):
        run(i, evs)
    graphs.append(gr)
    evs_all.append(evs)
ts = []
for i in range(30):
    flush.zero_()
    graphs[i].replay()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(evs_all[i][1].elapsed_time(evs_all[i][2]))
print("graph fresh draws  mean/min/max ms", (np.mean(ts), np.min(ts), np.max(ts)))
print("graph per-iteration us (it 5..29):", " ".join(f"{v * 1e3:.0f}" for v in ts))
