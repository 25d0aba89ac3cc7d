"""Diagnostic: per-CTA start/end times of the forward kernel from a SKEI_FWD_TRACE build
(libskei built with -DSKEI_FWD_TRACE at the path in argv[1]).  Prints the distribution of
start delays and end times relative to the earliest start, and units per CTA."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2411_05771_b200 as sk  # noqa: E402
import synth  # noqa: E402

sk.lib_path = sys.argv[1]
cfg = synth.CONFIGS["cfg3"]
plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
x1, y = synth.make_workload(cfg, 0)
x1 = torch.from_numpy(x1).cuda()
y = torch.from_numpy(y).cuda()
out = sk.alloc_pass_outputs(plan, cfg.B, cfg.m, "cuda")
ws = plan.workspace(cfg.B, cfg.m)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
its = [int(a[4:]) for a in sys.argv if a.startswith("--it")] or [0]
for it in its:
  g, idx = sk.draw_device(0, it, 0, 1, True, cfg.n_full, cfg.m)
  nrow = int(((4 * idx[0] <= cfg.n_full) | (4 * idx[0] >= 3 * cfg.n_full)).sum())
  for i in range(3):
    if "--flush" in sys.argv:
        flush.zero_()
    sk.sketched_pass(plan, x1, y, g, idx, out=out, ws=ws)
  torch.cuda.synchronize()
  n = 4 * 1024
  buf = (ctypes.c_ulonglong * n)()
  L = sk.lib()
  L.skei_debug_fwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
  assert L.skei_debug_fwd_trace(buf, n) == 0
  a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4).astype(np.int64)
  a = a[a[:, 1] > 0]
  t0 = a[:, 0].min()
  en = (a[:, 1] - t0) / 1e3
  info = a[0, 2]
  K, Lr, U = (info >> 16) & 0xff, (info >> 24) & 0xff, info >> 32
  un = a[:, 2] & 0xffff
  print(f"it {it}: nrow {nrow} K {K} Lr {Lr} U {U} units/CTA {np.bincount(un)} end p50 {np.median(en):.1f} max {en.max():.1f} busy {((a[:,1]-a[:,0])/1e3).sum()/(len(a)*en.max()):.3f}")
sys.exit(0)
n = 4 * 1024
buf = (ctypes.c_ulonglong * n)()
L = sk.lib()
L.skei_debug_fwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.skei_debug_fwd_trace(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4).astype(np.int64)
a = a[a[:, 1] > 0]
t0 = a[:, 0].min()
st, en, un, sm = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2], a[:, 3]
print(f"CTAs {len(a)}  distinct SMs {len(set(sm))}")
print("start us: min %.1f p50 %.1f p90 %.1f max %.1f" % (st.min(), np.median(st), np.percentile(st, 90), st.max()))
print("end   us: min %.1f p10 %.1f p50 %.1f max %.1f" % (en.min(), np.percentile(en, 10), np.median(en), en.max()))
print("units per CTA:", np.bincount(un))
busy = (en - st).sum() / (len(a) * en.max())
print("busy fraction (sum of CTA lifetimes / (CTAs x makespan)) %.3f" % busy)
