#!/usr/bin/env python
"""bench.py — throughput of the B200-native sketched-EI operator pass (arXiv 2411.05771).

Metric (BASELINE.json): "sketched EI operator passes/s at 512^2, 360->90 angles; % HBM/gather
roofline".  One step = one whole pass of SURVEY §8(a) (a1 draw, a2 rotate, a3 two forward
projections, a4 ramp, a5 FBP backprojection, a7 residuals, a8 gradient backprojection) over
one batch of config 3 (512x512 fp32, B = 16, 360 angles, 725 bins, m = 90 uniform sketch,
P = 2048), inputs resident in HBM, L2 flushed (256 MB write) before every timed step, each
step timed with CUDA events on the launching stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl skei|reference] [--config cfgN]

Multi-GPU: one rank per GPU.  Launched by torchrun (RANK / LOCAL_RANK / WORLD_SIZE in the
environment) or, when `--gpus N > 1` is given without them, bench.py re-launches itself
under `torch.distributed.run` with N ranks on this node (127.0.0.1).  The path partitions
by image batch with no data-path collective: for config 3 (the headline) every rank runs
its own 16-image batch (weak scaling, value = N*K passes / max-over-ranks device time);
for config 4 ("batch 64 split by batch across 1/2/4/8 GPUs") the 64 images are split
64/N per rank, draws keyed by the global image index (strong scaling, value = K whole
64-image passes / max-over-ranks device time).  `--impl reference` times the fp64 oracle
(the only reference this paper-only tier has) on the host cores, whole passes.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

UNIT = "passes/s"
# configs whose batch is split over the ranks (strong scaling; BASELINE.json cfg4 "batch 64
# split by batch across 1/2/4/8 GPUs"); every other config runs one batch per rank (weak)
STRONG_BATCH = {"cfg4"}
HBM_FALLBACK_GBS = 6548.8  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def metric_of(cfg):
    """BASELINE.json's metric, written for the config it is measured on."""
    return (f"sketched EI operator passes/s at {cfg.N}², {cfg.n_full}→{cfg.m} angles; "
            f"% HBM/gather roofline")


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json's driver-measured copy bandwidth, else the guide's
    fallback."""
    try:
        v = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


def host_cpu():
    """(logical cores, model name) of this host (lscpu's 'Model name' = /proc/cpuinfo)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args):
    """`--gpus N` with N > 1 outside torchrun: re-run this script under torch.distributed.run
    with N ranks (one per GPU), rendezvous on 127.0.0.1; rank 0 prints the JSON line.
    Returns the launcher's exit code, or None when this process is already a rank."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if args.gpus is not None and int(world_env) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}\n")
            return 2
        return None
    if (args.gpus or 1) <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def rank_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("SKEI_BENCH_RANKINFO"):  # launcher test: every rank reports its env
        sys.stderr.write(f"rankinfo rank={rank} local={local} world={world}\n")
        sys.stderr.flush()
    return world, rank, local
# stage boundaries recorded by skei_pass_profiled: 0 start | rotate+pack | 1 | forward x2
# (+ fused MC residual) | 2 | ramp | 3 | backprojection x2 (+ fused EI residual) | 4 | 5 end
STAGES = ["rotate_pack", "radon_fwd_x2", "ramp", "radon_adj_x2"]
LAUNCHES_PER_STEP = 5  # draw, rotate+pack, forward (2 jobs + MC), ramp, adjoint (2 jobs + EI)
E2E_SLOTS = 3  # e2e pipeline depth (slots of device buffers and streams)
E2E_REPS = 3  # e2e: repetitions of the K timed steps (the median is reported)
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (one per GPU); default: WORLD_SIZE under torchrun, else 1")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="skei", choices=["skei", "reference"])
    ap.add_argument("--config", default="cfg3", choices=list(synth.CONFIGS))
    ap.add_argument("--mode", default="uniform", choices=["uniform", "interleaved"])
    ap.add_argument("--split", default="batch", choices=["batch", "angle", "angle-ag", "angle-p2p", "angle-rs"],
                    help="batch: every rank runs its own batch (weak scaling, no collective); "
                         "angle: one batch, the sketch's angles split over the ranks with one "
                         "NCCL all-reduce of the partial backprojections (strong scaling, "
                         "BASELINE cfg5); angle-ag: the same split exchanging filtered "
                         "sinogram rows by all-gather, row-band backprojection (SURVEY 8(f) #2); "
                         "angle-p2p: the same with the exchange fused into the ramp kernel "
                         "(P2P stores into symmetric memory, no NCCL on the data path); "
                         "angle-rs: each rank backprojects its own angles and the "
                         "backprojector's epilogue stores every partial row into its band "
                         "owner's slot (reduce-scatter fused into the kernel, SURVEY 8(f) #2 (b))")
    ap.add_argument("--path", default="pass", choices=["pass", "ei-grad", "rei", "deviation"],
                    help="pass: the sketched-EI operator pass (the headline); ei-grad: the next "
                         "row, the EI branch's gradient T_g^T (I - M) 2 (x2 - x3) (skei_ei_grad); "
                         "rei: the REI pass, q = ramp(p2 + sigma eps) (skei_pass_rei)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-grad", action="store_true",
                    help="the e2e leg also reads the MC gradient back every step (D2H of B N^2 "
                         "fp32, besides mc / ei)")
    return ap.parse_args()


def workload_desc(cfg, mode):
    return {
        "workload": f"{cfg.name}: {cfg.N}x{cfg.N} fp32 batch {cfg.B}, {cfg.n_full} angles, "
                    f"{cfg.n_det} bins, sketch m={cfg.m} ({mode}), ramp FFT P={cfg.fft_len}, "
                    f"{'per-image' if cfg.per_image_draws else 'per-pass shared'} draws",
        "phantom": f"{cfg.K} random ellipses ({cfg.phantom}), seeded",
        "noise": f"sigma = {cfg.noise} max|y| Gaussian",
        "images_per_gpu": cfg.B,
        "l2": "flushed (256 MB write) before every timed step",
        "launch": "one CUDA graph per step (draw + 4 pass kernels), replayed on the timed stream",
    }


# ------------------------------------------------------------------ work counts
def taps_per_pass(cfg):
    """SURVEY §8(d)/App. A.6: taps = B (4 N^2 + 8 m N^2) (rotate 4/px; 2 fwd + 2 adj, 2 taps
    per (pixel, angle))."""
    return cfg.B * (4 * cfg.N ** 2 + 8 * cfg.m * cfg.N ** 2)


def hbm_bytes_per_pass(cfg):
    """Compulsory HBM bytes of the C-ABI call sequence: B (32 N^2 + 36 m n_det) (App. A.6)."""
    return cfg.B * (32 * cfg.N ** 2 + 36 * cfg.m * cfg.n_det)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle legs
def oracle_draws(cfg, mode, seed, it):
    """The pass's draws as the oracle computes them: one shared (g, S), or one per image
    (cfg4), keyed by the global image index."""
    import oracle
    md = 1 if mode == "uniform" else 0
    if cfg.per_image_draws:
        return [oracle.draw(seed, it, b, cfg.n_full, cfg.m, md) for b in range(cfg.B)]
    return [oracle.draw(seed, it, oracle.SHARED_IMAGE, cfg.n_full, cfg.m, md)] * cfg.B


def oracle_pass_batch(cfg, x1, y, draws, threads):
    """One whole pass of the batch through the fp64 oracle as it stands (oracle.c via
    ctypes, which releases the GIL): images in turn (threads = 1) or spread over `threads`
    host threads."""
    import oracle

    def one(b):
        g, idx = draws[b]
        oracle.sketched_pass(x1[b], y[b], g, idx, cfg.n_full)

    if threads <= 1:
        for b in range(cfg.B):
            one(b)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(cfg.B)))


def cpu_baseline_legs(cfg, mode, seed, seconds):
    """SURVEY §8(d)'s CPU baseline: the oracle timed on this host's cores on whole passes of
    the workload's batch, (i) single-threaded (a bounded sample of images if one pass would
    exceed `seconds`) and (ii) one thread per logical core over the images.  Returns the
    cpu_baseline object (value = the all-cores leg)."""
    cores, model = host_cpu()
    x1, y = synth.make_workload(cfg, seed)
    draws = oracle_draws(cfg, mode, seed, 0)
    import oracle
    t0, n = time.perf_counter(), 0
    while True:  # (i) single thread, image by image
        g, idx = draws[n % cfg.B]
        oracle.sketched_pass(x1[n % cfg.B], y[n % cfg.B], g, idx, cfg.n_full)
        n += 1
        el = time.perf_counter() - t0
        if n >= cfg.B or el >= seconds or el / n * (n + 1) > 1.5 * seconds:
            break
    single = (n / cfg.B) / el
    threads = min(cores, cfg.B)
    t0, npass = time.perf_counter(), 0
    while True:  # (ii) whole passes, images spread over the host's cores
        oracle_pass_batch(cfg, x1, y, draws, threads)
        npass += 1
        el2 = time.perf_counter() - t0
        if el2 >= 0.5 * seconds or npass >= 3:
            break
    return {"value": npass / el2, "unit": UNIT, "cores": threads, "kind": "oracle",
            "host_cores": cores, "cpu_model": model,
            "single_core": {"value": single, "unit": UNIT, "cores": 1,
                            "sample": f"{n} image(s) of the batch, one at a time ({el:.1f} s)"},
            "sample": f"{npass} whole {cfg.name} pass(es) ({cfg.B} images each) through the fp64 "
                      f"oracle, one host thread per image up to {threads} threads ({el2:.1f} s); "
                      f"the oracle's ramp is its direct O(n_det^2) convolution"}


def run_reference(args):
    """--impl reference: the fp64 oracle as it stands on this host's cores, every step one
    whole pass of the config's batch (its images spread over one thread per core); rank 0
    only under torchrun (the other ranks exit 0 without work)."""
    world, rank, _ = rank_env()
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    cores, model = host_cpu()
    threads = min(cores, cfg.B)
    x1, y = synth.make_workload(cfg, args.seed)
    times = []
    for i in range(args.warmup + args.steps):
        draws = oracle_draws(cfg, args.mode, args.seed, i)
        t0 = time.perf_counter()
        oracle_pass_batch(cfg, x1, y, draws, threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = float(np.mean(times)) * 1e3
    value = 1e3 / ms
    line = {
        "impl": "reference", "metric": metric_of(cfg), "value": value, "unit": UNIT,
        "n_gpus": args.gpus or world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if cfg.name in STRONG_BATCH else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": workload_desc(cfg, args.mode),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "host_cores": cores, "cpu_model": model,
                         "sample": f"every step = one whole {cfg.name} pass ({cfg.B} images, fresh "
                                   f"draw per step) through the fp64 oracle, {threads} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def run_angle(args):
    """--split angle: one batch (default cfg5, a single 1024^2 image), its m sketch angles
    split over the ranks (dist.angle_split_pass); one all_reduce(SUM) of [x_fbp | grad | mc]
    per step over NCCL.  Strong scaling: value = passes/s of the whole job."""
    import torch
    import torch.distributed as dist

    import paper_2411_05771_b200 as sk
    from paper_2411_05771_b200 import dist as skdist

    world, rank, local = rank_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[args.config]
    mode = sk.MODE_UNIFORM if args.mode == "uniform" else sk.MODE_INTERLEAVED
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len, device=local)
    x1_np, y_np = synth.make_workload(cfg, args.seed)
    x1 = torch.from_numpy(x1_np).to(dev)
    y = torch.from_numpy(y_np).to(dev)
    ops = skdist.CudaOps(plan)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    split_fn = {"angle-ag": skdist.angle_split_pass_allgather,
                "angle-p2p": skdist.angle_split_pass_p2p,
                "angle-rs": skdist.angle_split_pass_rs}.get(args.split, skdist.angle_split_pass)

    # the P2P splits' symmetric-memory buffers are allocated (and rendezvoused) once, outside
    # the timed loop
    p2p = (skdist.P2PBuffers(cfg.B, cfg.m, cfg.n_det, dev) if args.split == "angle-p2p" else
           skdist.RSBuffers(cfg.B, cfg.N, dev) if args.split == "angle-rs" else None)

    def step(it):
        g, idx = sk.draw_device(args.seed, it, 0, 1, True, cfg.n_full, cfg.m, mode)
        if p2p is not None:
            return split_fn(ops, x1, y, g, idx[0], bufs=p2p)
        return split_fn(ops, x1, y, g, idx[0])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            a, b = mk(), mk()
            a.record()
            out = step(args.warmup + i)
            b.record()
            times.append((a, b))
        torch.cuda.synchronize()
    total_ms = float(sum(a.elapsed_time(b) for a, b in times))
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    if rank == 0:
        line = {
            "metric": f"sketched EI operator passes/s, {cfg.name} ({cfg.N}^2, {cfg.n_full}->{cfg.m} "
                      f"angles) split by angle", "value": args.steps / (total_ms * 1e-3),
            "unit": "passes/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload_desc(cfg, args.mode),
                       "parallelism": f"angle split x{world}" + {
                           "angle-ag": " (NCCL all-gather of filtered rows, row-band backprojection)",
                           "angle-p2p": " (filtered rows stored to every rank by the ramp kernel "
                                        "over NVLink P2P, row-band backprojection)",
                           "angle-rs": " (partial backprojection rows stored to their band owner "
                                       "by the backprojector over NVLink P2P, fixed-order band "
                                       "sum)"}.get(args.split, ""),
                       **({"allgather_bytes": int(out["allgather_bytes"])} if args.split == "angle-ag"
                          else {"p2p_bytes": int(out["p2p_bytes"])} if args.split == "angle-p2p"
                          else {"rs_bytes_per_gpu": int(out["rs_bytes"])} if args.split == "angle-rs"
                          else {"allreduce_bytes": int(out["allreduce_bytes"])}),
                       "launch": "direct (not graphed): library calls + NCCL collectives"},
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ei_grad(args):
    """--path ei-grad (one GPU): skei_ei_grad on a cfg3 batch whose x2 and
    x_fbp come from one pass; one CUDA graph per step (5 launches), L2 flushed before every
    timed step, CUDA events.  The oracle (oracle.ei_grad, fp64, 1 core) is timed on a
    bounded sample of images."""
    if rank_env()[1] != 0:  # a one-GPU diagnostic: only rank 0 runs it
        return 0
    import torch

    import paper_2411_05771_b200 as sk

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    B, m, N = cfg.B, cfg.m, cfg.N
    plan = sk.Plan.get(N, cfg.n_det, cfg.n_full, cfg.fft_len, device=0)
    x1_np, y_np = synth.make_workload(cfg, args.seed)
    x1, y = torch.from_numpy(x1_np).to(dev), torch.from_numpy(y_np).to(dev)
    g, idx = sk.draw_device(args.seed, 0, 0, 1, True, cfg.n_full, m)
    out = sk.sketched_pass(plan, x1, y, g, idx)
    ws = plan.workspace(B, m)
    grad = torch.empty_like(x1)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    cap = torch.cuda.Stream(dev)
    gr = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(gr, stream=cap):
        sk.ei_grad(plan, out["x2"], out["xfbp"], g, idx, out=grad, ws=ws)
    for _ in range(args.warmup):
        gr.replay()
    torch.cuda.synchronize()
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    recs = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = mk(), mk()
            a.record(stream)
            gr.replay()
            b.record(stream)
            recs.append((a, b))
        torch.cuda.synchronize()
    ms = float(sum(a.elapsed_time(b) for a, b in recs))
    import oracle
    og, oidx = int(g[0]), idx[0].cpu().numpy()
    t0, n_img = time.perf_counter(), 0
    while time.perf_counter() - t0 < min(args.cpu_seconds, 20.0) or n_img == 0:
        oracle.ei_grad(x1_np[n_img % B], og, oidx, cfg.n_full, cfg.n_det)
        n_img += 1
    cpu_s = time.perf_counter() - t0
    taps = B * (4 * N * N + 4 * m * N * N)  # T^T 4/px; A_S d and A_S^T q: 2 taps per (px, angle)
    props = torch.cuda.get_device_properties(dev)
    peak_gbs = props.multi_processor_count * 128 * (clk.summary()["sm_max_mhz"] or 1965) * 1e6 / 1e9
    line = {
        "metric": f"EI-branch gradients/s (batches of {B}) at {N}², {cfg.n_full}→{m} angles",
        "value": args.steps / (ms * 1e-3), "unit": "gradients/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {**workload_desc(cfg, args.mode),
                                        "launch": "one CUDA graph per step (5 launches)",
                                        "path": "skei_ei_grad (SURVEY 8(f) #1)"},
        "roofline": {"bound": "smem", "unit": "GB/s", "taps_per_step": taps,
                     "achieved": 4 * taps * args.steps / (ms * 1e-3) / 1e9,
                     "peak": peak_gbs, "frac": 4 * taps * args.steps / (ms * 1e-3) / 1e9 / peak_gbs,
                     "algorithmic": "4 B per tap; T_g^T 4 taps/px, A_S d and A_S^T q 2 taps per "
                                    "(px, angle)",
                     "peak_source": "148 SMs x 128 B/clk x SM max clock (theoretical shared-memory "
                                    "bandwidth; the pass bench's live probe measures 99.6% of it)"},
        "cpu_baseline": {"value": (n_img / B) / cpu_s, "unit": "gradients/s", "cores": 1,
                         "kind": "oracle", "sample": f"{n_img} image(s) through oracle.ei_grad "
                                                     f"({cpu_s:.1f} s; {B} images = 1 gradient)"},
        "gpu_launches": 5 * args.steps, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_rei(args):
    """--path rei (one GPU): skei_pass_rei on the cfg3 batch, sigma = 0.005
    max|y| (the config's noise level), fresh draw and noise stream every step (graphed per
    step: draw + 6 launches), L2 flushed before every timed step, CUDA events; oracle REI
    pass timed beside it on a bounded sample."""
    if rank_env()[1] != 0:  # a one-GPU diagnostic: only rank 0 runs it
        return 0
    import torch

    import paper_2411_05771_b200 as sk

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    B, m = cfg.B, cfg.m
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len, device=0)
    x1_np, y_np = synth.make_workload(cfg, args.seed)
    x1, y = torch.from_numpy(x1_np).to(dev), torch.from_numpy(y_np).to(dev)
    sigma = cfg.noise * float(np.abs(y_np).max())
    out = sk.alloc_pass_outputs(plan, B, m, dev)
    ws = plan.workspace(B, m)
    gbuf = torch.empty(1, dtype=torch.int32, device=dev)
    ibuf = torch.empty(1, m, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    cap = torch.cuda.Stream(dev)
    n = args.warmup + args.steps
    graphs = []
    torch.cuda.synchronize()
    for it in range(n):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cap):
            sk.draw_device(args.seed, it, 0, 1, True, cfg.n_full, m, sk.MODE_UNIFORM, g=gbuf, idx=ibuf)
            sk.sketched_pass_rei(plan, x1, y, gbuf, ibuf, sigma, args.seed, it, 0, out=out, ws=ws)
        graphs.append(gr)
    for i in range(args.warmup):
        graphs[i].replay()
    torch.cuda.synchronize()
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    recs = []
    with ClockSampler(0) as clk:
        for i in range(args.steps):
            flush.zero_()
            a, b = mk(), mk()
            a.record(stream)
            graphs[args.warmup + i].replay()
            b.record(stream)
            recs.append((a, b))
        torch.cuda.synchronize()
    ms = float(sum(a.elapsed_time(b) for a, b in recs))
    import oracle
    og, oidx = oracle.draw(args.seed, 0, oracle.SHARED_IMAGE, cfg.n_full, m)
    t0, n_img = time.perf_counter(), 0
    while time.perf_counter() - t0 < min(args.cpu_seconds, 20.0) or n_img == 0:
        oracle.sketched_pass_rei(x1_np[n_img % B], y_np[n_img % B], og, oidx, cfg.n_full, sigma,
                                 args.seed, 0, n_img % B)
        n_img += 1
    cpu_s = time.perf_counter() - t0
    line = {
        "metric": f"REI sketched-EI operator passes/s at {cfg.N}², {cfg.n_full}→{m} angles",
        "value": args.steps / (ms * 1e-3), "unit": "passes/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {**workload_desc(cfg, args.mode), "path": "skei_pass_rei (SURVEY 8(f) #3)",
                   "rei_sigma": sigma, "launch": "one CUDA graph per step (draw + 6 launches)"},
        "cpu_baseline": {"value": (n_img / B) / cpu_s, "unit": "passes/s", "cores": 1,
                         "kind": "oracle", "sample": f"{n_img} image(s) through the oracle REI pass "
                                                     f"({cpu_s:.1f} s; {B} images = 1 pass)"},
        "gpu_launches": 7 * args.steps, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_deviation(args):
    """--path deviation (one GPU): the Theorem-1 deviation
    ||A^T (S^T S - I) A||_2 at the config's geometry for sketch sizes n_full/8 .. n_full/2
    (interleaved sketches), `--steps` power iterations each from a random start image; the
    timed unit is one power iteration (2 forward projections: all n_full angles and the
    sketch, 2 backprojections, 1 norm), CUDA events, one stream."""
    if rank_env()[1] != 0:  # a one-GPU diagnostic: only rank 0 runs it
        return 0
    import torch

    import paper_2411_05771_b200 as sk

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len, device=0)
    v0 = torch.from_numpy(np.random.default_rng(args.seed).standard_normal(
        (1, cfg.N, cfg.N)).astype(np.float32)).to(dev)
    ws = plan.workspace(1, cfg.n_full)
    table, ms_it = {}, None
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    with ClockSampler(0) as clk:
        for div in (8, 4, 2):
            m = cfg.n_full // div
            _, idx = sk.draw(args.seed, 0, sk.SHARED_IMAGE, cfg.n_full, m, sk.MODE_INTERLEAVED)
            it = torch.tensor(idx, dtype=torch.int32, device=dev)
            sk.sketch_deviation(plan, it, v0.clone(), args.warmup, ws=ws)
            a, b = mk(), mk()
            v = v0.clone()
            a.record()
            lam = sk.sketch_deviation(plan, it, v, args.steps, ws=ws)
            b.record()
            torch.cuda.synchronize()
            table[str(m)] = float(lam[0])
            if m == cfg.m:
                ms_it = a.elapsed_time(b) / args.steps
    line = {
        "metric": f"Theorem-1 deviation power iterations/s at {cfg.N}², {cfg.n_full} angles, m={cfg.m}",
        "value": 1e3 / ms_it if ms_it else None, "unit": "iterations/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_it,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{cfg.name} geometry: {cfg.N}x{cfg.N}, "
                                                    f"{cfg.n_full} angles, {cfg.n_det} bins, one "
                                                    "random start image, interleaved sketches",
                                        "l2": "not flushed (iterative: each iteration reads the "
                                              "previous one's output)",
                                        "launch": "direct, 8 launches per iteration",
                                        "path": "skei_sketch_deviation (SURVEY 8(f) #4)"},
        "delta_by_m": table, "gpu_launches": 8 * args.steps, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    rc = launch_ranks(args)
    if rc is not None:
        return rc
    if args.path == "deviation":
        return run_deviation(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.path == "ei-grad":
        return run_ei_grad(args)
    if args.path == "rei":
        return run_rei(args)
    if args.split in ("angle", "angle-ag", "angle-p2p", "angle-rs"):
        if args.config == "cfg3" and "--config" not in sys.argv:
            args.config = "cfg5"
        return run_angle(args)

    import torch
    import torch.distributed as dist

    import paper_2411_05771_b200 as sk

    world, rank, local = rank_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = synth.CONFIGS[args.config]
    mode = sk.MODE_UNIFORM if args.mode == "uniform" else sk.MODE_INTERLEAVED
    shared = not cfg.per_image_draws
    m, N = cfg.m, cfg.N
    # this rank's images (global indices): a share of the config's batch (strong scaling,
    # cfg4) or a whole batch of its own (weak scaling, rank r: images r B ... r B + B - 1)
    strong = cfg.name in STRONG_BATCH
    from paper_2411_05771_b200.dist import batch_range
    images = batch_range(cfg.B, rank, world) if strong else range(rank * cfg.B, (rank + 1) * cfg.B)
    B, img0 = len(images), images.start
    lcfg = dataclasses.replace(cfg, B=B)  # the work one rank does per step
    plan = sk.Plan.get(N, cfg.n_det, cfg.n_full, cfg.fft_len, device=local)

    # inputs: this rank's images, resident in HBM
    x1_np, y_np = synth.make_workload(cfg, args.seed, images=images)
    x1 = torch.from_numpy(x1_np).to(dev)
    y = torch.from_numpy(y_np).to(dev)
    out = sk.alloc_pass_outputs(plan, B, m, dev)
    ws = plan.workspace(B, m)
    gbuf = torch.empty(1 if shared else B, dtype=torch.int32, device=dev)
    ibuf = torch.empty(1 if shared else B, m, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(it, events, fused=True):
        if fused:  # the timed form: one call, the draw overlapped with packing x1
            sk.sketched_pass_draw(plan, x1, y, args.seed, it, m, mode, shared, img0, g=gbuf,
                                  idx=ibuf, out=out, ws=ws, events=events)
            return
        sk.draw_device(args.seed, it, img0, 1 if shared else B, shared, cfg.n_full, m, mode,
                       g=gbuf, idx=ibuf)
        sk.sketched_pass_profiled(plan, x1, y, gbuf, ibuf, events, out, ws)

    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def mk_created():
        e = mk()
        e.record(stream)  # creates the cudaEvent_t outside any capture
        return e

    # Every step (draw a1 + pass a2..a8: 5 kernels) is captured once into its own CUDA graph
    # (the draw's iteration index is a kernel argument).  The timed graphs carry only the two
    # event-record nodes around the dominant kernel (the forward projector: its duration is
    # measured live in the timed region); a second set of graphs with every stage boundary
    # gives the stage breakdown, replayed after the timed region (untimed).
    n_iter = args.warmup + args.steps
    n_brk = min(10, args.steps)
    fwd_events = [[None, mk_created(), mk_created(), None, None, None] for _ in range(n_iter)]
    brk_events = [[mk_created() for _ in range(6)] for _ in range(n_brk)]
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)

    def capture(it, events, fused=True):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cap):
            step(it, events, fused)
        return gr

    # pass index of step i: the same on every rank for a split batch (one pass of the whole
    # batch), distinct per rank for independent batches
    def pass_it(i):
        return i if strong else i * world + rank

    graphs = [capture(pass_it(i), fwd_events[i]) for i in range(n_iter)]
    # the breakdown graphs launch the draw and the pass separately (each stage alone)
    brk_graphs = [capture(pass_it(n_iter + i), brk_events[i], False) for i in range(n_brk)]
    torch.cuda.synchronize()
    for i in range(args.warmup):
        graphs[i].replay()
    torch.cuda.synchronize()

    # shared-memory bandwidth probe (roofline denominator of the gather kernels)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.empty(2 * nsm, device=dev)
    sk.smem_probe(2 * nsm, 50, sink)
    e0, e1 = mk(), mk()
    e0.record()
    sk.smem_probe(2 * nsm, 1000, sink)
    e1.record()
    torch.cuda.synchronize()
    probe_gbs = 2 * nsm * 1024 * 16 * 32 * 1000 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    # L2 read bandwidth probe: the forward re-stages its packed line blocks from
    # L2, so this bounds its TMA traffic (a 32 MB buffer, well under the 126 MB L2)
    l2buf = torch.ones(8 << 20, device=dev)
    sk.l2_probe(l2buf, nsm, 2, sink)
    e0.record()
    sk.l2_probe(l2buf, nsm, 10, sink)
    e1.record()
    torch.cuda.synchronize()
    l2_gbs = nsm * l2buf.numel() * 4 * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del l2buf

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    recs = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev_start, ev_end = mk(), mk()
            ev_start.record(stream)
            graphs[args.warmup + i].replay()
            ev_end.record(stream)
            recs.append((ev_start, fwd_events[args.warmup + i], ev_end))
        torch.cuda.synchronize()
    step_ms = np.array([a.elapsed_time(c) for a, _, c in recs])
    fwd_ms = np.array([evs[1].elapsed_time(evs[2]) for _, evs, _ in recs])
    if os.environ.get("SKEI_BENCH_DUMP"):  # diagnostics: per-step forward times
        sys.stderr.write("fwd_us " + " ".join(f"{v * 1e3:.0f}" for v in fwd_ms) + "\n")
    total_ms = float(step_ms.sum())
    # stage breakdown (untimed replays of the fully instrumented graphs)
    brk = []
    for i in range(n_brk):
        flush.zero_()
        e0 = mk()
        e0.record(stream)
        brk_graphs[i].replay()
        brk.append(e0)
    torch.cuda.synchronize()
    stage_ms = np.array([[evs[j].elapsed_time(evs[j + 1]) for j in range(4)] for evs in brk_events])
    draw_ms = np.array([e0.elapsed_time(evs[0]) for e0, evs in zip(brk, brk_events)])
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    passes_per_step = 1 if strong else world  # whole passes the job completes per step
    value = passes_per_step * args.steps / (total_ms * 1e-3)
    # up to 10 windows of consecutive timed steps (this rank's times)
    wins = [w for w in np.array_split(step_ms, min(10, args.steps)) if len(w)]
    win_vals = [passes_per_step * len(w) / (w.sum() * 1e-3) for w in wins]

    # ---- end to end through the public host-buffer call (skei_pass_host).  E2E_SLOTS slots
    # (device inputs/outputs, workspace, pinned draw/staging/result buffers, stream) rotate, so
    # step i's host preparation and H2D overlap the passes of steps i-1, i-2 on the SMs — what
    # a user streaming batches through the library does (with two slots, a slot's next host
    # gather + H2D could only start once its previous pass ended, idling the SMs).  Every step still copies its own inputs
    # from pinned host memory, runs the whole pass and reads its mc/ei back; the L2 is
    # flushed in-stream before every step; the clock is the host wall clock over all steps.
    e2e = None
    if not args.no_e2e:
        hx1 = torch.from_numpy(x1_np).pin_memory()
        hy = torch.from_numpy(y_np).pin_memory()
        ng = 1 if shared else B
        slots = []
        for _ in range(E2E_SLOTS):
            d = sk.alloc_pass_outputs(plan, B, m, dev)
            d.update(x1=torch.empty_like(x1), y=torch.empty_like(y), g=torch.empty_like(gbuf),
                     idx=torch.empty_like(ibuf))
            slots.append(dict(d=d, ws=plan.workspace(B, m), st=torch.cuda.Stream(dev),
                              hg=torch.empty(ng, dtype=torch.int32).pin_memory(),
                              hidx=torch.empty(ng, m, dtype=torch.int32).pin_memory(),
                              hmc=torch.empty(B).pin_memory(), hei=torch.empty(B).pin_memory(),
                              ys=torch.empty(B, m, cfg.n_det).pin_memory(),
                              hgrad=torch.empty(B, N, N).pin_memory() if args.e2e_grad else None,
                              done=None, fl=torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)))
        results = []

        def e2e_step(it):
            sl = slots[it % E2E_SLOTS]
            if sl["done"] is not None:  # this slot's previous step: its results are back
                sl["done"].synchronize()
                results.append(float(sl["hmc"][0]))
            for b in range(ng):  # host draw (skei_draw)
                gi, ii = sk.draw(args.seed, it, sk.SHARED_IMAGE if shared else img0 + b,
                                 cfg.n_full, m, mode)
                sl["hg"][b] = gi
                sl["hidx"][b] = torch.tensor(ii, dtype=torch.int32)
            with torch.cuda.stream(sl["st"]):
                sk.sketched_pass_host(plan, hx1, hy, sl["hg"], sl["hidx"], sl["d"], sl["hmc"],
                                      sl["hei"], sl["ws"], sl["fl"], h_ystage=sl["ys"])
                if sl["hgrad"] is not None:  # the MC gradient back to the host as well
                    sl["hgrad"].copy_(sl["d"]["grad"], non_blocking=True)
                # L2 flush behind the pass in the same stream (so it never holds up the next
                # step's H2D on the other stream): this slot's next pass starts cold
                sl["fl"].zero_()
                ev = torch.cuda.Event()
                ev.record(sl["st"])
            sl["done"] = ev

        for i in range(2 * E2E_SLOTS):
            e2e_step(i)
        torch.cuda.synchronize()
        for sl in slots:
            sl["done"] = None
        # E2E_REPS back-to-back repetitions of the K steps, each timed on its own (max over
        # ranks); the line reports the median repetition — the host wall clock of one
        # repetition is exposed to host scheduling hiccups of the box
        reps = []
        for rep in range(E2E_REPS):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for i in range(args.steps):
                e2e_step(1000 + rep * args.steps + i)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([el], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t.item())
            reps.append(el)
        el = float(np.median(reps))
        # only each image's m sketched rows of y cross the link (skei_pass_host: pitched copy or gather)
        y_h2d = B * m * cfg.n_det * 4
        h2d = hx1.numel() * 4 + y_h2d + ng * 4 + ng * m * 4
        d2h = 2 * B * 4 + (B * N * N * 4 if args.e2e_grad else 0)
        e2e = {"value": passes_per_step * args.steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "reps": [passes_per_step * args.steps / r for r in reps],
               "returns": "mc, ei and the MC gradient" if args.e2e_grad else
                          "mc, ei (the gradient and x_fbp stay on the device; --e2e-grad reads "
                          "the gradient back too)",
               "timing": "host wall clock over all steps; per step: host draw, H2D of x1, y_S "
                         "(the sketched rows of y: an equispaced sketch's rows are copied in place "
                         "as a pitched sub-array of y, a random sketch's are gathered into a pinned "
                         "staging buffer by the library; each image's own rows for per-image "
                         "sketches), g, idx "
                         "from pinned memory, the pass, D2H of its results, in-stream L2 flush "
                         "(256 MB write) behind it; slots with their own streams rotate, so one "
                         "step's H2D overlaps the previous steps' passes (3 slots); the median "
                         f"of {E2E_REPS} repetitions of the K steps"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel: the forward projector launch (A_S x1 and A_S x2),
    # its duration measured by the in-graph events of the timed steps
    stage_mean = stage_ms.mean(axis=0)
    sm_max = 1965.0
    peak_theory = nsm * 128 * sm_max * 1e6 / 1e9  # GB/s: 148 SMs x 128 B/clk x 1965 MHz
    peak = max(peak_theory, probe_gbs)
    fwd_taps = 2 * B * 2 * m * N * N      # two projections, 2 taps per (pixel, angle)
    taps = {"radon_fwd_x2": fwd_taps}
    dname = "radon_fwd_x2"
    achieved = 4.0 * fwd_taps / (float(fwd_ms.mean()) * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):  # the capture's per-launch DRAM bytes, for the config it was taken on
        try:
            tj = json.load(open(tf))
            if tj.get("config", "cfg3") == args.config and getattr(args, "mode", None) in (None, "uniform"):
                traffic = tj.get(dname)
        except Exception:
            traffic = None
    hbm_gbs, hbm_src = hbm_peak()
    t_gather = 4.0 * taps_per_pass(lcfg) / (peak * 1e9)
    t_hbm = hbm_bytes_per_pass(lcfg) / (hbm_gbs * 1e9)
    pass_frac = max(t_gather, t_hbm) / (ms_per_step * 1e-3)
    roofline = {
        "bound": "smem", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic,
        "peak_source": f"max(theoretical {nsm} SMs x 128 B/clk x {sm_max:.0f} MHz = {peak_theory:.0f}, "
                       f"live LDS.128 probe = {probe_gbs:.0f}) GB/s; MEASURED_PEAKS.json has no shared-memory figure",
        "algorithmic": f"4 B per tap, {taps[dname]:.4g} taps per launch "
                       f"(2 jobs x {B} images x {m} angles x {N}^2 px x 2 taps)",
        "kernel_ms": float(fwd_ms.mean()),
        "l2_probe_gbs": l2_gbs,
        "pass_frac": pass_frac,
        "pass_roofline": f"max(T_gather = 4 B x {taps_per_pass(lcfg):.4g} taps / peak, T_hbm = "
                         f"{hbm_bytes_per_pass(lcfg):.4g} B / {hbm_gbs:g} GB/s ({hbm_src})) / "
                         f"measured step time (one rank's {B} images)",
    }

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_legs(cfg, args.mode, args.seed, args.cpu_seconds)

    desc = workload_desc(cfg, args.mode)
    desc["images_per_gpu"] = B
    if world > 1 or strong:
        desc["parallelism"] = (f"batch split x{world}: {cfg.B} images, {B} per rank, draws keyed "
                               f"by the global image index, no data-path collective" if strong else
                               f"batch x{world}: every rank its own {cfg.B}-image batch, no "
                               f"data-path collective")
    line = {
        "metric": metric_of(cfg), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": desc,
        "windows": {"n": len(win_vals), "median": float(np.median(win_vals)),
                    "min": float(np.min(win_vals)), "max": float(np.max(win_vals)),
                    "unit": UNIT, "rank": "rank 0's step times"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": LAUNCHES_PER_STEP * args.steps,
        "clocks": clk.summary(),
        "stages_ms": {**{"draw": float(draw_ms.mean())},
                      **{s: float(v) for s, v in zip(STAGES, stage_mean)}},
        "images_per_s": value * (cfg.B if strong else B),
        "taps_per_s": taps_per_pass(cfg) * value,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
