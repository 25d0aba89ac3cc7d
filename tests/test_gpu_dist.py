"""GPU checks of the angle-split partials (paper_2411_05771_b200.dist) on one GPU: the
shards' partial FBP (density scale of the full sketch), partial MC gradient and partial mc,
summed in rank order, equal the single-GPU pass within the north_star tolerance.  (Only
one GPU is available to this build; the NCCL all-reduce itself is exercised by the gloo
tests on CPU and by bench.py --split angle under torchrun.)"""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_05771_b200 as sk
import synth
from paper_2411_05771_b200 import dist as skdist

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _close(got, ref, name):
    got = got.double().cpu().numpy() if torch.is_tensor(got) else np.asarray(got, np.float64)
    ref = ref.double().cpu().numpy() if torch.is_tensor(ref) else np.asarray(ref, np.float64)
    err = np.abs(got - ref).max()
    assert err <= TOL * np.abs(ref).max(), f"{name}: {err:.3e} vs {np.abs(ref).max():.3e}"


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg5", 4), ("cfg5", 8)])
def test_angle_shard_partials_sum_to_full_pass(name, world):
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    full = sk.sketched_pass(plan, x1, y, g, idx)
    ops = skdist.CudaOps(plan)
    x2 = ops.rotate(x1, g)
    xfbp = torch.zeros_like(x1)
    grad = torch.zeros_like(x1)
    mc = torch.zeros(cfg.B, device="cuda")
    idx_h = idx[0].cpu()
    for r in range(world):
        sub = skdist.angle_shard(idx_h, r, world).cuda()
        p1 = ops.forward(x1, sub)
        p2 = ops.forward(x2, sub)
        mcr, rr = ops.residual(p1, y, sub)
        xfbp += ops.fbp(p2, sub, cfg.m)
        grad += ops.adjoint(rr, sub, 2.0)
        mc += mcr
    _close(xfbp, full["xfbp"], "xfbp")
    _close(grad, full["grad"], "grad")
    _close(mc, full["mc"], "mc")
    ei = ops.ei(x2, xfbp, idx)
    _close(ei, full["ei"], "ei")
    # and against the oracle for the first image (sampled rows of x_fbp, all of mc)
    og, oidx = oracle.draw(0, 0, oracle.SHARED_IMAGE, cfg.n_full, cfg.m)
    ref = oracle.sketched_pass(x1n[0], yn[0], og, oidx, cfg.n_full)
    _close(xfbp[0], ref["xfbp"], "xfbp vs oracle")
    _close(mc[0:1], np.array([ref["mc"]]), "mc vs oracle")


def test_angle_split_pass_single_rank_equals_pass():
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    out = skdist.angle_split_pass(skdist.CudaOps(plan), x1, y, g, idx[0])
    full = sk.sketched_pass(plan, x1, y, g, idx)
    for k in ("x2", "xfbp", "grad", "mc", "ei"):
        _close(out[k], full[k], k)


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg2", 3), ("cfg5", 4), ("cfg5", 8)])
def test_allgather_split_bands_tile_full_pass(name, world):
    """SURVEY §8(f) #2 (a) simulated on one GPU: every 'rank' projects, filters and computes
    the residual of its angle shard (shard_phase); the shards' q and r rows, concatenated in
    rank order (what the all-gather delivers), are backprojected by every rank for its row
    band (band_phase, skei_backproject_band).  The bands tile x_fbp and grad of the
    single-GPU pass; the mc and ei partials sum to its mc and ei."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    full = sk.sketched_pass(plan, x1, y, g, idx)
    ops = skdist.CudaOps(plan)
    idx_h = idx[0].cpu()
    shards = [skdist.shard_phase(ops, x1, y, g, idx_h.cuda(), r, world) for r in range(world)]
    q = torch.cat([s["q"] for s in shards], dim=1).contiguous()
    r = torch.cat([s["r"] for s in shards], dim=1).contiguous()
    bands = [skdist.band_phase(ops, q, r, idx, shards[0]["x2"], rk, world) for rk in range(world)]
    assert [b["rows"].start for b in bands] == sorted(b["rows"].start for b in bands)
    _close(torch.cat([b["xfbp"] for b in bands], dim=1), full["xfbp"], "xfbp bands")
    _close(torch.cat([b["grad"] for b in bands], dim=1), full["grad"], "grad bands")
    _close(sum(s["mc"] for s in shards), full["mc"], "mc")
    _close(sum(b["ei"] for b in bands), full["ei"], "ei")


def test_allgather_split_single_rank_equals_pass():
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    out = skdist.angle_split_pass_allgather(skdist.CudaOps(plan), x1, y, g, idx[0])
    full = sk.sketched_pass(plan, x1, y, g, idx)
    for k in ("x2", "xfbp", "grad", "mc", "ei"):
        _close(out[k], full[k], k)


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg2", 3), ("cfg5", 4), ("cfg5", 8)])
def test_p2p_fused_allgather_split_tiles_full_pass(name, world):
    """SURVEY §8(f) #2 with the exchange fused into the ramp kernel (P2P stores into every
    rank's buffers), simulated on one GPU with `world` virtual ranks and real pointer lists:
    every rank's buffers end up holding the whole q and r (identical to one ramp of the
    full sketch), and the row bands tile x_fbp and grad of the single-GPU pass."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    full = sk.sketched_pass(plan, x1, y, g, idx)
    out = skdist.simulate_p2p_split(skdist.CudaOps(plan), x1, y, g, idx[0], world)
    for b in out["bufs"]:
        _close(b[0], full["q"], "q in every rank's buffer")
        _close(b[1], full["r"], "r in every rank's buffer")
        assert torch.equal(b[0], out["bufs"][0][0]) and torch.equal(b[1], out["bufs"][0][1])
    bands = out["bands"]
    _close(torch.cat([bd["xfbp"] for bd in bands], dim=1), full["xfbp"], "xfbp bands")
    _close(torch.cat([bd["grad"] for bd in bands], dim=1), full["grad"], "grad bands")
    _close(out["mc"], full["mc"], "mc")
    _close(sum(bd["ei"] for bd in bands), full["ei"], "ei")


def test_p2p_split_single_rank_equals_pass():
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    out = skdist.angle_split_pass_p2p(skdist.CudaOps(plan), x1, y, g, idx[0])
    full = sk.sketched_pass(plan, x1, y, g, idx)
    for k in ("x2", "xfbp", "grad", "mc", "ei"):
        _close(out[k], full[k], k)
