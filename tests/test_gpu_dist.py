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


def _oracle_images(cfg, x1n, yn):
    """The oracle's pass (fp64) for the images it checks: the first and last of the batch
    (cfg2), the single image of cfg5 (same draw as the device's)."""
    og, oidx = oracle.draw(0, 0, oracle.SHARED_IMAGE, cfg.n_full, cfg.m)
    images = sorted({0, cfg.B - 1})
    return {b: oracle.sketched_pass(x1n[b], yn[b], og, oidx, cfg.n_full) for b in images}


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
    # and against the oracle directly: the shard partials summed in rank order are the
    # oracle's full-sketch x_fbp, MC gradient, mc and ei (the partition identity)
    for b, ref in _oracle_images(cfg, x1n, yn).items():
        _close(xfbp[b], ref["xfbp"], f"xfbp[{b}] vs oracle")
        _close(grad[b], ref["grad"], f"grad[{b}] vs oracle")
        _close(mc[b:b + 1], np.array([ref["mc"]]), f"mc[{b}] vs oracle")
        _close(ei[b:b + 1], np.array([ref["ei"]]), f"ei[{b}] vs oracle")


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
    # the bands tile the oracle's x_fbp and grad, the shards' mc and the bands' ei partials
    # sum to the oracle's (the partition identity)
    _check_split_vs_oracle(cfg, x1n, yn, bands, sum(s["mc"] for s in shards),
                           sum(b["ei"] for b in bands))


def _check_split_vs_oracle(cfg, x1n, yn, bands, mc, ei):
    xf = torch.cat([bd["xfbp"] for bd in bands], dim=1)
    gr = torch.cat([bd["grad"] for bd in bands], dim=1)
    for b, ref in _oracle_images(cfg, x1n, yn).items():
        for bd in bands:
            rows = bd["rows"]
            _close(bd["xfbp"][b], ref["xfbp"][rows.start:rows.stop], f"xfbp band {rows}[{b}] vs oracle")
            _close(bd["grad"][b], ref["grad"][rows.start:rows.stop], f"grad band {rows}[{b}] vs oracle")
        _close(xf[b], ref["xfbp"], f"xfbp[{b}] vs oracle")
        _close(gr[b], ref["grad"], f"grad[{b}] vs oracle")
        _close(mc[b:b + 1], np.array([ref["mc"]]), f"mc[{b}] vs oracle")
        _close(ei[b:b + 1], np.array([ref["ei"]]), f"ei[{b}] vs oracle")


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
    # every rank's gathered q and r against the oracle's ramp of the full sketch and its
    # residual rows; the bands, mc and ei against the oracle's pass
    for b, ref in _oracle_images(cfg, x1n, yn).items():
        for bf in out["bufs"]:
            _close(bf[0][b], ref["q"], f"q[{b}] in a rank's buffer vs oracle")
            _close(bf[1][b], ref["r"], f"r[{b}] in a rank's buffer vs oracle")
    _check_split_vs_oracle(cfg, x1n, yn, bands, out["mc"], sum(bd["ei"] for bd in bands))


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


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg2", 3), ("cfg5", 4), ("cfg5", 8)])
def test_rs_fused_split_bands_tile_full_pass(name, world):
    """the backprojection's reduce-scatter fused into the backprojector
    (every output row stored into its band owner's slot), simulated on one GPU with `world`
    virtual ranks and real pointer lists.  The bands tile x_fbp and grad of the single-GPU
    pass and of the oracle (partition identity of PAPER.md L70 / L92); each band equals its
    slots summed in rank order bit for bit; the slot rows beyond a band are never read."""
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    full = sk.sketched_pass(plan, x1, y, g, idx)
    out = skdist.simulate_rs_split(skdist.CudaOps(plan), x1, y, g, idx[0], world)
    bands = out["bands"]
    for rk, bd in enumerate(bands):
        nrows = len(bd["rows"])
        assert bd["rows"] == skdist.batch_range(cfg.N, rk, world)
        slots = out["bufs"][rk][:, :, :, :nrows]
        assert not torch.isnan(slots).any(), "a slot row of the band was not stored"
        acc = torch.zeros_like(slots[0])
        for s in range(world):  # slot (rank) order, as the reduce kernel
            acc = acc + slots[s]
        assert torch.equal(bd["xfbp"], acc[0]) and torch.equal(bd["grad"], acc[1])
    _close(torch.cat([bd["xfbp"] for bd in bands], dim=1), full["xfbp"], "xfbp bands")
    _close(torch.cat([bd["grad"] for bd in bands], dim=1), full["grad"], "grad bands")
    _close(out["mc"], full["mc"], "mc")
    _close(sum(bd["ei"] for bd in bands), full["ei"], "ei")
    _check_split_vs_oracle(cfg, x1n, yn, bands, out["mc"], sum(bd["ei"] for bd in bands))
    # deterministic: a second run stores and sums the same bits
    again = skdist.simulate_rs_split(skdist.CudaOps(plan), x1, y, g, idx[0], world)
    for a, b in zip(bands, again["bands"]):
        assert torch.equal(a["xfbp"], b["xfbp"]) and torch.equal(a["grad"], b["grad"])
        assert torch.equal(a["ei"], b["ei"])


def test_rs_split_single_rank_equals_pass():
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1n, yn = synth.make_workload(cfg, seed=0)
    x1 = torch.from_numpy(x1n).cuda()
    y = torch.from_numpy(yn).cuda()
    g, idx = sk.draw_device(0, 0, 0, 1, True, cfg.n_full, cfg.m)
    out = skdist.angle_split_pass_rs(skdist.CudaOps(plan), x1, y, g, idx[0])
    full = sk.sketched_pass(plan, x1, y, g, idx)
    for k in ("x2", "xfbp", "grad", "mc", "ei"):
        _close(out[k], full[k], k)


def test_rs_scatter_rejects_bad_arguments():
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    q = torch.zeros(1, 4, cfg.n_det, device="cuda")
    idx = torch.arange(4, dtype=torch.int32, device="cuda")
    buf = torch.zeros(sk.rs_recv_floats(plan, 1, 2), device="cuda")
    with pytest.raises(sk.SkeiError):  # rank outside the world
        sk.backproject_scatter(plan, q, q, idx, 4, [buf.data_ptr()] * 2, 2)
    with pytest.raises(sk.SkeiError):  # more than 8 peers
        sk.backproject_scatter(plan, q, q, idx, 4, [buf.data_ptr()] * 9, 0)
    with pytest.raises(sk.SkeiError):  # m_total < m
        sk.backproject_scatter(plan, q, q, idx, 3, [buf.data_ptr()] * 2, 0)
