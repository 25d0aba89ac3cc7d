"""World-size-2 gloo tests of the multi-GPU partition logic (paper_2411_05771_b200.dist) on
CPU.  The operators are the fp64 oracle's (tests may call oracle/), so these tests check the
partitioning — shard boundaries, density scale of the full sketch, the packed all-reduce,
EI on the reduced x_fbp, batch split by global image index — not the CUDA kernels (the
GPU tests do that)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2411_05771_b200 import dist as skdist


class OracleOps:
    """The pass's operators from the fp64 oracle (float64 torch tensors)."""

    def __init__(self, n_full):
        self.n_full = n_full

    def rotate(self, x1, g):
        return torch.from_numpy(oracle.rotate(x1.numpy(), int(g)))

    def forward(self, x, idx):
        return torch.from_numpy(oracle.fwd(x.numpy(), np.asarray(idx), self.n_full, self.n_det))

    def residual(self, p1, y, idx):
        mcs, rs = [], []
        for b in range(p1.shape[0]):
            yb = y[b].numpy()
            mc, _, r = oracle.residual(p1[b].numpy(), yb, np.asarray(idx), np.zeros((1, 1)), np.zeros((1, 1)))
            mcs.append(mc)
            rs.append(r)
        return torch.tensor(mcs, dtype=torch.float64), torch.from_numpy(np.stack(rs))

    def fbp(self, p2, idx, m_total, out=None):
        v = torch.from_numpy(oracle.fbp(p2.numpy(), np.asarray(idx), self.n_full, self.N, m_total=m_total))
        if out is not None:
            out.copy_(v)
            return out
        return v

    def adjoint(self, r, idx, scale, out=None):
        v = torch.from_numpy(oracle.adj(r.numpy(), np.asarray(idx), self.n_full, self.N, scale))
        if out is not None:
            out.copy_(v)
            return out
        return v

    def ei(self, x2, x3, idx):
        return ((x2 - x3) ** 2).sum(dim=(1, 2))

    def ramp(self, p):
        return torch.from_numpy(oracle.ramp(p.numpy()))

    def backproject_band(self, q, r, idx, x2, row0, rows, m_total):
        band = slice(row0, row0 + rows)
        xf = oracle.adj(q.numpy(), np.asarray(idx), self.n_full, self.N, np.pi / (2 * m_total))[:, band]
        gr = oracle.adj(r.numpy(), np.asarray(idx), self.n_full, self.N, 2.0)[:, band]
        ei = ((x2.numpy()[:, band] - xf) ** 2).sum(axis=(1, 2))
        return torch.from_numpy(np.ascontiguousarray(xf)), torch.from_numpy(np.ascontiguousarray(gr)), torch.from_numpy(ei)


def make_ops(cfg):
    ops = OracleOps(cfg.n_full)
    ops.N, ops.n_det = cfg.N, cfg.n_det
    return ops


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    cfg = synth.CONFIGS["cfg1"]
    x1, y = synth.make_workload(cfg, seed=0)
    g, idx = oracle.draw(0, 0, oracle.SHARED_IMAGE, cfg.n_full, cfg.m)
    return cfg, torch.from_numpy(x1.astype(np.float64)), torch.from_numpy(y.astype(np.float64)), g, idx


def _angle_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, x1, y, g, idx = _inputs()
    out = skdist.angle_split_pass(make_ops(cfg), x1, y, g, idx)
    q.put((rank, {k: out[k].numpy() for k in ("x2", "xfbp", "grad", "mc", "ei")}, list(out["idx"])))
    dist.barrier()
    dist.destroy_process_group()


def _allgather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, x1, y, g, idx = _inputs()
    out = skdist.angle_split_pass_allgather(make_ops(cfg), x1, y, g, np.asarray(idx))
    q.put((rank, {k: out[k].numpy() for k in ("x2", "xfbp", "grad", "mc", "ei")},
           (out["rows"].start, out["rows"].stop)))
    dist.barrier()
    dist.destroy_process_group()


def _batch_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["cfg2"]
    mine = skdist.batch_range(cfg.B, rank, world)
    # inputs and draws keyed by the GLOBAL image index: each rank builds only its images
    x1, y = synth.make_workload(cfg, seed=0, images=mine)
    res = []
    for k, b in enumerate(mine):
        gb, ib = oracle.draw(0, 0, b, cfg.n_full, cfg.m)
        o = oracle.sketched_pass(x1[k], y[k], gb, ib, cfg.n_full)
        res.append(torch.tensor([o["mc"], o["ei"], float(np.abs(o["grad"]).sum())], dtype=torch.float64))
    local = torch.stack(res)
    sizes = [len(skdist.batch_range(cfg.B, r, world)) for r in range(world)]
    gathered = [torch.zeros(s, 3, dtype=torch.float64) for s in sizes]
    dist.all_gather(gathered, local)
    if rank == 0:
        q.put(torch.cat(gathered).numpy())
    dist.barrier()
    dist.destroy_process_group()


def _run(worker, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world if worker is not _batch_worker else 1)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return outs


def test_batch_range_partition():
    for B in (1, 2, 7, 16, 64):
        for world in (1, 2, 3, 4, 8):
            if world > B:
                continue
            rs = [skdist.batch_range(B, r, world) for r in range(world)]
            assert [i for r in rs for i in r] == list(range(B))
            assert max(len(r) for r in rs) - min(len(r) for r in rs) <= 1
    with pytest.raises(ValueError):
        skdist.angle_shard(list(range(3)), 0, 4)


def test_allreduce_volume():
    # cfg5 single 1024^2 image: 2 N^2 + 1 fp32 = 8,388,612 bytes
    assert skdist.allreduce_bytes(1, 1024) == 8388612


def test_angle_split_gloo_matches_single_process():
    """Two ranks, each with half of the sketch: after the packed all-reduce x_fbp, grad, mc
    and ei equal the full-sketch pass (SURVEY §8(e) partition identities)."""
    cfg, x1, y, g, idx = _inputs()
    full = skdist.angle_split_pass(make_ops(cfg), x1, y, g, idx)  # world 1: the plain pass
    ref = {}
    for b in range(cfg.B):
        o = oracle.sketched_pass(x1[b].numpy(), y[b].numpy(), g, idx, cfg.n_full)
        for k in ("xfbp", "grad", "mc", "ei"):
            ref.setdefault(k, []).append(o[k])
    for k in ("xfbp", "grad"):
        np.testing.assert_allclose(full[k].numpy(), np.stack(ref[k]), rtol=0, atol=1e-11)
    outs = _run(_angle_worker)
    shards = sorted(outs, key=lambda t: t[0])
    assert shards[0][2] + shards[1][2] == list(idx)  # contiguous shards cover the sketch
    for _, o, _ in shards:
        for k in ("xfbp", "grad"):
            np.testing.assert_allclose(o[k], full[k].numpy(), rtol=0, atol=1e-10)
        np.testing.assert_allclose(o["mc"], full["mc"].numpy(), rtol=1e-12)
        np.testing.assert_allclose(o["ei"], full["ei"].numpy(), rtol=1e-12)


def test_batch_split_gloo_matches_single_process():
    """Two ranks each run their global images (draws keyed by the global index): the
    gathered per-image results equal the single-process loop exactly."""
    cfg = synth.CONFIGS["cfg2"]
    x1, y = synth.make_workload(cfg, seed=0)
    ref = []
    for b in range(cfg.B):
        gb, ib = oracle.draw(0, 0, b, cfg.n_full, cfg.m)
        o = oracle.sketched_pass(x1[b], y[b], gb, ib, cfg.n_full)
        ref.append([o["mc"], o["ei"], float(np.abs(o["grad"]).sum())])
    (got,) = _run(_batch_worker)
    np.testing.assert_array_equal(got, np.array(ref))


def test_angle_split_allgather_gloo_matches_single_process():
    """two ranks each project + filter half of the sketch, all-gather the
    filtered and residual rows, and backproject all angles for their row band; the bands
    tile x_fbp and grad of the full-sketch pass, and the reduced mc, ei equal it."""
    cfg, x1, y, g, idx = _inputs()
    ref = {k: [] for k in ("xfbp", "grad", "mc", "ei")}
    for b in range(cfg.B):
        o = oracle.sketched_pass(x1[b].numpy(), y[b].numpy(), g, idx, cfg.n_full)
        for k in ref:
            ref[k].append(o[k])
    ref = {k: np.stack(v) if k in ("xfbp", "grad") else np.array(v) for k, v in ref.items()}
    outs = sorted(_run(_allgather_worker), key=lambda t: t[0])
    assert outs[0][2][0] == 0 and outs[0][2][1] == outs[1][2][0] and outs[1][2][1] == cfg.N
    for k in ("xfbp", "grad"):
        got = np.concatenate([o[k] for _, o, _ in outs], axis=1)
        np.testing.assert_allclose(got, ref[k], rtol=0, atol=1e-11)
    for _, o, _ in outs:
        np.testing.assert_allclose(o["mc"], ref["mc"], rtol=1e-12)
        np.testing.assert_allclose(o["ei"], ref["ei"], rtol=1e-12)


def test_allgather_volume():
    # cfg5: 2 B m n_det fp32 = 2,967,552 bytes exchanged vs 8,388,612 all-reduced
    assert skdist.allgather_bytes(1, 256, 1449) == 2967552



@pytest.mark.parametrize("world", [2, 3, 5])
def test_rs_layout_reduces_to_full_pass(world):
    """SURVEY §8(f) #2 (b) host logic: each virtual rank's oracle partials (its angle shard,
    the full sketch's density scale) placed by rs_slot_offset — the layout the backprojector's
    reduce-scatter epilogue stores into — and each owner's slots summed in rank order give
    the bands of the full-sketch pass's x_fbp and grad; every band row is stored exactly once
    per slot, and the bands tile the image (rows from batch_range)."""
    cfg, x1, y, g, idx = _inputs()
    ops = make_ops(cfg)
    B, N, m = cfg.B, cfg.N, len(idx)
    bmax = -(-N // world)
    recv = [np.full((world, 2 * B * bmax * N), np.nan) for _ in range(world)]
    x2 = torch.stack([ops.rotate(x1[b], g) for b in range(B)])
    for rk in range(world):
        sub = skdist.angle_shard(idx, rk, world)
        p1 = torch.stack([ops.forward(x1[b], sub) for b in range(B)])
        p2 = torch.stack([ops.forward(x2[b], sub) for b in range(B)])
        _, r = ops.residual(p1, y, sub)
        parts = [torch.stack([ops.fbp(p2[b], sub, m) for b in range(B)]).numpy(),
                 torch.stack([ops.adjoint(r[b], sub, 2.0) for b in range(B)]).numpy()]
        for j in range(2):
            for b in range(B):
                for row in range(N):
                    o, off = skdist.rs_slot_offset(B, N, world, j, b, row, 0)
                    assert np.isnan(recv[o][rk, off:off + N]).all(), "stored twice"
                    recv[o][rk, off:off + N] = parts[j][b, row]
    rows_seen = []
    for o in range(world):
        band = skdist.batch_range(N, o, world)
        rows_seen += list(band)
        slots = recv[o].reshape(world, 2, B, bmax, N)[:, :, :, :len(band)]
        assert not np.isnan(slots).any()
        acc = np.zeros_like(slots[0])
        for s in range(world):
            acc = acc + slots[s]
        for b in range(B):
            ref = oracle.sketched_pass(x1[b].numpy(), y[b].numpy(), g, idx, cfg.n_full)
            np.testing.assert_allclose(acc[0, b], ref["xfbp"][band.start:band.stop], rtol=0, atol=1e-11)
            np.testing.assert_allclose(acc[1, b], ref["grad"][band.start:band.stop], rtol=0, atol=1e-11)
    assert rows_seen == list(range(N))
