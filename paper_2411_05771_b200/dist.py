"""Multi-GPU partitioning of the sketched-EI operator pass.

One process per GPU (torchrun), torch.distributed for the plumbing.  Two partitions:

* batch split (BASELINE.json cfg4, "split by batch across 1/2/4/8 GPUs"): rank r owns the
  global images [r B/G, (r+1) B/G).  Images are independent and the draws are keyed by the
  global image index (R5), so every rank runs the whole pass on its images with no
  data-path collective; results equal the 1-GPU run bit for bit.
* angle split (cfg5, "single image ... split by angle ... with NCCL all-reduce of partial
  backprojections"): rank r owns the contiguous slice S_r of the sketch's m angles.  Every
  operator of the pass is a sum over angles except the rotation and the EI norm, so

      x_fbp = (pi / 2m) A_S^T ramp(A_S x2) = sum_r (pi / 2m) A_{S_r}^T ramp(A_{S_r} x2)
      grad  = 2 A_S^T (A_S x1 - y_S)        = sum_r 2 A_{S_r}^T r_r
      mc    = ||A_S x1 - y_S||^2            = sum_r ||r_r||^2

  (the sketch is a row subset; §1.1: ||Ax - y||^2 = sum_i ||S_i A x -
  S_i y||^2).  Each rank computes its partials with the FBP density scale of the FULL
  sketch size m (skei_fbp's m_total), packs [x_fbp | grad | mc] into one buffer, and one
  all_reduce(SUM) over NVLink/NVSwitch completes them; ei = ||x2 - x_fbp||^2 is then
  evaluated on the summed x_fbp (redundantly on every rank).

The compute is injected (`ops`): `CudaOps` calls the C ABI (libskei.so); the CPU tests pass
an oracle-backed implementation so the partition logic runs under gloo without a GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

__all__ = ["batch_range", "angle_shard", "CudaOps", "angle_split_pass", "batch_split_images",
           "angle_split_pass_allgather", "shard_phase", "band_phase", "angle_split_pass_p2p",
           "P2PBuffers", "simulate_p2p_split", "RSBuffers", "rs_slot_offset",
           "angle_split_pass_rs", "simulate_rs_split"]


def batch_range(B: int, rank: int, world: int) -> range:
    """Global image indices of `rank` when B images are split over `world` ranks (contiguous,
    sizes differ by at most one)."""
    if B < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad split B={B} rank={rank} world={world}")
    q, rem = divmod(B, world)
    lo = rank * q + min(rank, rem)
    return range(lo, lo + q + (1 if rank < rem else 0))


def batch_split_images(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    r = batch_range(x.shape[0], rank, world)
    return x[r.start:r.stop]


def angle_shard(idx, rank: int, world: int):
    """The contiguous slice of the sketch (m ascending angle indices) owned by `rank`."""
    m = len(idx)
    if m < world:
        raise ValueError(f"angle split needs m >= world ({m} < {world})")
    r = batch_range(m, rank, world)
    return idx[r.start:r.stop]


@dataclass
class CudaOps:
    """The pass's operators on one GPU, through the C ABI (paper_2411_05771_b200)."""
    plan: object

    def rotate(self, x1, g):
        import paper_2411_05771_b200 as sk
        return sk.rotate(self.plan, x1, g)

    def forward(self, x, idx):
        import paper_2411_05771_b200 as sk
        return sk.radon_fwd(self.plan, x, idx)

    def residual(self, p1, y, idx):
        import paper_2411_05771_b200 as sk
        mc, _, r = sk.ei_residual(self.plan, p1, y, idx, None, None)
        return mc, r

    def fbp(self, p2, idx, m_total, out=None):
        import paper_2411_05771_b200 as sk
        return sk.fbp(self.plan, p2, idx, m_total=m_total, out=out)

    def adjoint(self, r, idx, scale, out=None):
        import paper_2411_05771_b200 as sk
        return sk.radon_adj(self.plan, r, idx, scale, out=out)

    def ei(self, x2, x3, idx):
        import paper_2411_05771_b200 as sk
        _, ei, _ = sk.ei_residual(self.plan, None, None, idx, x2, x3)
        return ei

    def ramp(self, p):
        import paper_2411_05771_b200 as sk
        return sk.ramp_filter(self.plan, p)

    def backproject_band(self, q, r, idx, x2, row0, rows, m_total):
        import paper_2411_05771_b200 as sk
        return sk.backproject_band(self.plan, q, r, idx, x2, row0, rows, m_total=m_total)

    def ramp_allgather(self, p, r, row0, m_total, peer_q, peer_r):
        import paper_2411_05771_b200 as sk
        return sk.ramp_allgather(self.plan, p, r, row0, m_total, peer_q, peer_r)

    def backproject_scatter(self, q, r, idx, m_total, peer_recv, rank):
        import paper_2411_05771_b200 as sk
        return sk.backproject_scatter(self.plan, q, r, idx, m_total, peer_recv, rank)

    def band_reduce(self, recv, world, rank, x2):
        import paper_2411_05771_b200 as sk
        return sk.band_reduce(self.plan, recv, world, rank, x2)


def angle_split_pass(ops, x1, y, g, idx, group=None):
    """One sketched-EI pass of a batch whose sketch `idx` (m ascending indices) is split over
    the ranks of `group` (the whole world if None).  Returns a dict with x2, x_fbp, grad
    (complete on every rank after the all-reduce), mc and ei ([B]), and this rank's p1, p2, r
    shards with their angle indices.  Single-rank groups reduce to the plain pass."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m = len(idx)
    sub = angle_shard(idx, rank, world)
    x2 = ops.rotate(x1, g)
    p1 = ops.forward(x1, sub)
    p2 = ops.forward(x2, sub)
    B, N = x1.shape[0], x1.shape[-1]
    nn = B * N * N
    # one packed buffer [x_fbp (B N^2) | grad (B N^2) | mc (B)]: the kernels write their
    # partials straight into it, then one all_reduce(SUM) completes all three
    packed = torch.empty(2 * nn + B, dtype=x1.dtype, device=x1.device)
    xfbp = packed[:nn].view(B, N, N)
    grad = packed[nn:2 * nn].view(B, N, N)
    mc = packed[2 * nn:]
    mc_part, r = ops.residual(p1, y, sub)
    ops.fbp(p2, sub, m, out=xfbp)      # density scale pi / (2 m) of the FULL sketch
    ops.adjoint(r, sub, 2.0, out=grad)
    mc.copy_(mc_part)
    if world > 1:
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    ei = ops.ei(x2, xfbp, idx)
    return {"x2": x2, "xfbp": xfbp, "grad": grad, "mc": mc, "ei": ei,
            "p1": p1, "p2": p2, "r": r, "idx": sub, "allreduce_bytes": packed.numel() * packed.element_size()}


def allreduce_bytes(B: int, N: int) -> int:
    """Bytes of the angle split's single all-reduce: (2 B N^2 + B) fp32."""
    return 4 * (2 * B * N * N + B)


def ring_bytes_per_gpu(B: int, N: int, world: int) -> float:
    """Bytes each GPU sends in a ring all-reduce of the packed buffer: 2 (G-1)/G x payload."""
    return 2.0 * (world - 1) / world * allreduce_bytes(B, N) if world > 1 else 0.0


def expected_scale(m_total: int) -> float:
    return math.pi / (2.0 * m_total)


# ---------------------------------------------------------------------------------------
# Communication-reduced single-image split: every rank projects and
# filters its angle shard, the ranks all-gather the filtered rows q and the residual rows r
# (2 B m n_det floats in total, 1.48 MB each at cfg5), and every rank backprojects ALL the
# angles for its own row band of the image (skei_backproject_band: x_fbp, grad and the
# band's ei partial).  One all-reduce of 2 B scalars (mc, ei) completes the losses.  Per
# GPU that moves (G-1)/G x 2.97 MB instead of the 2 (G-1)/G x 8.4 MB of the all-reduce of
# whole-image partials; the outputs x_fbp and grad stay row-sharded (band r on rank r).

def shard_phase(ops, x1, y, g, idx, rank: int, world: int):
    """Before the exchange: x2 (replicated), this rank's angle shard, its filtered rows
    q and residual rows r, and its mc partial."""
    sub = angle_shard(idx, rank, world)
    x2 = ops.rotate(x1, g)
    p1 = ops.forward(x1, sub)
    p2 = ops.forward(x2, sub)
    mc_part, r = ops.residual(p1, y, sub)
    return {"x2": x2, "idx": sub, "q": ops.ramp(p2), "r": r, "mc": mc_part}


def band_phase(ops, q_full, r_full, idx, x2, rank: int, world: int):
    """After the exchange: this rank's row band of x_fbp and grad from all m angles, and the
    band's ei partial."""
    N = x2.shape[-1]
    band = batch_range(N, rank, world)
    xf, gr, ei = ops.backproject_band(q_full, r_full, idx, x2, band.start, len(band), idx.shape[-1])
    return {"rows": band, "xfbp": xf, "grad": gr, "ei": ei}


def angle_split_pass_allgather(ops, x1, y, g, idx, group=None):
    """One pass of a batch whose sketch `idx` is split over the ranks of `group`, exchanging
    filtered sinogram rows instead of partial images (module comment above).  Returns x2,
    this rank's row bands of x_fbp and grad (`rows`), and the complete mc and ei ([B])."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sh = shard_phase(ops, x1, y, g, idx, rank, world)
    B, n_det = sh["q"].shape[0], sh["q"].shape[-1]
    sizes = [len(batch_range(len(idx), r, world)) for r in range(world)]
    mx = max(sizes)
    # equal-sized all-gather buffers: [B][2][mx][n_det] per rank (q rows, r rows), padded
    send = torch.zeros(B, 2, mx, n_det, dtype=sh["q"].dtype, device=sh["q"].device)
    send[:, 0, :sh["q"].shape[1]] = sh["q"]
    send[:, 1, :sh["r"].shape[1]] = sh["r"]
    if world > 1:
        recv = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(recv, send, group=group)
    else:
        recv = [send]
    q_full = torch.cat([recv[i][:, 0, :sizes[i]] for i in range(world)], dim=1).contiguous()
    r_full = torch.cat([recv[i][:, 1, :sizes[i]] for i in range(world)], dim=1).contiguous()
    bd = band_phase(ops, q_full, r_full, idx, sh["x2"], rank, world)
    scal = torch.cat([sh["mc"].to(bd["ei"].dtype), bd["ei"]])
    if world > 1:
        dist.all_reduce(scal, op=dist.ReduceOp.SUM, group=group)
    return {"x2": sh["x2"], "xfbp": bd["xfbp"], "grad": bd["grad"], "rows": bd["rows"],
            "mc": scal[:B], "ei": scal[B:], "idx": sh["idx"],
            "allgather_bytes": send.numel() * send.element_size() * world}


def allgather_bytes(B: int, m: int, n_det: int) -> int:
    """Bytes all ranks contribute to the exchange of the all-gather split: 2 B m n_det fp32."""
    return 4 * 2 * B * m * n_det


# ---------------------------------------------------------------------------------------
# The same split with the exchange fused into the ramp kernel (no NCCL on
# the data path): every rank's ramp kernel stores each filtered row — and each residual row —
# straight into the full-size q and r buffers of EVERY rank (P2P stores over NVLink into
# symmetric memory, its own buffer among them), so the 2.97 MB all-gather overlaps the FFT
# tile by tile; a device-side barrier then releases the row-band backprojection.

class P2PBuffers:
    """Full-size q and r buffers [B][m][n_det] on every rank plus the peers' pointers: torch
    symmetric memory over the group (world > 1), or plain local tensors (world 1)."""

    def __init__(self, B, m, n_det, device, group=None):
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.world = world
        if world > 1:
            import torch.distributed._symmetric_memory as symm
            grp = group if group is not None else dist.group.WORLD
            if hasattr(symm, "enable_symm_mem_for_group"):
                symm.enable_symm_mem_for_group(grp.group_name)
            self.buf = symm.empty((2, B, m, n_det), dtype=torch.float32, device=device)
            self.handle = symm.rendezvous(self.buf, grp.group_name)
            step = B * m * n_det * 4
            ptrs = [int(p) for p in self.handle.buffer_ptrs]
            self.peer_q = ptrs
            self.peer_r = [p + step for p in ptrs]
        else:
            self.buf = torch.empty((2, B, m, n_det), dtype=torch.float32, device=device)
            self.handle = None
            self.peer_q = [self.buf[0].data_ptr()]
            self.peer_r = [self.buf[1].data_ptr()]
        self.q, self.r = self.buf[0], self.buf[1]

    def barrier(self, channel: int = 0):
        """Stream-ordered device barrier over the group: every rank's stream has reached
        this point (e.g. its stores have landed in every buffer)."""
        if self.handle is not None:
            self.handle.barrier(channel=channel)


def angle_split_pass_p2p(ops, x1, y, g, idx, group=None, bufs: P2PBuffers | None = None):
    """One pass with the sketch `idx` split over the ranks of `group`, the filtered and residual
    rows exchanged by the ramp kernel's own P2P stores (module comment above); outputs as
    angle_split_pass_allgather (row bands of x_fbp and grad, complete mc and ei)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m = len(idx)
    sub = angle_shard(idx, rank, world)
    row0 = batch_range(m, rank, world).start
    x2 = ops.rotate(x1, g)
    p1 = ops.forward(x1, sub)
    p2 = ops.forward(x2, sub)
    mc_part, r = ops.residual(p1, y, sub)
    B, n_det = p2.shape[0], p2.shape[-1]
    if bufs is None:
        bufs = P2PBuffers(B, m, n_det, p2.device, group)
    else:
        # reused buffers: no rank may overwrite a peer's q / r while that peer still
        # backprojects the previous pass from them (write-after-read across ranks)
        bufs.barrier(channel=1)
    ops.ramp_allgather(p2, r, row0, m, bufs.peer_q, bufs.peer_r)
    bufs.barrier()
    bd = band_phase(ops, bufs.q, bufs.r, idx, x2, rank, world)
    scal = torch.cat([mc_part.to(bd["ei"].dtype), bd["ei"]])
    if world > 1:
        dist.all_reduce(scal, op=dist.ReduceOp.SUM, group=group)
    return {"x2": x2, "xfbp": bd["xfbp"], "grad": bd["grad"], "rows": bd["rows"],
            "mc": scal[:B], "ei": scal[B:], "idx": sub,
            "p2p_bytes": 2 * B * len(sub) * n_det * 4 * world}


def simulate_p2p_split(ops, x1, y, g, idx, world: int):
    """The P2P split's data path on ONE GPU: `world` virtual ranks, each with its own full-size
    q/r buffers; every virtual rank's ramp kernel stores its rows into all of them (the same
    kernel and pointer lists as across GPUs), then each virtual rank backprojects its band.
    Returns the per-rank band outputs and the shard scalars (test helper)."""
    m = len(idx)
    x2 = ops.rotate(x1, g)
    B, n_det = x1.shape[0], ops.plan.n_det
    bufs = [torch.empty((2, B, m, n_det), dtype=torch.float32, device=x1.device) for _ in range(world)]
    peer_q = [b[0].data_ptr() for b in bufs]
    peer_r = [b[1].data_ptr() for b in bufs]
    mc = torch.zeros(B, dtype=torch.float32, device=x1.device)
    for rk in range(world):
        sub = angle_shard(idx, rk, world)
        p1 = ops.forward(x1, sub)
        p2 = ops.forward(x2, sub)
        mc_part, r = ops.residual(p1, y, sub)
        ops.ramp_allgather(p2, r, batch_range(m, rk, world).start, m, peer_q, peer_r)
        mc += mc_part
    bands = [band_phase(ops, bufs[rk][0], bufs[rk][1], idx, x2, rk, world) for rk in range(world)]
    return {"x2": x2, "bands": bands, "mc": mc, "bufs": bufs}



# ---------------------------------------------------------------------------------------
# The split's other communication-reduced form: the backprojection's
# reduce-scatter fused into the backprojector.  Every rank projects, filters and backprojects
# only its angle shard; the adjoint kernel's epilogue stores each output row of the partial
# x_fbp and grad straight into the receive buffer of the rank owning that row's band (P2P
# stores into symmetric memory, slot = the sending rank), so the exchange — (G-1)/G x 2 B n^2
# floats per GPU, half the all-reduce's — overlaps the backprojection tile by tile.  After a
# device barrier each rank sums its G slots in rank order (skei_band_reduce: a fixed order,
# bitwise reproducible) into its bands of x_fbp and grad plus the band's ei partial; one
# all-reduce of 2 B scalars (mc, ei) completes the losses.  Outputs are row-sharded like the
# all-gather form's; the rows are batch_range(n, rank, G).

def rs_slot_offset(B: int, n: int, world: int, job: int, b: int, row: int, col: int):
    """(owner rank, float offset within the owner's receive buffer slot) of output element
    (job, image b, row, col) — the layout skei_backproject_scatter stores into (host mirror
    of radon_adj.cu out_at, used by the CPU layout test)."""
    q, rem = divmod(n, world)
    o = row // (q + 1) if row < rem * (q + 1) else rem + (row - rem * (q + 1)) // q
    start = batch_range(n, o, world).start
    bmax = -(-n // world)
    return o, ((job * B + b) * bmax + row - start) * n + col


class RSBuffers:
    """One receive buffer [world][2][B][bmax][n] per rank plus the peers' pointers: torch
    symmetric memory over the group (world > 1), or a plain local tensor (world 1)."""

    def __init__(self, B, n, device, group=None):
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.world = world
        bmax = -(-n // world)
        shape = (world, 2, B, bmax, n)
        if world > 1:
            import torch.distributed._symmetric_memory as symm
            grp = group if group is not None else dist.group.WORLD
            if hasattr(symm, "enable_symm_mem_for_group"):
                symm.enable_symm_mem_for_group(grp.group_name)
            self.buf = symm.empty(shape, dtype=torch.float32, device=device)
            self.handle = symm.rendezvous(self.buf, grp.group_name)
            self.peers = [int(p) for p in self.handle.buffer_ptrs]
        else:
            self.buf = torch.empty(shape, dtype=torch.float32, device=device)
            self.handle = None
            self.peers = [self.buf.data_ptr()]

    def barrier(self, channel: int = 0):
        if self.handle is not None:
            self.handle.barrier(channel=channel)


def angle_split_pass_rs(ops, x1, y, g, idx, group=None, bufs: RSBuffers | None = None):
    """One pass with the sketch `idx` split over the ranks of `group`, the backprojection's
    reduce-scatter fused into the backprojector (comment above); outputs as
    angle_split_pass_allgather (row bands of x_fbp and grad, complete mc and ei)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m = len(idx)
    sub = angle_shard(idx, rank, world)
    x2 = ops.rotate(x1, g)
    p1 = ops.forward(x1, sub)
    p2 = ops.forward(x2, sub)
    mc_part, r = ops.residual(p1, y, sub)
    q = ops.ramp(p2)
    B, N = x1.shape[0], x1.shape[-1]
    if bufs is None:
        bufs = RSBuffers(B, N, x1.device, group)
    else:
        # reused buffers: no rank may store into a peer's slots while that peer still sums
        # them for the previous pass (write-after-read across ranks)
        bufs.barrier(channel=1)
    ops.backproject_scatter(q, r, sub, m, bufs.peers, rank)
    bufs.barrier()
    xf, gr, ei = ops.band_reduce(bufs.buf, world, rank, x2)
    scal = torch.cat([mc_part.to(ei.dtype), ei])
    if world > 1:
        dist.all_reduce(scal, op=dist.ReduceOp.SUM, group=group)
    return {"x2": x2, "xfbp": xf, "grad": gr, "rows": batch_range(N, rank, world),
            "mc": scal[:B], "ei": scal[B:], "idx": sub,
            "rs_bytes": 2 * B * N * N * 4 * (world - 1) // max(world, 1)}


def simulate_rs_split(ops, x1, y, g, idx, world: int):
    """The reduce-scatter split's data path on ONE GPU: `world` virtual ranks with their own
    receive buffers; every virtual rank's backprojector stores its partial rows into all of
    them (the same kernel and pointer lists as across GPUs), then each virtual rank sums its
    slots.  Returns the per-rank bands (x_fbp, grad, ei partial) and the summed mc (test
    helper)."""
    m = len(idx)
    x2 = ops.rotate(x1, g)
    B, N = x1.shape[0], x1.shape[-1]
    bmax = -(-N // world)
    bufs = [torch.full((world, 2, B, bmax, N), float("nan"), dtype=torch.float32,
                       device=x1.device) for _ in range(world)]
    peers = [b.data_ptr() for b in bufs]
    mc = torch.zeros(B, dtype=torch.float32, device=x1.device)
    for rk in range(world):
        sub = angle_shard(idx, rk, world)
        p1 = ops.forward(x1, sub)
        p2 = ops.forward(x2, sub)
        mc_part, r = ops.residual(p1, y, sub)
        ops.backproject_scatter(ops.ramp(p2), r, sub, m, peers, rk)
        mc += mc_part
    bands = []
    for rk in range(world):
        xf, gr, ei = ops.band_reduce(bufs[rk], world, rk, x2)
        bands.append({"rows": batch_range(N, rk, world), "xfbp": xf, "grad": gr, "ei": ei})
    return {"x2": x2, "bands": bands, "mc": mc, "bufs": bufs}
