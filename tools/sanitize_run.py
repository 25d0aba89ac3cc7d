"""Every kernel of libskei.so once, at small sizes, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick
    compute-sanitizer --tool synccheck python tools/sanitize_run.py

(one tool per gpurun call, B200_PROFILING.md).  Covers the mbarrier / bulk-copy pipelines of
the forward (triple-buffered BB = 4, job-fused BB = 2, single-buffer n = 1024-like line
blocks via a wide image, stream-K split units), the backprojector's producer warp and
chunked windows, the self-resetting completion counters (two passes back to back on one
workspace), the ramp (plain and peer-store modes), draws, rotation and its transpose, the
REI noise, the deviation's reductions and the row-band backprojection.  Prints one line per
step and "sanitize_run ok" at the end; the sanitizer's own summary follows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2411_05771_b200 as sk  # noqa: E402
from paper_2411_05771_b200 import dist  # noqa: E402


def step(name):
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def run_geometry(n, n_det, n_full, m, B, mode, per_image, quick):
    dev = torch.device("cuda:0")
    plan = sk.Plan.get(n, n_det, n_full, 0, device=0)
    gen = torch.Generator().manual_seed(n * 7 + B)
    x1 = torch.rand((B, n, n), generator=gen).to(dev)
    y = torch.rand((B, n_full, n_det), generator=gen).to(dev)
    tag = f"n{n} det{n_det} full{n_full} m{m} B{B} {'per-image' if per_image else 'shared'}"
    if per_image:
        g, idx = sk.draw_device(1, 0, 0, B, False, n_full, m, mode)
    else:
        g, idx = sk.draw_device(1, 0, 0, 1, True, n_full, m, mode)
    step(f"draw {tag}")
    out = sk.sketched_pass(plan, x1, y, g, idx)
    step(f"pass {tag}")
    sk.sketched_pass(plan, x1, y, g, idx, out=out)  # counters reset by the first pass
    step(f"pass again {tag}")
    if quick:
        return
    o2 = sk.sketched_pass_draw(plan, x1, y, 3, 1, m, mode=mode, shared=not per_image)
    step(f"pass_draw {tag}")
    gr = sk.ei_grad(plan, out["x2"], out["xfbp"], g, idx)
    step(f"ei_grad {tag}")
    sk.sketched_pass_rei(plan, x1, y, g, idx, 0.01, 5, 0, 0)
    step(f"rei {tag}")
    sk.rotate_adjoint(plan, gr, g)
    step(f"rotate_adjoint {tag}")
    del o2


def main():
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    print(sk.version(), flush=True)
    # cfg1: BB = 4 groups (B = 2 -> BB = 2), small image
    run_geometry(64, 91, 32, 8, 2, 0, False, quick)
    # odd batch with per-image sketches: job-fused BB = 2 groups
    run_geometry(64, 91, 32, 8, 3, 1, True, quick)
    # cfg2-like, BB = 4 groups, uniform sketch
    run_geometry(256, 363, 128, 32, 4 if quick else 8, 1, False, quick)
    if not quick:
        # a wide image: one line block per buffer (the cfg5 staging path), B = 1 fused
        run_geometry(1024, 1449, 64, 16, 1, 1, False, quick)
    plan = sk.Plan.get(64, 91, 32, 0, device=0)
    dev = torch.device("cuda:0")
    x = torch.rand((2, 64, 64), device=dev)
    g, idx = sk.draw_device(2, 0, 0, 1, True, 32, 8, 0)
    # the standalone calls
    p = sk.radon_fwd(plan, x, idx)
    sk.radon_adj(plan, p, idx, 2.0)
    sk.ramp_filter(plan, p)
    sk.fbp(plan, p, idx)
    sk.fbp_adjoint(plan, x, idx)
    sk.ei_residual(plan, p, torch.rand((2, 32, 91), device=dev), idx, x, x * 0.5)
    step("standalone calls")
    v = torch.rand((2, 64, 64), device=dev)
    sk.sketch_deviation(plan, idx, v, 3)
    step("deviation")
    ops = dist.CudaOps(plan)
    y = torch.rand((2, 32, 91), device=dev)
    gg = torch.tensor([37], dtype=torch.int32, device=dev)
    dist.simulate_p2p_split(ops, x, y, gg, idx[0], 2)
    step("ramp_allgather + backproject_band (2 virtual ranks)")
    sink = torch.empty(4, device=dev)
    sk.smem_probe(2, 2, sink)
    sk.l2_probe(torch.rand(1 << 16, device=dev), 2, 2, sink)
    step("probes")
    print("sanitize_run ok", flush=True)


if __name__ == "__main__":
    main()
