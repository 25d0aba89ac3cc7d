"""GPU parity of the next row: the backward of the EI branch.

rotate_adjoint (T_g^T), fbp_adjoint ((pi/2m) ramp A_S) and the fused EI gradient
T_g^T (I - M) 2 (x2 - x3) through the C ABI against the fp64 oracle (oracle.rotate_adj,
oracle.ei_grad), plus the torch.autograd wrappers.  Bar: max|gpu - ref| <= tol * max|ref|
with tol = 1e-4 for the operators and the tolerance derived in DESIGN.md §5 for the EI
gradient (it differences two nearly equal images).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2411_05771_b200 as sk
import synth
from paper_2411_05771_b200 import autograd as ska

from test_gpu_parity import close, dev, idx_t

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("N,B,g", [(64, 2, 37), (64, 3, 301), (256, 4, 123), (96, 1, 1), (512, 4, 211)])
def test_rotate_adjoint_parity(N, B, g):
    cfg = synth.CONFIGS["cfg1"]
    plan = sk.Plan.get(N, int(np.ceil(N * 2 ** 0.5)), cfg.n_full, 0)
    y = synth.rand_images(B, N, 5)
    out = sk.rotate_adjoint(plan, dev(y), idx_t([g]))
    for b in range(B):
        close(out[b], oracle.rotate_adj(y[b], g), f"T^T N={N} g={g} b={b}")


def test_rotate_adjoint_per_image_angles():
    N, B = 64, 3
    plan = sk.Plan.get(N, 91, 32, 0)
    y = synth.rand_images(B, N, 6)
    gs = [10, 95, 250]
    out = sk.rotate_adjoint(plan, dev(y), idx_t(gs))
    for b in range(B):
        close(out[b], oracle.rotate_adj(y[b], gs[b]), f"T^T b={b}")


def test_rotate_adjoint_quarter_turns_exact():
    N = 64
    plan = sk.Plan.get(N, 91, 32, 0)
    y = dev(synth.rand_images(4, N, 7))
    for g, k in ((360, 0), (90, -1), (180, 2), (270, 1)):
        assert torch.equal(sk.rotate_adjoint(plan, y, idx_t([g])), torch.rot90(y, k, dims=(1, 2))), g


def test_rotate_adjoint_identity_on_gpu():
    N, B = 256, 4
    plan = sk.Plan.get(N, 363, 128, 0)
    x = dev(synth.rand_images(B, N, 8))
    y = dev(synth.rand_images(B, N, 9))
    g = idx_t([77])
    lhs = float((sk.rotate(plan, x, g).double() * y.double()).sum())
    rhs = float((x.double() * sk.rotate_adjoint(plan, y, g).double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * float(x.double().norm() * y.double().norm())


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_fbp_adjoint_parity(name):
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x = synth.rand_images(cfg.B, cfg.N, 10)
    g, idx = sk.draw(0, 5, sk.SHARED_IMAGE, cfg.n_full, cfg.m)
    p = sk.fbp_adjoint(plan, dev(x), idx_t(idx))
    for b in range(cfg.B):
        ref = oracle.ramp(oracle.fwd(x[b], idx, cfg.n_full, cfg.n_det)) * (np.pi / (2 * cfg.m))
        close(p[b], ref, f"{name} fbp^T b={b}")


def _ei_case(name, it=2):
    cfg = synth.CONFIGS[name]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    x1, y = synth.make_workload(cfg, 0)
    g, idx = sk.draw_device(0, it, 0, 1, True, cfg.n_full, cfg.m)
    out = sk.sketched_pass(plan, dev(x1), dev(y), g, idx)
    return cfg, plan, x1, g, idx, out


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_ei_grad_parity(name):
    """The fused EI gradient vs oracle.ei_grad (computed from x1 alone, fp64)."""
    cfg, plan, x1, g, idx, out = _ei_case(name)
    grad = sk.ei_grad(plan, out["x2"], out["xfbp"], g, idx)
    og = int(g[0])
    oidx = idx[0].cpu().numpy()
    for b in range(cfg.B):
        ref = oracle.ei_grad(x1[b], og, oidx, cfg.n_full, cfg.n_det)
        close(grad[b], ref, f"{name} ei grad b={b}", tol=EI_TOL)


def test_ei_grad_full_size_sampled():
    """cfg3 (bench size), first and last image."""
    cfg, plan, x1, g, idx, out = _ei_case("cfg3")
    grad = sk.ei_grad(plan, out["x2"], out["xfbp"], g, idx)
    og, oidx = int(g[0]), idx[0].cpu().numpy()
    for b in (0, cfg.B - 1):
        close(grad[b], oracle.ei_grad(x1[b], og, oidx, cfg.n_full, cfg.n_det), f"cfg3 ei grad b={b}",
              tol=EI_TOL)


def test_autograd_ei_branch_matches_fused_gradient():
    """torch autograd through Rotate -> Project -> SketchedFBP reproduces the fused gradient
    (same operators, composed by autograd) and the oracle."""
    cfg, plan, x1, g, idx, out = _ei_case("cfg2")
    x = dev(x1).requires_grad_(True)
    x2 = ska.Rotate.apply(x, plan, g)
    x3 = ska.SketchedFBP.apply(ska.Project.apply(x2, plan, idx), plan, idx)
    ei = ((x2.double() - x3.double()) ** 2).sum(dim=(1, 2))
    ei.sum().backward()
    fused = sk.ei_grad(plan, out["x2"], out["xfbp"], g, idx)
    close(x.grad, fused.double().cpu().numpy(), "autograd vs fused", tol=1e-4)
    og, oidx = int(g[0]), idx[0].cpu().numpy()
    for b in range(cfg.B):
        close(x.grad[b], oracle.ei_grad(x1[b], og, oidx, cfg.n_full, cfg.n_det), f"autograd b={b}",
              tol=EI_TOL)
        assert abs(float(ei[b].detach()) - float(out["ei"][b])) <= 1e-4 * float(out["ei"][b])


def test_autograd_operator_backwards_are_transposes():
    """<J v, w> = <v, J^T w> for Project and SketchedFBP through autograd."""
    cfg = synth.CONFIGS["cfg2"]
    plan = sk.Plan.get(cfg.N, cfg.n_det, cfg.n_full, cfg.fft_len)
    _, idx = sk.draw_device(0, 4, 0, 1, True, cfg.n_full, cfg.m)
    x = dev(synth.rand_images(2, cfg.N, 11)).requires_grad_(True)
    w = dev(synth.rand_sinograms(2, cfg.m, cfg.n_det, 12))
    (ska.Project.apply(x, plan, idx) * w).sum().backward()
    lhs = float((sk.radon_fwd(plan, x.detach(), idx).double() * w.double()).sum())
    rhs = float((x.detach().double() * x.grad.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)
    p = dev(synth.rand_sinograms(2, cfg.m, cfg.n_det, 13)).requires_grad_(True)
    v = dev(synth.rand_images(2, cfg.N, 14))
    (ska.SketchedFBP.apply(p, plan, idx) * v).sum().backward()
    lhs = float((sk.fbp(plan, p.detach(), idx).double() * v.double()).sum())
    rhs = float((p.detach().double() * p.grad.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


EI_TOL = 1e-4
