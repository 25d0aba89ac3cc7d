"""torch.autograd wrappers of the pass operators (the backward of the EI
branch, for full training).  Forward and backward of every operator run in libskei.so:

    Rotate          x2 = T_g x1                  grad: T_g^T          (skei_rotate / _adjoint)
    Project         p  = A_S x                   grad: A_S^T          (skei_radon_fwd / _adj)
    SketchedFBP     x  = (pi/2m) A_S^T ramp p    grad: (pi/2m) ramp A_S  (skei_fbp / _adjoint)

so the EI term ||T_g x1 - F(A_S^+ A_S T_g x1)||^2 (Eq. 6, Alg. 1
L120-L122) back-propagates to x1 (and to the network F) through the library's kernels.
`ei_grad` is the fused closed form for the identity network (skei_ei_grad).
"""
from __future__ import annotations

import torch

from . import Plan, fbp, fbp_adjoint, radon_adj, radon_fwd, rotate, rotate_adjoint

__all__ = ["Rotate", "Project", "SketchedFBP"]


class Rotate(torch.autograd.Function):
    """x2 = T_g x (bilinear, zero outside; R11) with backward T_g^T."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, plan: Plan, g: torch.Tensor):
        ctx.plan, ctx.g = plan, g
        return rotate(plan, x.contiguous(), g)

    @staticmethod
    def backward(ctx, gy: torch.Tensor):
        return rotate_adjoint(ctx.plan, gy.contiguous(), ctx.g), None, None


class Project(torch.autograd.Function):
    """p = A_S x (sketched pixel-driven projector) with backward A_S^T."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, plan: Plan, idx: torch.Tensor):
        ctx.plan, ctx.idx = plan, idx
        return radon_fwd(plan, x.contiguous(), idx)

    @staticmethod
    def backward(ctx, gp: torch.Tensor):
        return radon_adj(ctx.plan, gp.contiguous(), ctx.idx, 1.0), None, None


class SketchedFBP(torch.autograd.Function):
    """x = (pi / 2 m_total) A_S^T ramp(p) (A_S^+, R7/R9) with backward (pi / 2 m_total) ramp A_S."""

    @staticmethod
    def forward(ctx, p: torch.Tensor, plan: Plan, idx: torch.Tensor, m_total: int | None = None):
        ctx.plan, ctx.idx, ctx.m_total = plan, idx, m_total
        return fbp(plan, p.contiguous(), idx, m_total=m_total)

    @staticmethod
    def backward(ctx, gx: torch.Tensor):
        return fbp_adjoint(ctx.plan, gx.contiguous(), ctx.idx, m_total=ctx.m_total), None, None, None
