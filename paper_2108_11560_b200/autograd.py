"""torch.autograd binding of log K_v(x) (arXiv 2108.11560).

The paper computes the derivatives of log K from the differentiated integrands
(Sec. 4.1) precisely so that log K can sit inside gradient-based
fits (the NIG likelihood).  Here:

* forward: one fused launch of the FP64 / FP32 entry point giving log K, d/dv
  and d/dx together (the derivatives are kept for the backward pass);
* backward: grad * (d log K/dv, d log K/dx) from the forward's outputs -- no
  second launch;
* double backward (FP64): the second-order kernel (bessel_logk_hess_f64,
  the f^(n,m) with n + m = 2 in the same pass).

Argument marshalling only, like the rest of the binding: every value comes
from the CUDA kernels; the chain rule's products are the caller's autograd
graph.

    v = torch.tensor([2.5, 10.0], dtype=torch.float64, device="cuda", requires_grad=True)
    x = torch.tensor([1.0, 3.0], dtype=torch.float64, device="cuda", requires_grad=True)
    log_bessel_k_autograd(v, x).sum().backward()     # v.grad, x.grad
"""
from __future__ import annotations

import torch

from . import DEFAULT_NBINS, log_bessel_k, log_bessel_k_hess

__all__ = ["log_bessel_k_autograd"]


def _flat(v, x):
    if v.shape != x.shape:
        raise ValueError(f"v and x must have the same shape, got {tuple(v.shape)} and {tuple(x.shape)}")
    if v.dtype != x.dtype:
        raise TypeError("v and x must have the same dtype")
    return v.detach().reshape(-1).contiguous(), x.detach().reshape(-1).contiguous()


class _Derivs(torch.autograd.Function):
    """(d log K/dv, d log K/dx) as a differentiable function of (v, x), so that
    a graph built through the first derivatives (create_graph=True) reaches
    the second-order kernel."""

    @staticmethod
    def forward(ctx, v, x, nbins):
        vf, xf = _flat(v, x)
        dv, dx = log_bessel_k(vf, xf, nbins=nbins, outputs=("dv", "dx"))
        ctx.save_for_backward(v, x)
        ctx.nbins = nbins
        return dv.view_as(v), dx.view_as(x)

    @staticmethod
    def backward(ctx, gdv, gdx):
        v, x = ctx.saved_tensors
        if v.dtype != torch.float64:
            raise NotImplementedError("second derivatives are provided for float64 (bessel_logk_hess_f64)")
        vf, xf = _flat(v, x)
        _, _, _, dvv, dxx, dvx = log_bessel_k_hess(vf, xf, nbins=ctx.nbins)
        dvv, dxx, dvx = dvv.view_as(v), dxx.view_as(x), dvx.view_as(v)
        gv = gdv * dvv + gdx * dvx
        gx = gdv * dvx + gdx * dxx
        return gv, gx, None


class _LogBesselK(torch.autograd.Function):
    @staticmethod
    def forward(ctx, v, x, nbins):
        vf, xf = _flat(v, x)
        lk, dv, dx = log_bessel_k(vf, xf, nbins=nbins)
        ctx.save_for_backward(v, x, dv.view_as(v), dx.view_as(x))
        ctx.nbins = nbins
        return lk.view_as(v)

    @staticmethod
    def backward(ctx, g):
        v, x, dv, dx = ctx.saved_tensors
        if torch.is_grad_enabled():
            # create_graph: the derivatives as a differentiable function of (v, x)
            dv, dx = _Derivs.apply(v, x, ctx.nbins)
        return g * dv, g * dx, None


def log_bessel_k_autograd(v, x, nbins=DEFAULT_NBINS):
    """log K_v(x) of CUDA tensors (float64 or float32, same shape), differentiable
    in v and x (first order always, second order for float64)."""
    if not (isinstance(v, torch.Tensor) and isinstance(x, torch.Tensor) and v.is_cuda and x.is_cuda):
        raise TypeError("v and x must be CUDA tensors")
    return _LogBesselK.apply(v, x, int(nbins))
