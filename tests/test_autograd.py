"""torch.autograd binding (paper_2108_11560_b200/autograd.py): the gradients
are the kernel's own derivative outputs (Sec. 4.1), checked
against finite differences of the kernel's log K (gradcheck) and, for the
second order, against the Hessian kernel (gradgradcheck)."""
import numpy as np
import pytest
import torch

from paper_2108_11560_b200.autograd import log_bessel_k_autograd


def test_rejects_cpu_tensors():
    with pytest.raises(TypeError):
        log_bessel_k_autograd(torch.ones(3, dtype=torch.float64), torch.ones(3, dtype=torch.float64))


def _inputs(n, dt, seed=3):
    rng = np.random.default_rng(seed)
    v = torch.tensor(rng.uniform(-20, 20, n), dtype=dt, device="cuda")
    x = torch.tensor(10.0 ** rng.uniform(-1, 1.5, n), dtype=dt, device="cuda")
    return v, x


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [torch.float64, torch.float32])
def test_backward_is_the_kernels_derivatives(dt):
    import paper_2108_11560_b200 as blk
    v, x = _inputs(600, dt)
    v2, x2 = v.reshape(20, 30).clone().requires_grad_(), x.reshape(20, 30).clone().requires_grad_()
    lk = log_bessel_k_autograd(v2, x2)
    g = torch.linspace(-1.0, 2.0, 600, dtype=dt, device="cuda").reshape(20, 30)
    lk.backward(g)
    ref_lk, ref_dv, ref_dx = blk.log_bessel_k(v, x)   # the same (automatic) lanes per element
    torch.cuda.synchronize()
    assert lk.shape == (20, 30)
    assert torch.equal(lk.detach().reshape(-1), ref_lk)
    assert torch.equal(v2.grad.reshape(-1), g.reshape(-1) * ref_dv)
    assert torch.equal(x2.grad.reshape(-1), g.reshape(-1) * ref_dx)


@pytest.mark.gpu
def test_gradcheck_fp64():
    v, x = _inputs(24, torch.float64, seed=5)
    v = v.clone().requires_grad_()
    x = x.clone().requires_grad_()
    assert torch.autograd.gradcheck(lambda a, b: log_bessel_k_autograd(a, b), (v, x),
                                    eps=1e-6, atol=1e-6, rtol=1e-5)


@pytest.mark.gpu
def test_gradgradcheck_fp64():
    v, x = _inputs(16, torch.float64, seed=7)
    v = v.clone().requires_grad_()
    x = x.clone().requires_grad_()
    assert torch.autograd.gradgradcheck(lambda a, b: log_bessel_k_autograd(a, b), (v, x),
                                        eps=1e-6, atol=1e-5, rtol=1e-4)


@pytest.mark.gpu
def test_second_order_fp32_not_provided():
    v, x = _inputs(8, torch.float32)
    v = v.clone().requires_grad_()
    (g,) = torch.autograd.grad(log_bessel_k_autograd(v, x).sum(), v, create_graph=True)
    with pytest.raises(NotImplementedError):
        g.sum().backward()
