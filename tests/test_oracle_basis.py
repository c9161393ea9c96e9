"""Pins for oracle O2 (basis) and O4's LayerNorm: closed forms and quadrature.
Cites: PAPER.md Eq. 12/13; SURVEY §8(c) O2."""
import math

import numpy as np
import pytest
import torch

from oracle.model import envelope, fourier, layer_norm, srbf

DT = torch.float64


@pytest.mark.parametrize("p", [6, 8, 10])
def test_envelope_endpoints(p):
    x = torch.tensor([0.0, 1.0], dtype=DT, requires_grad=True)
    u = envelope(x, p)
    (du,) = torch.autograd.grad(u.sum(), x)
    assert float(u[0].detach()) == 1.0
    assert abs(float(u[1].detach())) < 1e-12           # u(1) = 0
    assert abs(float(du[1])) < 1e-10          # u'(1) = 0 (smooth cutoff)
    # second derivative at 1 is also forced to zero by the DimeNet polynomial
    xx = torch.tensor([1.0], dtype=DT, requires_grad=True)
    (g1,) = torch.autograd.grad(envelope(xx, p).sum(), xx, create_graph=True)
    (g2,) = torch.autograd.grad(g1.sum(), xx)
    assert abs(float(g2)) < 1e-9


def test_envelope_half(golden):
    u = envelope(torch.tensor([0.5], dtype=DT), 8)
    assert float(u) == pytest.approx(golden["envelope_half_p8"]["value"], abs=1e-15)


def test_paper_printed_envelopes_are_not_smooth():
    """Documents reading Q2: Eq. 12 as printed gives u(1) = -4 and Eq. 13 gives
    u(1) = -84 at p = 8, so neither printed form is a cutoff envelope."""
    p, x = 8, 1.0
    eq12 = 1 - (p + 1) * (p + 2) / 2 * x ** p + p * (p + 2) * x ** (p + 1) - p * (p + 2) / 2 * x ** (p + 2)
    eq13 = 1 - (p + 2) / 2 * ((p + 1) * x ** p + 2 * p * x ** (p + 1) - p * x ** (p + 2))
    assert eq12 == -4.0 and eq13 == -84.0
    assert abs(float(envelope(torch.tensor([1.0], dtype=DT), p))) < 1e-12


def test_srbf_cutoff_and_orthonormality():
    freq = torch.arange(1, 32, dtype=DT) * math.pi
    rc = 5.0
    z = srbf(torch.tensor([rc], dtype=DT), freq, rc, 8)
    assert torch.all(torch.abs(z) < 1e-12)                 # ẽ(r_c) = 0
    # Without the envelope the DimeNet radial functions sqrt(2/rc) sin(nπr/rc)/r
    # are orthonormal under the r² dr measure on [0, rc].
    r = torch.linspace(1e-6, rc * (1 - 1e-5), 200001, dtype=DT)   # u(rc)=0: avoid 0/0
    f = srbf(r, freq, rc, 8) / envelope(r / rc, 8)[:, None]
    w = r * r
    gram = torch.trapezoid(f[:, :, None] * f[:, None, :] * w[:, None, None], r, dim=0)
    np.testing.assert_allclose(gram.numpy(), np.eye(31), atol=2e-4)


def test_fourier_closed_forms():
    th = torch.tensor([0.0, math.pi / 2], dtype=DT)
    F = fourier(th, 31).numpy()
    s2p, sp = 1 / math.sqrt(2 * math.pi), 1 / math.sqrt(math.pi)
    exp0 = [s2p] + [sp, 0.0] * 15
    np.testing.assert_allclose(F[0], exp0, atol=1e-15)
    exp90 = [s2p]
    for k in range(1, 16):
        exp90 += [math.cos(k * math.pi / 2) * sp, math.sin(k * math.pi / 2) * sp]
    np.testing.assert_allclose(F[1], exp90, atol=1e-14)
    # orthonormal on [0, 2π]
    t = torch.linspace(0, 2 * math.pi, 100001, dtype=DT)
    B = fourier(t, 31)
    gram = torch.trapezoid(B[:, :, None] * B[:, None, :], t, dim=0)
    np.testing.assert_allclose(gram.numpy(), np.eye(31), atol=1e-4)


def test_layernorm_example(golden):
    v = golden["layernorm_123"]
    y = layer_norm(torch.tensor([1.0, 2.0, 3.0], dtype=DT), torch.ones(3, dtype=DT), torch.zeros(3, dtype=DT))
    np.testing.assert_allclose(y.numpy(), v["value"], atol=v["tol"])
