"""MD inference loop: velocity-Verlet NVE through the C ABI
(chg_md_verlet + chg_build_graph from device positions + chg_forward_conservative)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from chg_inputs import init_flat_params, si_diamond  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402
from paper_2412_20796_b200.md import NVE, maxwell_boltzmann  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    c = chg.Context(0)
    yield c
    c.close()


def _model(ctx):
    cfg = chg.default_model_cfg(); cfg.mlp_precision = 0
    m = chg.Model(ctx, cfg)
    m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
    return m


def test_verlet_half_steps_match_the_formula(ctx):
    import torch
    rng = np.random.default_rng(0)
    n, dt = 37, 0.7
    x, v = rng.normal(size=(n, 3)), rng.normal(size=(n, 3)) * 0.01
    f, m = rng.normal(size=(n, 3)).astype(np.float32), rng.uniform(1, 200, n)
    cu = lambda a: torch.as_tensor(a, device="cuda").contiguous()
    X, V, F, IM = cu(x), cu(v), cu(f), cu(1.0 / m)
    ctx.md_verlet(X, V, F, IM, dt, drift=True)
    c = 9.648533212e-3
    v1 = v + 0.5 * dt * c * f.astype(np.float64) / m[:, None]
    x1 = x + dt * v1
    np.testing.assert_allclose(V.cpu().numpy(), v1, rtol=0, atol=1e-15)
    np.testing.assert_allclose(X.cpu().numpy(), x1, rtol=0, atol=1e-15)
    ctx.md_verlet(X, V, F, IM, dt, drift=False)
    np.testing.assert_allclose(V.cpu().numpy(), v1 + 0.5 * dt * c * f.astype(np.float64) / m[:, None], rtol=0,
                               atol=1e-15)
    np.testing.assert_allclose(X.cpu().numpy(), x1, rtol=0, atol=0)


def test_nve_conserves_energy(ctx):
    b = si_diamond()
    mass = np.full(b.positions.shape[0], 28.0855)
    v0 = maxwell_boltzmann(mass, 300.0, seed=1)
    m = _model(ctx)
    md = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, v0, dt_fs=0.5)
    e0 = md.total_energy()
    ke0 = md.kinetic_energy()
    drift = []
    for _ in range(20):
        md.step(10)
        drift.append(float(np.abs(md.total_energy() - e0).max()))
    assert np.all(np.isfinite(drift))
    # 200 steps of 0.5 fs: |ΔE_total| stays a small fraction of the kinetic energy scale
    assert max(drift) < 0.02 * float(ke0.max()) + 1e-4, (drift, ke0)
    assert float(np.abs(md.kinetic_energy() - ke0).max()) > 0      # the system moved
    m.close()


def test_nve_time_reversible(ctx):
    b = si_diamond()
    mass = np.full(b.positions.shape[0], 28.0855)
    m = _model(ctx)
    md = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, maxwell_boltzmann(mass, 300.0, 2), 0.5)
    x0 = md.pos.cpu().numpy().copy()
    md.step(20)
    md.vel.neg_()
    md.step(20)
    assert np.abs(md.pos.cpu().numpy() - x0).max() < 1e-5
    m.close()
