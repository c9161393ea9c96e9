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


def _model(ctx, prec=0):
    cfg = chg.default_model_cfg(); cfg.mlp_precision = prec
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


# ---- NEXT-2: fixed-topology (skin) graphs and the captured MD step --------------------------

def _cons(ctx, m, g):
    out = ctx.forward_conservative(m, g)
    return out["energy"].astype(np.float64), out["forces"].astype(np.float64)


def test_skin_graph_equals_exact_lists(ctx):
    """Pairs of a skin graph beyond the model cutoffs carry zero bases (clamped envelope, reading
    Q2): energy and conservative forces equal the exact lists' (summation order aside), at the
    build positions and after chg_graph_refresh at displaced ones; the moved flag follows skin/2."""
    import torch
    b = si_diamond()
    m = _model(ctx)
    pos = torch.as_tensor(b.positions, device="cuda").contiguous()
    lat = torch.as_tensor(b.lattice, device="cuda").contiguous()
    sp = torch.as_tensor(b.species, device="cuda").contiguous()
    gs = ctx.build_graph(b.atom_ptr, pos, lat, sp, 5.0, 3.0, skin=1.0)
    ge = ctx.build_graph(b.atom_ptr, pos, lat, sp, 5.0, 3.0)
    ns, ne = gs.counts(), ge.counts()
    assert all(x >= y for x, y in zip(ns, ne)) and ns[1] > ne[1] and ns[2] > ne[2]   # strictly more pairs / bonds
    es, fs = _cons(ctx, m, gs)
    ee, fe = _cons(ctx, m, ge)
    assert np.abs(es - ee).max() <= 1e-5 * max(1.0, np.abs(ee).max())
    assert np.abs(fs - fe).max() <= 1e-5
    ge.close()
    # displaced positions: refresh the skin graph, compare with exact lists built there
    rng = np.random.default_rng(3)
    x1 = b.positions + rng.uniform(-0.2, 0.2, b.positions.shape)       # |dx| < skin / 2
    pos.copy_(torch.as_tensor(x1, device="cuda"))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx.refresh_graph(gs, pos, flag)
    es, fs = _cons(ctx, m, gs)
    ge = ctx.build_graph(b.atom_ptr, pos, lat, sp, 5.0, 3.0)
    ee, fe = _cons(ctx, m, ge)
    assert np.abs(es - ee).max() <= 1e-5 * max(1.0, np.abs(ee).max())
    assert np.abs(fs - fe).max() <= 1e-5
    ctx.sync()
    assert int(flag.item()) == 0
    pos[0, 0] += 1.0                                                   # one atom beyond skin / 2 (|x1 - x0| <= 0.2)
    torch.cuda.synchronize()
    ctx.refresh_graph(gs, pos, flag)
    ctx.sync()
    assert int(flag.item()) == 1
    gs.close(); ge.close(); m.close()


@pytest.mark.parametrize("prec", [0, 1])
def test_captured_md_step_matches_uncaptured(ctx, prec):
    """chg_md_capture / chg_md_run replay exactly the skin-graph step enqueued call by call, and
    the skin MD trajectory follows the rebuilt-every-step one (fp32 CUDA cores and 3xTF32
    tensor cores inside the captured graph)."""
    b = si_diamond()
    mass = np.full(b.positions.shape[0], 28.0855)
    v0 = maxwell_boltzmann(mass, 300.0, seed=4)
    m = _model(ctx, prec)
    runs = {}
    for name, kw in (("rebuild", {}), ("skin", dict(skin=1.0)), ("captured", dict(skin=1.0, captured=True))):
        md = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, v0, dt_fs=0.5, **kw)
        md.step(30)
        runs[name] = (md.pos.cpu().numpy().copy(), md.vel.cpu().numpy().copy(), md.total_energy())
        md.close()
    assert np.array_equal(runs["skin"][0], runs["captured"][0])
    assert np.array_equal(runs["skin"][1], runs["captured"][1])
    assert np.abs(runs["skin"][0] - runs["rebuild"][0]).max() < 1e-6
    assert np.abs(runs["skin"][2] - runs["rebuild"][2]).max() < 1e-5
    m.close()


def test_captured_md_rebuilds_when_atoms_move(ctx):
    """A fast atom trips the skin / 2 flag: the lists are rebuilt and the step re-captured, and
    the trajectory still follows the rebuilt-every-step one."""
    b = si_diamond()
    mass = np.full(b.positions.shape[0], 28.0855)
    v0 = np.zeros_like(b.positions)
    v0[0] = (0.02, 0.0, 0.0)                                           # 0.02 Å/fs: 0.3 Å per 30 steps
    m = _model(ctx)
    ref = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, v0, dt_fs=0.5)
    ref.step(60)
    md = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, v0, dt_fs=0.5, skin=0.4, captured=True,
             check_every=5)
    md.step(60)
    assert md.rebuilds >= 2
    assert np.abs(md.pos.cpu().numpy() - ref.pos.cpu().numpy()).max() < 1e-6
    md.close(); ref.close(); m.close()


def test_refresh_geometry_is_bit_identical_to_a_fresh_build(ctx):
    """chg_graph_refresh evaluates each listed pair by the build's canonical fp64 expression: the
    refreshed vectors equal, bit for bit, those of a graph built afresh at the new positions
    (pairs present in both lists; the pair sets may differ at the list cutoff)."""
    import torch
    b = si_diamond()
    pos = torch.as_tensor(b.positions, device="cuda").contiguous()
    lat = torch.as_tensor(b.lattice, device="cuda").contiguous()
    sp = torch.as_tensor(b.species, device="cuda").contiguous()
    gs = ctx.build_graph(b.atom_ptr, pos, lat, sp, 5.0, 3.0, skin=0.6)
    x1 = b.positions + np.random.default_rng(5).uniform(-0.25, 0.25, b.positions.shape)
    pos.copy_(torch.as_tensor(x1, device="cuda"))
    torch.cuda.synchronize()
    ctx.refresh_graph(gs, pos)
    gf = ctx.build_graph(b.atom_ptr, pos, lat, sp, 5.0, 3.0, skin=0.6)
    ctx.sync()

    def pairs(g):
        x = g.export()
        rp, out = x["row_ptr"], {}
        for i in range(len(rp) - 1):
            for e in range(rp[i], rp[i + 1]):
                out[(i, int(x["nbr"][e]), tuple(int(t) for t in x["img"][e]))] = x["vec"][e]
        return out

    ps, pf = pairs(gs), pairs(gf)
    common = set(ps) & set(pf)
    assert len(common) > 0.95 * max(len(ps), len(pf))
    for k in common:
        assert np.array_equal(ps[k], pf[k]), k
    gs.close(); gf.close()
