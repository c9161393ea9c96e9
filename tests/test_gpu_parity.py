"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star, reading Q30):
  graph lists bit-exact; vec = fp32(oracle d) exactly;
  E/atom |Δ| <= 1e-5·max(|ε|, 1 eV); F max-abs <= 1e-4 eV/Å; σ max-abs <= 1e-4 GPa;
  m max-abs <= 1e-5 μB; gradients per tensor ‖Δ‖/‖g‖ <= 1e-4 (fp32 path);
  intermediate features per tensor ‖Δ‖/‖ref‖ <= 1e-5.
Parameters and labels are rounded to fp32 once and given to BOTH sides.
"""
import numpy as np
import pytest

from chg_inputs import (Batch, concat_batches, dimer, init_flat_params, lifepo4_like_cell, make_config_batch,
                        mptrj_like_batch,
                        si_diamond, simple_cubic, skewed_oxide_batch)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle.graph import build_graph_batch  # noqa: E402
from oracle.model import ModelConfig, param_layout, run_forward  # noqa: E402
from oracle.train import LossConfig, adam_step, loss_and_grad  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402

CFG = ModelConfig()


@pytest.fixture(scope="module")
def ctx():
    c = chg.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def params():
    p = init_flat_params(param_layout(CFG), seed=0, bias_scale=0.1)
    return p.astype(np.float32).astype(np.float64)


def _gpu_graph(ctx, b, ra=5.0, rb=3.0):
    return ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species, ra, rb)


def _labels32(b):
    return dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
                stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32),
                magmom_mask=b.magmom_mask.astype(np.uint8))


def _labels64(b):
    lb = _labels32(b)
    return Batch(atom_ptr=b.atom_ptr, positions=b.positions, lattice=b.lattice, species=b.species,
                 energy_per_atom=lb["energy_per_atom"].astype(np.float64),
                 forces=lb["forces"].astype(np.float64), stress=lb["stress"].astype(np.float64),
                 magmom=lb["magmom"].astype(np.float64), magmom_mask=lb["magmom_mask"])


def _large_cell(n, edge, shear=0.0, shift=False, seed=3001):
    """A >= 256-atom cell with every width >= 3 cutoffs (cell-list path of the builder);
    optional shear (triclinic) and atoms moved by whole lattice vectors (wrapping)."""
    b = lifepo4_like_cell(n_atoms=n, edge=edge, seed=seed)
    L = b.lattice[0].copy()
    f = b.positions @ np.linalg.inv(L)
    if shear:
        L[1] += shear * L[0]
        L[2] += 0.5 * shear * L[1]
    if shift:
        rng = np.random.default_rng(seed)
        f = f + rng.integers(-1, 2, size=f.shape)
    pos = f @ L
    return Batch(atom_ptr=b.atom_ptr, positions=pos, lattice=L[None], species=b.species,
                 energy_per_atom=b.energy_per_atom, forces=b.forces, stress=b.stress, magmom=b.magmom,
                 magmom_mask=b.magmom_mask)


GRAPH_CASES = {
    "cells_300": lambda: _large_cell(300, 16.0),
    "cells_300_triclinic_shifted": lambda: _large_cell(300, 17.5, shear=0.12, shift=True),
    "si_diamond": lambda: si_diamond(),
    "si_diamond_r6": lambda: si_diamond(),
    "simple_cubic_r6": lambda: simple_cubic(3.0),
    "dimer": lambda: dimer(2.0),
    "isolated": lambda: dimer(7.0, 30.0),
    "c2": lambda: make_config_batch("C2"),
    "oxides": lambda: skewed_oxide_batch(6, seed=77),
    "jitter_si_2x2x1": lambda: si_diamond(jitter=0.05, reps=(2, 2, 1)),
}


@pytest.mark.parametrize("case", list(GRAPH_CASES))
def test_graph_bit_exact(ctx, case):
    b = GRAPH_CASES[case]()
    ra = 6.0 if case.endswith("r6") else 5.0
    og = build_graph_batch(b, ra, 3.0)
    gg = _gpu_graph(ctx, b, ra, 3.0)
    N, E, B, A = gg.counts()
    assert (N, E, B, A) == (og.n_atoms, og.n_edges, og.n_bonds, og.n_angles)
    ex = gg.export()
    for k, v in og.lists().items():
        np.testing.assert_array_equal(ex[k], v, err_msg=k)
    np.testing.assert_array_equal(ex["vec"][:, :3], og.d.astype(np.float32))
    np.testing.assert_array_equal(ex["vec"][:, 3], og.r.astype(np.float32))
    np.testing.assert_array_equal(gg.per_struct(), og.counts)


def test_graph_device_inputs(ctx):
    """Device-resident inputs: geometry validated on the GPU (k_geo); same lists as host inputs."""
    import torch
    b = make_config_batch("C2")
    og = build_graph_batch(b)
    gg = ctx.build_graph(b.atom_ptr, torch.as_tensor(b.positions, device="cuda"),
                         torch.as_tensor(b.lattice, device="cuda"), torch.as_tensor(b.species, device="cuda"))
    ex = gg.export()
    for k, v in og.lists().items():
        np.testing.assert_array_equal(ex[k], v, err_msg=k)
    np.testing.assert_array_equal(gg.per_struct(), og.counts)
    bad = b.lattice.copy(); bad[3] = 0.0
    with pytest.raises(chg.ChgError) as e:
        ctx.build_graph(b.atom_ptr, torch.as_tensor(b.positions, device="cuda"), torch.as_tensor(bad, device="cuda"),
                        torch.as_tensor(b.species, device="cuda"))
    assert e.value.name == "CHG_ERR_GEOMETRY" and "structure 3" in str(e.value)
    thin = b.lattice.copy(); thin[5, 2] *= 1e-3
    with pytest.raises(chg.ChgError) as e:
        ctx.build_graph(b.atom_ptr, torch.as_tensor(b.positions, device="cuda"), torch.as_tensor(thin, device="cuda"),
                        torch.as_tensor(b.species, device="cuda"))
    assert e.value.name == "CHG_ERR_GEOMETRY"


def test_graph_errors(ctx):
    b = si_diamond()
    with pytest.raises(chg.ChgError) as e:
        ctx.build_graph(b.atom_ptr, b.positions, np.zeros((1, 3, 3)), b.species)
    assert e.value.name == "CHG_ERR_GEOMETRY"
    with pytest.raises(chg.ChgError) as e:
        ctx.build_graph(b.atom_ptr, b.positions, b.lattice, np.full(8, 95, np.int32))
    assert e.value.name == "CHG_ERR_SPECIES"
    pos = b.positions.copy(); pos[1] = pos[0]
    with pytest.raises(chg.ChgError) as e:
        ctx.build_graph(b.atom_ptr, pos, b.lattice, b.species)
    assert e.value.name == "CHG_ERR_GEOMETRY"
    with pytest.raises(chg.ChgError) as e:
        ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species, 3.0, 5.0)
    assert e.value.name == "CHG_ERR_ARG"


def test_layout_matches_oracle(ctx):
    m = chg.Model(ctx)
    lay = m.layout()
    ref = param_layout(CFG)
    assert [x[0] for x in lay] == [x[0] for x in ref]
    assert [tuple(x[1]) for x in lay] == [tuple(x[1]) for x in ref]
    off = np.cumsum([0] + [int(np.prod(s)) for _, s in ref])[:-1]
    assert [x[2] for x in lay] == off.tolist()
    assert m.P == 430026


def _rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (n if n > 0 else 1.0)


FWD_CASES = {"si_jitter": lambda: si_diamond(jitter=0.05, seed=7), "c2": lambda: make_config_batch("C2"),
             "oxides": lambda: skewed_oxide_batch(4, seed=78)}


@pytest.mark.parametrize("case", list(FWD_CASES))
def test_forward_parity(ctx, params, case):
    b = FWD_CASES[case]()
    og = build_graph_batch(b)
    ref = run_forward(og, b.species, b.lattice, params, CFG, keep=True)
    m = chg.Model(ctx)
    m.set_params(params.astype(np.float32))
    gg = _gpu_graph(ctx, b)
    out = ctx.forward(m, gg, train=True)
    # intermediates (localise failures)
    for name, key in [("ea_t", "ea_t"), ("eb_t", "eb_t"), ("a_t", "a_t")]:
        got = ctx.debug(name)[:, :31]
        assert _rel(got, ref[key].detach().numpy()) < 1e-6, name
    for name in ["v0", "e0", "ea", "eb", "a0", "v1", "e1", "a1", "v2", "e2", "a2", "v3", "e3", "v4"]:
        got = ctx.debug(name)
        r = ref[name].detach().numpy()
        if r.size == 0:
            continue
        assert _rel(got, r) < 1e-5, (name, _rel(got, r))
    eps_ref = ref["energy_per_atom"].detach().numpy()
    assert np.all(np.abs(out["energy_per_atom"] - eps_ref) <= 1e-5 * np.maximum(np.abs(eps_ref), 1.0))
    assert np.max(np.abs(out["forces"] - ref["forces"].detach().numpy())) <= 1e-4
    assert np.max(np.abs(out["stress"] - ref["stress"].detach().numpy())) <= 1e-4
    assert np.max(np.abs(out["magmom"] - ref["magmom"].detach().numpy())) <= 1e-5


@pytest.mark.parametrize("case", ["si_jitter", "c2", "oxides"])
def test_backward_parity(ctx, params, case):
    b = _labels64(FWD_CASES[case]())
    og = build_graph_batch(b)
    terms, gref, _ = loss_and_grad(og, b, params, CFG, LossConfig())
    m = chg.Model(ctx)
    m.set_params(params.astype(np.float32))
    gg = _gpu_graph(ctx, b)
    ctx.forward(m, gg, train=True, host=False)
    loss = ctx.backward(m, gg, _labels32(b))
    for k, key in enumerate(["total", "E", "F", "S", "M"]):
        assert abs(loss[k] - terms[key]) <= 1e-5 * max(abs(terms[key]), 1e-6), key
    g = m.grads()
    off = 0
    for name, shape in param_layout(CFG):
        n = int(np.prod(shape))
        gr, gg_ = gref[off:off + n], g[off:off + n]
        off += n
        if np.all(gr == 0):
            assert np.all(gg_ == 0), name
            continue
        assert _rel(gg_, gr) <= 1e-4, (name, _rel(gg_, gr))


def test_backward_accumulates_and_is_deterministic(ctx, params):
    b = make_config_batch("C2")
    m = chg.Model(ctx)
    m.set_params(params.astype(np.float32))
    gg = _gpu_graph(ctx, b)
    ctx.forward(m, gg, train=True, host=False)
    ctx.backward(m, gg, _labels32(b))
    g1 = m.grads()
    m.set(1, np.zeros(m.P, np.float32))
    ctx.forward(m, gg, train=True, host=False)
    ctx.backward(m, gg, _labels32(b))
    g2 = m.grads()
    np.testing.assert_array_equal(g1, g2)           # bit-identical repeat (no atomics)
    ctx.forward(m, gg, train=True, host=False)
    ctx.backward(m, gg, _labels32(b))
    np.testing.assert_array_equal(m.grads(), g1 + g1)


def test_backward_needs_forward(ctx, params):
    b = si_diamond()
    m = chg.Model(ctx)
    m.set_params(params.astype(np.float32))
    g1 = _gpu_graph(ctx, b)
    g2 = _gpu_graph(ctx, b)
    ctx.forward(m, g1, train=True, host=False)
    with pytest.raises(chg.ChgError) as e:
        ctx.backward(m, g2, _labels32(b))
    assert e.value.name == "CHG_ERR_STATE"
    ctx.forward(m, g1, train=False, host=False)
    with pytest.raises(chg.ChgError) as e:
        ctx.backward(m, g1, _labels32(b))
    assert e.value.name == "CHG_ERR_STATE"


def test_adam_step_parity(ctx, params):
    """The fused Adam kernel against oracle Adam (O9) fed the SAME gradient
    (the oracle's, rounded to fp32), two steps so the bias corrections and the
    moment recursions are both exercised.  Tolerance: fp32 rounding of θ, m, v."""
    b = _labels64(make_config_batch("C2"))
    og = build_graph_batch(b)
    _, gref, _ = loss_and_grad(og, b, params, CFG, LossConfig())
    g32 = gref.astype(np.float32)
    g64 = g32.astype(np.float64)
    lr = 3e-4
    m = chg.Model(ctx)
    m.set_params(params.astype(np.float32))
    th, mm, vv = params.copy(), np.zeros_like(params), np.zeros_like(params)
    # the ABI takes β1, β2 as fp32 (chg_adam_cfg): give the oracle the same values
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    for step in (1, 2):
        th, mm, vv = adam_step(th, mm, vv, g64, step, lr, beta1=b1, beta2=b2)
        m.set(1, g32)
        ctx.step(m, lr=lr, step=step)
        assert np.all(m.grads() == 0)               # gradients zeroed by the step
        np.testing.assert_allclose(m.params(), th, rtol=0, atol=1e-6 * lr + 2e-7 * np.abs(th).max())
        np.testing.assert_allclose(m.get(2), mm, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(m.get(3), vv, rtol=1e-5, atol=1e-18)


def test_training_step_end_to_end(ctx, params):
    """build → forward → backward → Adam through the ABI: the update direction
    matches the oracle's wherever the oracle gradient is clearly non-zero."""
    b = _labels64(make_config_batch("C2"))
    og = build_graph_batch(b)
    _, gref, _ = loss_and_grad(og, b, params, CFG, LossConfig())
    lr = 3e-4
    m = chg.Model(ctx)
    p32 = params.astype(np.float32)
    m.set_params(p32)
    gg = _gpu_graph(ctx, b)
    ctx.forward(m, gg, train=True, host=False)
    ctx.backward(m, gg, _labels32(b))
    ctx.step(m, lr=lr, step=1)
    d = m.params().astype(np.float64) - p32
    ulp = np.spacing(np.abs(p32) + np.float32(lr)).astype(np.float64)   # fp32 rounding of θ - lr·ĝ
    assert np.all(np.abs(d) <= lr * 1.001 + ulp)
    big = np.abs(gref) > 1e-4 * np.abs(gref).max()
    assert np.mean(np.sign(d[big]) == -np.sign(gref[big])) > 0.999


def test_nonfinite_gradient_leaves_state(ctx, params):
    b = si_diamond(jitter=0.05)
    p = params.astype(np.float32).copy()
    lay = {n: (s, o) for n, s, o in chg.Model(ctx).layout()}
    s, o = lay["atom0.core.W1"]
    p[o] = np.nan                                   # -> NaN features and gradients (Huber' alone is bounded)
    m = chg.Model(ctx)
    m.set_params(p)
    gg = _gpu_graph(ctx, b)
    ctx.forward(m, gg, train=True, host=False)
    ctx.backward(m, gg, _labels32(b))
    before = m.params().copy()
    with pytest.raises(chg.ChgError) as e:
        ctx.step(m, lr=1e-3, step=1)
    assert e.value.name == "CHG_ERR_NONFINITE"
    np.testing.assert_array_equal(m.params(), before)
    assert np.all(m.get(2) == 0) and np.all(m.get(3) == 0)
