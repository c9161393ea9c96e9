"""Captured training step (chg_capture_step / chg_exec_step: one CUDA graph per (model, graph))
and the deferred finite check (chg_adam_cfg.defer_check), through the C ABI.

* Replaying the captured step K times gives parameters, Adam moments and gradients
  BIT-IDENTICAL to K ordinary forward / backward / step calls (same kernels, same order, fixed
  reduction trees) in every precision mode.
* A non-finite gradient under defer_check: chg_step returns OK without synchronising, the
  update is skipped on the device, and the next call reports CHG_ERR_NONFINITE naming the
  tensor.
* A capture is refused after a ctx workspace was re-allocated (CHG_ERR_STATE)."""
import numpy as np
import pytest

from chg_inputs import init_flat_params, make_config_batch

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2412_20796_b200 import chg  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = chg.Context(0)
    yield c
    c.close()


def _dev_labels(b):
    f = lambda x: torch.as_tensor(np.asarray(x, np.float32), device="cuda").contiguous()  # noqa: E731
    return dict(energy_per_atom=f(b.energy_per_atom), forces=f(b.forces), stress=f(b.stress), magmom=f(b.magmom),
                magmom_mask=torch.as_tensor(b.magmom_mask, device="cuda").contiguous())


def _model(ctx, prec):
    cfg = chg.default_model_cfg()
    cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0, bias_scale=0.1).astype(np.float32))
    return m


@pytest.mark.parametrize("prec", sorted(chg.PRECISION_MODES))
def test_captured_step_bit_identical(ctx, prec):
    b = make_config_batch("C2", 1, n_struct=12)
    lab = _dev_labels(b)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    m1, m2 = _model(ctx, prec), _model(ctx, prec)
    lrs = [3e-4, 2e-4, 1e-4]
    for k, lr in enumerate(lrs):
        ctx.forward(m1, g, train=True, host=False)
        ctx.backward(m1, g, lab, sync_loss=False)
        ctx.step(m1, lr=lr, step=k + 1)
    x = ctx.capture_step(m2, g, lab)
    for k, lr in enumerate(lrs):
        x.step(lr, k + 1)
    ctx.sync()
    for which in (0, 1, 2, 3):
        np.testing.assert_array_equal(m2.get(which), m1.get(which), err_msg=str(which))
    assert np.any(m2.params() != init_flat_params([(n, s) for n, s, _ in m2.layout()], seed=0,
                                                  bias_scale=0.1).astype(np.float32))
    x.close(); g.close(); m1.close(); m2.close()


def test_deferred_nonfinite_check(ctx):
    b = make_config_batch("C2", 2, n_struct=4)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    m = _model(ctx, 0)
    p0 = m.params()
    ctx.forward(m, g, train=True, host=False)
    ctx.backward(m, g, _dev_labels(b), sync_loss=False)
    grads = m.grads()
    names = [n for n, _, _ in m.layout()]
    offs = [o for _, _, o in m.layout()]
    k = names.index("bond1.gate.W1")
    grads[offs[k] + 5] = np.nan
    m.set(1, grads)
    ctx.step(m, lr=3e-4, step=1, defer_check=True)          # returns without synchronising
    with pytest.raises(chg.ChgError) as e:
        ctx.sync()
    assert e.value.name == "CHG_ERR_NONFINITE" and "bond1.gate.W1" in str(e.value)
    np.testing.assert_array_equal(m.params(), p0)           # the update was skipped on the device
    ctx.sync()                                               # reported once
    g.close(); m.close()


def test_capture_refused_after_workspace_growth(ctx):
    small = make_config_batch("C2", 3, n_struct=2)
    big = make_config_batch("C3", 3, n_struct=64)
    m = _model(ctx, 2)
    gs = ctx.build_graph(small.atom_ptr, small.positions, small.lattice, small.species)
    x = ctx.capture_step(m, gs, _dev_labels(small))
    x.step(1e-4, 1)
    gb = ctx.build_graph(big.atom_ptr, big.positions, big.lattice, big.species)
    ctx.forward(m, gb, train=True, host=False)               # grows the workspaces
    with pytest.raises(chg.ChgError) as e:
        x.step(1e-4, 2)
    assert e.value.name == "CHG_ERR_STATE"
    ctx.sync()
    x.close(); gs.close(); gb.close(); m.close()
