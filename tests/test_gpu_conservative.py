"""Conservative forces / stress of the energy head through the C ABI (chg_forward_conservative,
SURVEY §8(f) NEXT-1) against the oracle's autograd derivative (O10: F = −∂E/∂r,
σ = (160.21766208/V)·∂E/∂ε, pinned by central finite differences in test_oracle_model.py).

Bars: fp32 mode — forces ≤ 1e-4 eV/Å, stress ≤ 1e-4 GPa, E/atom ≤ 1e-5 rel (NS); TF32 mode —
‖ΔF‖/‖F‖ and ‖Δσ‖/‖σ‖ ≤ 2e-3 (NS loosened).  The pass must leave parameter gradients untouched
and consume the train-mode activations (a following chg_backward is refused).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from chg_inputs import init_flat_params, make_config_batch, si_diamond, skewed_oxide_batch  # noqa: E402
from oracle.graph import build_graph_batch  # noqa: E402
from oracle.model import ModelConfig, derived_force_stress, param_layout  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402

pytestmark = pytest.mark.gpu
CFG = ModelConfig()


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    c = chg.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def params():
    p = init_flat_params(param_layout(CFG), seed=0, bias_scale=0.1)
    return p.astype(np.float32).astype(np.float64)


CASES = {"si_jitter": lambda: si_diamond(jitter=0.05, seed=7), "c2_8": lambda: make_config_batch("C2", 0, n_struct=8),
         "oxides": lambda: skewed_oxide_batch(3, seed=79)}


def _rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12)


@pytest.mark.parametrize("prec", sorted(chg.PRECISION_MODES))
@pytest.mark.parametrize("case", list(CASES))
def test_conservative_forces_stress(ctx, params, case, prec):
    b = CASES[case]()
    og = build_graph_batch(b)
    ref = derived_force_stress(og, b.positions, b.lattice, b.species, params, CFG)
    cfg = chg.default_model_cfg(); cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    m.set_params(params.astype(np.float32))
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    out = ctx.forward_conservative(m, g)
    F, S = ref["forces"].detach().numpy(), ref["stress"].detach().numpy()
    E = ref["energy"].detach().numpy()
    natoms = np.diff(b.atom_ptr)
    if prec in (0, 1):  # fp32 strict and 3xTF32: the NS F / sigma / E bars
                        # (TF32: F and sigma are position / strain GRADIENTS: NS-loosened 2e-3 relative;
                        # BF16: 2e-2 relative)
        assert np.max(np.abs(out["forces"] - F)) <= 1e-4, np.max(np.abs(out["forces"] - F))
        assert np.max(np.abs(out["stress"] - S)) <= 1e-4, np.max(np.abs(out["stress"] - S))
        epa = E / natoms
        assert np.all(np.abs(out["energy_per_atom"] - epa) <= 1e-5 * np.maximum(np.abs(epa), 1.0))
    else:
        bar = 2e-3 if prec == 2 else 2e-2
        assert _rel(out["forces"], F) <= bar, _rel(out["forces"], F)
        assert _rel(out["stress"], S) <= bar, _rel(out["stress"], S)
    # parameter gradients untouched; the activations were consumed
    assert np.all(m.grads() == 0)
    with pytest.raises(chg.ChgError) as e:
        ctx.backward(m, g, dict(energy_per_atom=b.energy_per_atom.astype(np.float32),
                                forces=b.forces.astype(np.float32), stress=b.stress.astype(np.float32),
                                magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask))
    assert e.value.name == "CHG_ERR_STATE"
    g.close(); m.close()


def test_conservative_translation_invariance(ctx, params):
    """Σ_i F_i = 0 (translation invariance of E) and σ symmetric (rotation invariance)."""
    b = make_config_batch("C2", 1, n_struct=6)
    m = chg.Model(ctx)
    m.set_params(params.astype(np.float32))
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    out = ctx.forward_conservative(m, g)
    for s in range(b.n_struct):
        a0, a1 = b.atom_ptr[s], b.atom_ptr[s + 1]
        f = out["forces"][a0:a1].astype(np.float64)
        assert np.max(np.abs(f.sum(0))) <= 1e-4 * max(1.0, np.abs(f).max() * (a1 - a0))
        st = out["stress"][s].astype(np.float64)
        assert np.max(np.abs(st - st.T)) <= 1e-4 * max(1.0, np.abs(st).max())
    g.close(); m.close()
