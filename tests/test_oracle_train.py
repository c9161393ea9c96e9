"""Pins for oracle O7 (loss), O9 (Adam, LR) and O11 (sampler, CV).
Cites PAPER.md P:370 (loss/Adam/cosine), Eq. 14; SPEC examples."""
import math

import numpy as np
import pytest
import torch

from chg_inputs import mptrj_like_batch
from oracle.graph import build_graph_batch
from oracle.model import DT
from oracle.train import (LossConfig, adam_step, balance_assign, coefficient_of_variation,
                          cosine_lr, huber, init_lr, loss_terms)


class _Lab:
    def __init__(self, S, N):
        self.energy_per_atom = np.zeros(S); self.forces = np.zeros((N, 3))
        self.stress = np.zeros((S, 3, 3)); self.magmom = np.zeros(N); self.magmom_mask = np.ones(N, np.uint8)


def _out(S, N, e=0.0):
    return {"energy_per_atom": torch.full((S,), e, dtype=DT), "forces": torch.zeros(N, 3, dtype=DT),
            "stress": torch.zeros(S, 3, 3, dtype=DT), "magmom": torch.zeros(N, dtype=DT)}


def test_huber_loss_values(golden):
    lab = _Lab(1, 4)
    assert float(loss_terms(_out(1, 4), lab, LossConfig(), 1, 4, 4)["total"]) == 0.0
    e = 0.05                                        # |e| < δ: energy term = 2·½e² = e²
    assert float(loss_terms(_out(1, 4, e), lab, LossConfig(), 1, 4, 4)["E"]) == pytest.approx(e * e, rel=1e-14)
    v = float(loss_terms(_out(1, 4, 1.0), lab, LossConfig(), 1, 4, 4)["E"])
    assert v == pytest.approx(golden["huber_e1_delta01_energy_term"]["value"], rel=1e-14)
    # Huber is C¹ at |x| = δ
    x = torch.tensor([0.1 - 1e-9, 0.1 + 1e-9], dtype=DT)
    h = huber(x, 0.1)
    assert abs(float(h[1] - h[0])) < 1e-9


def test_global_normalisers_make_shards_additive():
    """Q23/§8(b): with global normalisers, per-shard losses sum to the full-batch loss."""
    b = mptrj_like_batch(3, seed=7)
    rng = np.random.default_rng(0)
    S, N = b.n_struct, b.n_atoms
    out = {"energy_per_atom": torch.as_tensor(rng.normal(-5, 1, S)),
           "forces": torch.as_tensor(rng.normal(0, .3, (N, 3))),
           "stress": torch.as_tensor(rng.normal(0, 1, (S, 3, 3))),
           "magmom": torch.as_tensor(rng.normal(size=N))}
    M = int(b.magmom_mask.sum())
    full = float(loss_terms(out, b, LossConfig(), S, N, M)["total"])
    from chg_inputs import split_batch
    tot = 0.0
    for ids in ([0], [1, 2]):
        sb = split_batch(b, ids)
        atoms = np.concatenate([np.arange(b.atom_ptr[s], b.atom_ptr[s + 1]) for s in ids])
        o = {"energy_per_atom": out["energy_per_atom"][ids], "forces": out["forces"][atoms],
             "stress": out["stress"][ids], "magmom": out["magmom"][atoms]}
        lc = LossConfig(n_struct_global=S, n_atoms_global=N, n_magmom_global=M)
        tot += float(loss_terms(o, sb, lc, len(ids), len(atoms), int(sb.magmom_mask.sum()))["total"])
    assert tot == pytest.approx(full, rel=1e-13)


def test_lr_rule(golden):
    assert init_lr(2048) == pytest.approx(golden["lr_bs2048"]["value"], rel=1e-15)
    assert init_lr(128) == pytest.approx(golden["lr_bs128"]["value"], rel=1e-15)
    assert init_lr(64) == pytest.approx(1.5e-4, rel=1e-15)
    assert cosine_lr(0, 100, 1e-3) == 1e-3
    assert cosine_lr(100, 100, 1e-3) == pytest.approx(0.0, abs=1e-20)
    assert cosine_lr(50, 100, 1e-3) == pytest.approx(5e-4, rel=1e-12)


def test_adam_first_step():
    """Bias-corrected first step with g constant moves θ by −lr·sign(g)."""
    th = np.array([1.0, -2.0, 3.0])
    g = np.array([0.5, -3.0, 1e-3])
    t1, m, v = adam_step(th, np.zeros(3), np.zeros(3), g, 1, 1e-3)
    np.testing.assert_allclose(t1 - th, -1e-3 * np.sign(g), rtol=1e-4)
    t0, _, _ = adam_step(th, np.zeros(3), np.zeros(3), np.zeros(3), 1, 1e-3)
    np.testing.assert_array_equal(t0, th)


def test_sampler(golden):
    loads = list(range(1, 9))
    out = balance_assign(loads, 2)
    got = [[loads[i] for i in r] for r in out]
    assert got == golden["sampler_1to8_w2"]["value"]
    assert coefficient_of_variation([sum(x) for x in got]) == 0.0
    assert coefficient_of_variation([10, 30]) == pytest.approx(golden["cv_10_30"]["value"])
    assert balance_assign(loads, 1) == [sorted(range(8), key=lambda i: loads[i])[::1][:1] +
                                         balance_assign(loads, 1)[0][1:]]
    with pytest.raises(ValueError):
        balance_assign(loads, 0)
    # completeness on a random long-tail batch
    rng = np.random.default_rng(1)
    L = rng.lognormal(4, 1, size=257).astype(int) + 1
    a = balance_assign(list(L), 8)
    assert sorted(sum(a, [])) == list(range(257))


def test_sampler_improves_cv_directionally(golden):
    """CV 0.186 → 0.064.  Directional analogue: on long-tail batches the
    balanced assignment beats a contiguous split in ≥ 95 % of trials."""
    rng = np.random.default_rng(2)
    wins, ratios = 0, []
    for _ in range(200):
        L = rng.lognormal(7, 1.0, size=1024)          # 1024 samples, W = 4
        cont = [L[i * 256:(i + 1) * 256].sum() for i in range(4)]
        bal = [sum(L[j] for j in r) for r in balance_assign(list(L), 4)]
        c0, c1 = coefficient_of_variation(cont), coefficient_of_variation(bal)
        wins += c1 < c0
        ratios.append(c0 / max(c1, 1e-12))
    assert wins >= 190
    assert np.median(ratios) >= 2.0
