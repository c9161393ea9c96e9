"""Host logic of the training loop (CPU): Eq. 14 and the cosine schedule against the oracle's
independent definitions, and the LJ-toy data's forces against finite differences."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from chg_inputs import lj_dataset, lj_labels  # noqa: E402
from oracle.train import cosine_lr as o_cos, init_lr as o_init  # noqa: E402
from paper_2412_20796_b200.train import cosine_lr, init_lr  # noqa: E402


def test_lr_schedule_matches_oracle():
    assert init_lr(2048) == o_init(2048) and abs(init_lr(2048) - 0.0048) < 1e-15
    for step in (1, 7, 50, 100):
        assert cosine_lr(step, 100, 1e-3) == o_cos(step, 100, 1e-3)
    assert abs(cosine_lr(100, 100, 1e-3)) < 1e-18


def test_lj_data_forces_and_stress_finite_difference():
    b = lj_dataset(2, seed=3)
    L = b.lattice[0]; pos = b.positions[:b.atom_ptr[1]].copy()
    E, F, W = lj_labels(L, pos)
    h = 1e-5
    for (i, k) in [(0, 0), (1, 2)]:
        p = pos.copy(); p[i, k] += h; Ep = lj_labels(L, p)[0]
        p[i, k] -= 2 * h; Em = lj_labels(L, p)[0]
        assert abs(-(Ep - Em) / (2 * h) - F[i, k]) < 1e-6
    # strain derivative: r -> r(I+eps), L -> L(I+eps)
    for (k, c) in [(0, 0), (1, 2)]:
        ep = np.eye(3); ep[k, c] += h
        em = np.eye(3); em[k, c] -= h
        dE = (lj_labels(L @ ep, pos @ ep)[0] - lj_labels(L @ em, pos @ em)[0]) / (2 * h)
        assert abs(dE - W[k, c]) < 1e-6
    assert np.allclose(F.sum(0), 0, atol=1e-10)
