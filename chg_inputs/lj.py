"""LJ-toy dataset: small periodic argon-like cells labelled by a
Lennard-Jones pair potential, so a training run can show learning without MPtrj.

The labels are the DATA's ground truth (a textbook pair potential evaluated in fp64 numpy),
not any arithmetic of the method: energies per atom (eV), forces (eV/Å), stress (GPa, sign
convention of the model: σ = (1/V)·∂E/∂ε), no magnetic moments (mask all zero).
"""
from __future__ import annotations

import numpy as np

from .structures import Batch, _place

EV_A3_TO_GPA = 160.21766208


def lj_labels(L: np.ndarray, pos: np.ndarray, eps: float = 0.0104, sig: float = 3.4, rc: float = 6.0):
    """Shifted-energy LJ over all periodic images within rc: (E, F [n,3], dE/dε [3,3])."""
    n = pos.shape[0]
    rng_im = int(np.ceil(rc / np.min(np.abs(np.linalg.det(L)) / np.linalg.norm(
        np.cross(L[[1, 2, 0]], L[[2, 0, 1]]), axis=1)))) + 1
    shifts = np.array([(a, b, c) for a in range(-rng_im, rng_im + 1) for b in range(-rng_im, rng_im + 1)
                       for c in range(-rng_im, rng_im + 1)], np.float64) @ L
    e_rc = 4 * eps * ((sig / rc) ** 12 - (sig / rc) ** 6)
    E = 0.0
    F = np.zeros((n, 3))
    W = np.zeros((3, 3))
    for i in range(n):
        d = pos[i][None, None, :] - (pos[None, :, :] + shifts[:, None, :])   # [img, j, 3]
        r2 = np.sum(d * d, axis=-1)
        mask = (r2 < rc * rc) & (r2 > 1e-12)
        r2m = np.where(mask, r2, 1.0)
        sr6 = (sig * sig / r2m) ** 3
        e = np.where(mask, 4 * eps * (sr6 * sr6 - sr6) - e_rc, 0.0)
        E += 0.5 * e.sum()
        dedr_over_r = np.where(mask, 4 * eps * (-12 * sr6 * sr6 + 6 * sr6) / r2m, 0.0)   # (1/r) dE/dr
        g = dedr_over_r[..., None] * d                                                   # dE/dd per pair
        F[i] -= g.sum(axis=(0, 1))
        W += 0.5 * np.einsum("ijk,ijl->kl", d, g)
    return E, F, W


def lj_dataset(n_struct: int, seed: int, n_lo: int = 8, n_hi: int = 16, Z: int = 18) -> Batch:
    """n_struct cubic argon-like cells, N ~ U{n_lo..n_hi}, 40-48 Å^3 per atom, RSA d_min 3.0 Å."""
    rng = np.random.default_rng(seed)
    cells, pos_l, e_l, f_l, s_l = [], [], [], [], []
    for _ in range(n_struct):
        n = int(rng.integers(n_lo, n_hi + 1))
        L, pos = _place(rng, n, 40.0, 48.0, 3.0, cubic=True)
        E, F, W = lj_labels(L, pos)
        cells.append(L); pos_l.append(pos)
        e_l.append(E / n); f_l.append(F)
        s_l.append(EV_A3_TO_GPA * W / abs(np.linalg.det(L)))
    n_per = [p.shape[0] for p in pos_l]
    atom_ptr = np.zeros(n_struct + 1, np.int64)
    atom_ptr[1:] = np.cumsum(n_per)
    N = int(atom_ptr[-1])
    return Batch(atom_ptr=atom_ptr, positions=np.concatenate(pos_l), lattice=np.stack(cells),
                 species=np.full(N, Z, np.int32), energy_per_atom=np.array(e_l), forces=np.concatenate(f_l),
                 stress=np.stack(s_l), magmom=np.zeros(N), magmom_mask=np.zeros(N, np.uint8))
