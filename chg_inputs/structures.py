"""Seeded synthetic crystal batches (recipes: SURVEY.md §8(d) "Synthetic inputs").

Everything here is input generation only: random cells, random sequential
addition (RSA) of atoms, random species and random labels.  No graph, basis or
model arithmetic lives here (see chg_inputs/__init__.py).

Conventions (shared by both sides, stated in include/chg.h as well):
  * lattice rows are the lattice vectors a1, a2, a3 in Å (row-vector convention)
  * positions are Cartesian Å, fp64, NOT wrapped into the cell
  * species are atomic numbers Z in 1..94 (int32)
  * atom_ptr[s]..atom_ptr[s+1] are the atoms of structure s (int64)
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Sequence

import numpy as np

__all__ = [
    "Batch", "si_diamond", "simple_cubic", "dimer", "mptrj_like_batch",
    "skewed_oxide_batch", "lifepo4_like_cell", "concat_batches", "split_batch",
    "make_config_batch",
]


@dataclasses.dataclass
class Batch:
    atom_ptr: np.ndarray          # int64 [S+1]
    positions: np.ndarray         # float64 [N,3] Cartesian Å
    lattice: np.ndarray           # float64 [S,3,3] rows = lattice vectors
    species: np.ndarray           # int32 [N] Z in 1..94
    energy_per_atom: np.ndarray   # float64 [S] eV/atom (label)
    forces: np.ndarray            # float64 [N,3] eV/Å (label)
    stress: np.ndarray            # float64 [S,3,3] GPa (label)
    magmom: np.ndarray            # float64 [N] μB (label)
    magmom_mask: np.ndarray       # uint8 [N] 1 = labelled

    @property
    def n_struct(self) -> int:
        return int(self.atom_ptr.shape[0] - 1)

    @property
    def n_atoms(self) -> int:
        return int(self.atom_ptr[-1])

    def atoms_per_struct(self) -> np.ndarray:
        return np.diff(self.atom_ptr)


# ----------------------------------------------------------------------------
# cells and positions
# ----------------------------------------------------------------------------

def _lattice_from_params(a, b, c, alpha, beta, gamma) -> np.ndarray:
    """Cell matrix (rows = vectors) from lengths and angles (degrees)."""
    al, be, ga = (math.radians(x) for x in (alpha, beta, gamma))
    ca, cb, cg, sg = math.cos(al), math.cos(be), math.cos(ga), math.sin(ga)
    a1 = np.array([a, 0.0, 0.0])
    a2 = np.array([b * cg, b * sg, 0.0])
    cy = (ca - cb * cg) / sg
    cz = math.sqrt(max(1.0 - cb * cb - cy * cy, 1e-12))
    a3 = np.array([c * cb, c * cy, c * cz])
    return np.stack([a1, a2, a3])


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform proper rotation (det +1) from a random unit quaternion."""
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def _triclinic_cell(rng: np.random.Generator, volume: float, rotate: bool = True) -> np.ndarray:
    """Axis ratios U(0.7, 1.4), angles U(75°, 105°), scaled to `volume` Å³."""
    ratios = rng.uniform(0.7, 1.4, size=3)
    angles = rng.uniform(75.0, 105.0, size=3)
    L = _lattice_from_params(ratios[0], ratios[1], ratios[2], *angles)
    L *= (volume / abs(np.linalg.det(L))) ** (1.0 / 3.0)
    if rotate:
        L = L @ random_rotation(rng).T
    return L


_SHIFTS = np.array([[i, j, k] for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1)],
                   dtype=np.float64)


def _min_image_d2(cand_f: np.ndarray, placed_f: np.ndarray, L: np.ndarray) -> np.ndarray:
    """Squared minimum-image distances [b,p] between fractional sets."""
    df = cand_f[:, None, :] - placed_f[None, :, :]
    df -= np.round(df)
    dc = df @ L                                           # [b,p,3]
    if np.allclose(L, np.diag(np.diag(L))) and np.allclose(np.diag(L), L[0, 0]):
        # cubic cell: the wrapped vector is the minimum image (dmin < edge/2)
        return np.einsum("bpk,bpk->bp", dc, dc)
    sc = _SHIFTS @ L                                      # [27,3]
    dd = dc[:, :, None, :] + sc[None, None, :, :]         # [b,p,27,3]
    return np.min(np.einsum("bpsk,bpsk->bps", dd, dd), axis=2)


def _rsa_fractional(rng: np.random.Generator, L: np.ndarray, n: int, dmin: float,
                    max_rounds: int = 4000, batch: int = 64):
    """Random sequential addition in the periodic cell L with minimum image
    distance >= dmin.  Candidates are proposed `batch` at a time and accepted
    greedily in proposal order.  Returns fractional coords [n,3] or None."""
    d2min = dmin * dmin
    placed = np.zeros((0, 3))
    rounds = 0
    while placed.shape[0] < n:
        rounds += 1
        if rounds > max_rounds:
            return None
        cand = rng.uniform(0.0, 1.0, size=(batch, 3))
        if placed.shape[0] > 0:
            ok = np.all(_min_image_d2(cand, placed, L) >= d2min, axis=1)
        else:
            ok = np.ones(batch, dtype=bool)
        acc: List[np.ndarray] = []
        for ci in np.nonzero(ok)[0]:
            c = cand[ci:ci + 1]
            if acc and not np.all(_min_image_d2(c, np.concatenate(acc), L) >= d2min):
                continue
            acc.append(c)
            if placed.shape[0] + len(acc) >= n:
                break
        if acc:
            placed = np.concatenate([placed] + acc)
    return placed[:n]


def _place(rng, n, vol_per_atom_lo, vol_per_atom_hi, dmin, cubic=False):
    """Cell + RSA positions; grows the volume by 3 % on RSA failure."""
    vol = n * rng.uniform(vol_per_atom_lo, vol_per_atom_hi)
    for _ in range(50):
        if cubic:
            L = np.eye(3) * vol ** (1.0 / 3.0)
        else:
            L = _triclinic_cell(rng, vol)
        f = _rsa_fractional(rng, L, n, dmin)
        if f is not None:
            return L, f @ L
        vol *= 1.03
    raise RuntimeError("RSA failed to place atoms")


# ----------------------------------------------------------------------------
# labels
# ----------------------------------------------------------------------------

def _labels(rng, n_atoms_per: Sequence[int]):
    S = len(n_atoms_per)
    N = int(sum(n_atoms_per))
    e = rng.normal(-5.0, 1.0, size=S)
    f = rng.normal(0.0, 0.3, size=(N, 3))
    st = np.zeros((S, 3, 3))
    for s in range(S):
        u = rng.normal(0.0, 1.0, size=(3, 3))
        st[s] = np.triu(u) + np.triu(u, 1).T
    m = np.abs(rng.normal(0.0, 1.0, size=N))
    mask = (rng.uniform(size=N) < 0.16).astype(np.uint8)   # 16 % labelled
    return e, f, st, m, mask


def _assemble(cells, pos_list, spec_list, rng) -> Batch:
    n_per = [p.shape[0] for p in pos_list]
    e, f, st, m, mask = _labels(rng, n_per)
    atom_ptr = np.zeros(len(n_per) + 1, dtype=np.int64)
    atom_ptr[1:] = np.cumsum(n_per)
    return Batch(
        atom_ptr=atom_ptr,
        positions=np.concatenate(pos_list).astype(np.float64),
        lattice=np.stack(cells).astype(np.float64),
        species=np.concatenate(spec_list).astype(np.int32),
        energy_per_atom=e, forces=f, stress=st, magmom=m, magmom_mask=mask,
    )


# ----------------------------------------------------------------------------
# named structures
# ----------------------------------------------------------------------------

SI_DIAMOND_FRAC = np.array([
    [0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0],
    [.25, .25, .25], [.25, .75, .75], [.75, .25, .75], [.75, .75, .25]])


def si_diamond(a: float = 5.431, jitter: float = 0.0, seed: int = 7,
               reps=(1, 1, 1)) -> Batch:
    """C1: Si diamond conventional cell (8 atoms, Z=14); optional U(±jitter Å)
    displacement; optional supercell reps.  Labels per SURVEY §8(d) C1."""
    L = np.eye(3) * a
    frac = []
    for i in range(reps[0]):
        for j in range(reps[1]):
            for k in range(reps[2]):
                frac.append(SI_DIAMOND_FRAC + np.array([i, j, k]))
    frac = np.concatenate(frac)
    Ls = L * np.array(reps, dtype=np.float64)[:, None]
    pos = frac @ L
    if jitter > 0:
        rng = np.random.default_rng(seed)
        pos = pos + rng.uniform(-jitter, jitter, size=pos.shape)
    n = pos.shape[0]
    return Batch(
        atom_ptr=np.array([0, n], dtype=np.int64), positions=pos, lattice=Ls[None],
        species=np.full(n, 14, dtype=np.int32),
        energy_per_atom=np.array([-5.42]), forces=np.zeros((n, 3)),
        stress=np.zeros((1, 3, 3)), magmom=np.zeros(n), magmom_mask=np.ones(n, np.uint8))


def simple_cubic(a: float = 3.0, Z: int = 3) -> Batch:
    """One atom in a cubic cell of edge a."""
    return Batch(
        atom_ptr=np.array([0, 1], dtype=np.int64), positions=np.zeros((1, 3)),
        lattice=(np.eye(3) * a)[None], species=np.array([Z], np.int32),
        energy_per_atom=np.array([-1.0]), forces=np.zeros((1, 3)), stress=np.zeros((1, 3, 3)),
        magmom=np.zeros(1), magmom_mask=np.zeros(1, np.uint8))


def dimer(sep: float = 2.0, box: float = 20.0, Z=(8, 8)) -> Batch:
    """Isolated dimer in a large cubic box."""
    pos = np.array([[5.0, 5.0, 5.0], [5.0 + sep, 5.0, 5.0]])
    return Batch(
        atom_ptr=np.array([0, 2], dtype=np.int64), positions=pos,
        lattice=(np.eye(3) * box)[None], species=np.array(Z, np.int32),
        energy_per_atom=np.array([-2.0]), forces=np.zeros((2, 3)), stress=np.zeros((1, 3, 3)),
        magmom=np.zeros(2), magmom_mask=np.ones(2, np.uint8))


def mptrj_like_batch(n_struct: int, seed: int) -> Batch:
    """C2/C3 "MPtrj-shaped": N = clip(round(LogNormal(ln 24, 0.7)), 2, 200)
    (mean ≈ 31 atoms), triclinic cell with V = N·U(10,16) Å³, RSA with
    minimum image distance 1.6 Å; species O w.p. 0.45, else uniform 1..94."""
    rng = np.random.default_rng(seed)
    cells, pos, spec = [], [], []
    for _ in range(n_struct):
        n = int(np.clip(round(rng.lognormal(math.log(24.0), 0.7)), 2, 200))
        L, p = _place(rng, n, 10.0, 16.0, 1.6)
        z = np.where(rng.uniform(size=n) < 0.45, 8, rng.integers(1, 95, size=n))
        cells.append(L); pos.append(p); spec.append(z)
    return _assemble(cells, pos, spec, rng)


def skewed_oxide_batch(n_struct: int, seed: int) -> Batch:
    """C4: N = round(exp(U(ln 4, ln 400))), V = N·U(8.5,10.5) Å³, RSA with
    minimum distance 1.7 Å; species O 0.55, Li 0.20, Mn/Fe/Co/Ni 0.25."""
    rng = np.random.default_rng(seed)
    cells, pos, spec = [], [], []
    for _ in range(n_struct):
        n = int(round(math.exp(rng.uniform(math.log(4.0), math.log(400.0)))))
        L, p = _place(rng, n, 8.5, 10.5, 1.7)
        u = rng.uniform(size=n)
        tm = rng.choice(np.array([25, 26, 27, 28]), size=n)
        z = np.where(u < 0.55, 8, np.where(u < 0.75, 3, tm))
        cells.append(L); pos.append(p); spec.append(z)
    return _assemble(cells, pos, spec, rng)


def lifepo4_like_cell(n_atoms: int = 4096, edge: float = 34.92, seed: int = 3000) -> Batch:
    """C5: LiFePO4-like supercell: cubic box, RSA min distance 1.5 Å,
    composition Li:Fe:P:O = 1:1:1:4 (585/585/585/2341 at 4096 atoms)."""
    rng = np.random.default_rng(seed)
    L = np.eye(3) * edge
    f = _rsa_fractional(rng, L, n_atoms, 1.5, max_rounds=200000)
    if f is None:
        raise RuntimeError("RSA failed for C5")
    n_li = n_atoms // 7
    z = np.array([3] * n_li + [26] * n_li + [15] * n_li + [8] * (n_atoms - 3 * n_li), np.int32)
    z = rng.permutation(z)
    return _assemble([L], [f @ L], [z], rng)


# ----------------------------------------------------------------------------
# batch plumbing
# ----------------------------------------------------------------------------

def concat_batches(batches: Sequence[Batch]) -> Batch:
    n_per = np.concatenate([b.atoms_per_struct() for b in batches])
    atom_ptr = np.zeros(len(n_per) + 1, dtype=np.int64)
    atom_ptr[1:] = np.cumsum(n_per)
    cat = lambda name: np.concatenate([getattr(b, name) for b in batches])  # noqa: E731
    return Batch(atom_ptr=atom_ptr, positions=cat("positions"), lattice=cat("lattice"),
                 species=cat("species"), energy_per_atom=cat("energy_per_atom"),
                 forces=cat("forces"), stress=cat("stress"), magmom=cat("magmom"),
                 magmom_mask=cat("magmom_mask"))


def split_batch(b: Batch, struct_ids: Sequence[int]) -> Batch:
    """Sub-batch of the given structures, in the given order."""
    parts = []
    for s in struct_ids:
        a0, a1 = int(b.atom_ptr[s]), int(b.atom_ptr[s + 1])
        parts.append(Batch(
            atom_ptr=np.array([0, a1 - a0], np.int64), positions=b.positions[a0:a1],
            lattice=b.lattice[s:s + 1], species=b.species[a0:a1],
            energy_per_atom=b.energy_per_atom[s:s + 1], forces=b.forces[a0:a1],
            stress=b.stress[s:s + 1], magmom=b.magmom[a0:a1], magmom_mask=b.magmom_mask[a0:a1]))
    return concat_batches(parts)


def make_config_batch(name: str, index: int = 0, n_struct=None) -> Batch:
    """Named BASELINE configs (SURVEY §8(d) seeds): C1..C5."""
    name = name.upper()
    if name == "C1":
        return si_diamond()
    if name == "C2":
        return mptrj_like_batch(n_struct or 40, seed=1000 + index)
    if name == "C3":
        return mptrj_like_batch(n_struct or 128, seed=1000 + index)
    if name == "C4":
        return skewed_oxide_batch(n_struct or 128, seed=2000 + index)
    if name == "C5":
        return lifepo4_like_cell(seed=3000 + index)
    raise ValueError(name)
