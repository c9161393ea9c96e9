"""O1 — periodic atom graph, bond graph and angle list (oracle; test infrastructure).

Paper: PAPER.md P:95 (§II-B(1) "Molecular Graph Extraction"): atom graph G^a of
neighbours within the cutoff under periodic boundary conditions, edge attribute
r_ij; bond graph G^b whose nodes are G^a edges and whose edges are angle pairs
(e_ij, e_ik), θ_ijk = arccos(r_ij·r_ik / |r_ij||r_ik|).  Alg. 1 lines
P:253-256: r_j += I @ L; r_ij = r_i − r_j (image added to j).

Readings:
  Q8  directed edges (i→j, n) and (j→i, −n) are both present.
  Q9  angles = ordered pairs of DISTINCT bond edges sharing the centre i.
  Q10 closed cutoff; every unordered pair is evaluated ONCE, canonically:
      representative (a, b, m) with a < b, or a == b and m lexicographically
      positive; t = ((r_b + m1·a1) + m2·a2) + m3·a3; d = r_a − t;
      q = (dx² + dy²) + dz²; accept iff q <= rc·rc.  fp64, no fused multiply-add
      (numpy ufuncs round every product and sum separately).
  Q11 d_e = r_i − (r_j + n·L): centre i, x̂ points from j to i.
  Order: edges by (i, j, n1, n2, n3); bond edges keep edge order; angles of
  centre i with bonds b_1 < … < b_m are (b_p, b_q), q ≠ p, in (p, q) order.

Pure numpy; brute force over a per-structure image range that is a provable
superset (perpendicular widths) widened by `margin`.
"""
from __future__ import annotations

import dataclasses
from typing import Dict

import numpy as np


class GeometryError(ValueError):
    pass


@dataclasses.dataclass
class Graph:
    n_atoms: int
    row_ptr: np.ndarray     # int32 [N+1] edges CSR by centre atom
    center: np.ndarray      # int32 [E]
    nbr: np.ndarray         # int32 [E]
    img: np.ndarray         # int8  [E,3]
    d: np.ndarray           # float64 [E,3]  d_e = r_i - (r_j + n L)
    r: np.ndarray           # float64 [E]
    bond_id: np.ndarray     # int32 [E] bond index or -1
    bond_edge: np.ndarray   # int32 [B] edge index of each bond edge
    angle_ptr: np.ndarray   # int32 [B+1] angles CSR by first bond
    angle_b1: np.ndarray    # int32 [A]
    angle_b2: np.ndarray    # int32 [A]
    rev: np.ndarray         # int32 [E] index of (j, i, -n)
    swap: np.ndarray        # int32 [A] index of (b2, b1)
    cos_theta: np.ndarray   # float64 [A] clamp(d1·d2 / (r1 r2), -1, 1)
    struct_of_atom: np.ndarray  # int32 [N]
    counts: np.ndarray      # int64 [S,4] (N, E, B, A) per structure

    @property
    def n_edges(self) -> int:
        return int(self.nbr.shape[0])

    @property
    def n_bonds(self) -> int:
        return int(self.bond_edge.shape[0])

    @property
    def n_angles(self) -> int:
        return int(self.angle_b1.shape[0])

    def lists(self) -> Dict[str, np.ndarray]:
        """The integer lists compared bit-exactly against the CUDA path."""
        return dict(row_ptr=self.row_ptr, nbr=self.nbr, img=self.img, bond_id=self.bond_id,
                    bond_edge=self.bond_edge, angle_ptr=self.angle_ptr, angle_b1=self.angle_b1,
                    angle_b2=self.angle_b2, rev=self.rev, swap=self.swap)


def perpendicular_widths(L: np.ndarray) -> np.ndarray:
    """w_k = V / |a_{k+1} × a_{k+2}| (SPEC S:206 design decision)."""
    V = abs(np.linalg.det(L))
    return np.array([V / np.linalg.norm(np.cross(L[(k + 1) % 3], L[(k + 2) % 3])) for k in range(3)])


def _lexpos(n: np.ndarray) -> np.ndarray:
    """n lexicographically > 0 (first nonzero component positive)."""
    n1, n2, n3 = n[..., 0], n[..., 1], n[..., 2]
    return (n1 > 0) | ((n1 == 0) & (n2 > 0)) | ((n1 == 0) & (n2 == 0) & (n3 > 0))


def _structure_edges(pos: np.ndarray, L: np.ndarray, r_atom: float, r_bond: float,
                     margin: int, chunk: int = 64):
    """All directed edges of one structure in canonical order.
    Returns (ctr, nbr, img[int64], d, q, is_bond) with local atom indices."""
    n = pos.shape[0]
    V = abs(np.linalg.det(L))
    if not np.isfinite(V) or V <= 1e-6:
        raise GeometryError(f"|det L| = {V:g}")
    w = perpendicular_widths(L)
    f = pos @ np.linalg.inv(L)
    span = f.max(axis=0) - f.min(axis=0) if n > 0 else np.zeros(3)
    # |(Δf - n)_k| * w_k <= |d| <= r  =>  |n_k| <= span_k + r / w_k
    lim = np.ceil(span + r_atom / w).astype(np.int64) + margin
    rng_k = [np.arange(-lim[k], lim[k] + 1) for k in range(3)]
    imgs = np.stack(np.meshgrid(*rng_k, indexing="ij"), axis=-1).reshape(-1, 3)  # lex order
    K = imgs.shape[0]
    ra2 = r_atom * r_atom
    rb2 = r_bond * r_bond
    a1, a2, a3 = L[0], L[1], L[2]
    out = ([], [], [], [], [], [])
    jj = np.arange(n)
    chunk = max(1, min(chunk, 400_000 // max(1, n * K)))
    for i0 in range(0, n, chunk):
        ii = np.arange(i0, min(n, i0 + chunk))
        I = ii[:, None, None] * np.ones((1, n, K), np.int64)
        J = jj[None, :, None] * np.ones((len(ii), 1, K), np.int64)
        Nn = np.broadcast_to(imgs[None, None, :, :], (len(ii), n, K, 3))
        self_zero = (I == J) & np.all(Nn == 0, axis=-1)
        # canonical representative
        lt = I < J
        eq = I == J
        pos_lex = _lexpos(Nn)
        flip = (~lt & ~eq) | (eq & ~pos_lex)       # use (j, i, -n)
        A = np.where(flip, J, I)
        Bi = np.where(flip, I, J)
        M = np.where(flip[..., None], -Nn, Nn).astype(np.float64)
        pa = pos[A]
        pb = pos[Bi]
        t = pb + M[..., 0:1] * a1
        t = t + M[..., 1:2] * a2
        t = t + M[..., 2:3] * a3
        drep = pa - t
        q = (drep[..., 0] * drep[..., 0] + drep[..., 1] * drep[..., 1]) + drep[..., 2] * drep[..., 2]
        acc = (q <= ra2) & ~self_zero
        d = np.where(flip[..., None], -drep, drep)
        sel = np.nonzero(acc)          # C order = (i, j, n-lex) order
        out[0].append(I[sel]); out[1].append(J[sel]); out[2].append(Nn[sel])
        out[3].append(d[sel]); out[4].append(q[sel]); out[5].append(q[sel] <= rb2)
    cat = [np.concatenate(x) if x else np.zeros(0) for x in out]
    ctr, nbr, img, d, q, isb = cat
    if q.size and np.any(q < 1e-12):
        raise GeometryError("coincident atoms (accepted pair with d^2 < 1e-12)")
    return (ctr.astype(np.int64), nbr.astype(np.int64), img.reshape(-1, 3).astype(np.int64),
            d.reshape(-1, 3), q, isb.astype(bool))


def build_graph(atom_ptr, positions, lattice, species, r_atom: float = 5.0, r_bond: float = 3.0,
                n_species: int = 94, margin: int = 1) -> Graph:
    """O1.  See module docstring.  Raises GeometryError / ValueError on bad input
    (|det L| <= 1e-6 Å³, Z outside 1..n_species, non-finite input,
    r_bond > r_atom, coincident atoms)."""
    atom_ptr = np.asarray(atom_ptr, np.int64)
    positions = np.asarray(positions, np.float64)
    lattice = np.asarray(lattice, np.float64).reshape(-1, 3, 3)
    species = np.asarray(species)
    if not (0 < r_bond <= r_atom):
        raise ValueError("need 0 < r_bond <= r_atom")
    if not (np.all(np.isfinite(positions)) and np.all(np.isfinite(lattice))):
        raise ValueError("non-finite input")
    if species.size and (species.min() < 1 or species.max() > n_species):
        raise ValueError("species out of range")
    S = atom_ptr.shape[0] - 1
    ctr_l, nbr_l, img_l, d_l, q_l, b_l = [], [], [], [], [], []
    counts = np.zeros((S, 4), np.int64)
    for s in range(S):
        a0, a1 = int(atom_ptr[s]), int(atom_ptr[s + 1])
        try:
            c, nb, im, d, q, isb = _structure_edges(positions[a0:a1], lattice[s], r_atom, r_bond, margin)
        except GeometryError as ex:
            raise GeometryError(f"structure {s}: {ex}") from None
        ctr_l.append(c + a0); nbr_l.append(nb + a0); img_l.append(im); d_l.append(d)
        q_l.append(q); b_l.append(isb)
        counts[s, 0] = a1 - a0
        counts[s, 1] = c.shape[0]
        counts[s, 2] = int(isb.sum())
    ctr = np.concatenate(ctr_l) if S else np.zeros(0, np.int64)
    nbr = np.concatenate(nbr_l) if S else np.zeros(0, np.int64)
    img = np.concatenate(img_l) if S else np.zeros((0, 3), np.int64)
    d = np.concatenate(d_l) if S else np.zeros((0, 3))
    q = np.concatenate(q_l) if S else np.zeros(0)
    isb = np.concatenate(b_l) if S else np.zeros(0, bool)
    N = int(atom_ptr[-1])
    E = ctr.shape[0]
    row_ptr = np.zeros(N + 1, np.int64)
    np.add.at(row_ptr, ctr + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    r = np.sqrt(q)
    bond_edge = np.nonzero(isb)[0]
    bond_id = np.full(E, -1, np.int64)
    bond_id[bond_edge] = np.arange(bond_edge.shape[0])
    # angles: centre i with bonds b_1..b_m -> (b_p, b_q), q != p
    b_ctr = ctr[bond_edge]
    B = bond_edge.shape[0]
    angle_ptr = np.zeros(B + 1, np.int64)
    a1_l, a2_l = [], []
    bstart = np.searchsorted(b_ctr, np.arange(N), side="left")
    bend = np.searchsorted(b_ctr, np.arange(N), side="right")
    for b in range(B):
        i = b_ctr[b]
        others = [c for c in range(bstart[i], bend[i]) if c != b]
        angle_ptr[b + 1] = angle_ptr[b] + len(others)
        a1_l.extend([b] * len(others)); a2_l.extend(others)
    angle_b1 = np.array(a1_l, np.int64)
    angle_b2 = np.array(a2_l, np.int64)
    A = angle_b1.shape[0]
    # rev: (i, j, n) -> (j, i, -n)
    key = {(int(ctr[e]), int(nbr[e]), *map(int, img[e])): e for e in range(E)}
    rev = np.array([key[(int(nbr[e]), int(ctr[e]), *map(int, -img[e]))] for e in range(E)], np.int64)
    akey = {(int(angle_b1[a]), int(angle_b2[a])): a for a in range(A)}
    swap = np.array([akey[(int(angle_b2[a]), int(angle_b1[a]))] for a in range(A)], np.int64)
    if A:
        e1, e2 = bond_edge[angle_b1], bond_edge[angle_b2]
        c = np.sum(d[e1] * d[e2], axis=1) / (r[e1] * r[e2])
        cos_theta = np.clip(c, -1.0, 1.0)
    else:
        cos_theta = np.zeros(0)
    for s in range(S):
        a0, a1 = int(atom_ptr[s]), int(atom_ptr[s + 1])
        bs = np.searchsorted(b_ctr, a0, "left"); be = np.searchsorted(b_ctr, a1, "left")
        counts[s, 3] = angle_ptr[be] - angle_ptr[bs]
    struct_of_atom = np.repeat(np.arange(S), np.diff(atom_ptr))
    i32 = lambda x: np.ascontiguousarray(x, np.int32)  # noqa: E731
    return Graph(n_atoms=N, row_ptr=i32(row_ptr), center=i32(ctr), nbr=i32(nbr),
                 img=np.ascontiguousarray(img, np.int8), d=d, r=r, bond_id=i32(bond_id),
                 bond_edge=i32(bond_edge), angle_ptr=i32(angle_ptr), angle_b1=i32(angle_b1),
                 angle_b2=i32(angle_b2), rev=i32(rev), swap=i32(swap), cos_theta=cos_theta,
                 struct_of_atom=i32(struct_of_atom), counts=counts)


def build_graph_batch(batch, r_atom=5.0, r_bond=3.0, margin=1) -> Graph:
    return build_graph(batch.atom_ptr, batch.positions, batch.lattice, batch.species,
                       r_atom, r_bond, margin=margin)
