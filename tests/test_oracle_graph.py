"""Pins for oracle O1 (graph): closed-form counts, an independent k-d tree
enumeration (scipy), symmetry invariants, invariance of r/θ multisets, errors.
Cites: PAPER.md P:95 (graph extraction), SURVEY §8(c) O1 pins."""
import math

import numpy as np
import pytest
from scipy.spatial import cKDTree

from chg_inputs import (concat_batches, dimer, mptrj_like_batch, random_rotation, si_diamond,
                        simple_cubic)
from chg_inputs.structures import Batch
from oracle.graph import GeometryError, build_graph, build_graph_batch, perpendicular_widths


def test_simple_cubic_counts(golden):
    g = build_graph_batch(simple_cubic(3.0), 6.0, 3.0)
    assert g.n_edges == golden["simple_cubic_a3_r6_edges"]["value"]
    v = golden["simple_cubic_a3_r6_rb3"]["value"]
    assert g.n_bonds == v["bonds"] and g.n_angles == v["angles"]
    # θ = π appears (collinear opposite neighbours): clamp exercised
    assert np.isclose(g.cos_theta.min(), -1.0, atol=0) or g.cos_theta.min() == -1.0
    assert set(np.round(g.cos_theta, 12)) == {-1.0, 0.0}


def test_si_diamond_counts(golden):
    v = golden["si_diamond_5p431_r5_r3"]["value"]
    g = build_graph_batch(si_diamond(), 5.0, 3.0)
    assert (g.n_edges, g.n_bonds, g.n_angles) == (v["edges"], v["bonds"], v["angles"])
    np.testing.assert_allclose(g.cos_theta, v["cos_theta"], atol=1e-12)
    assert build_graph_batch(si_diamond(), 6.0, 3.0).n_edges == golden["si_diamond_5p431_r6_edges"]["value"]


def test_dimer_and_water(golden):
    g = build_graph_batch(dimer(2.0, 20.0), 6.0, 3.0)
    v = golden["dimer_counts"]["value"]
    assert g.n_edges == v["edges"] and g.n_angles == v["angles"]
    ang = math.radians(golden["water_angle_deg"]["value"])
    pos = np.array([[5.0, 5.0, 5.0], [6.0, 5.0, 5.0], [5.0 + math.cos(ang), 5.0 + math.sin(ang), 5.0]])
    b = Batch(atom_ptr=np.array([0, 3]), positions=pos, lattice=(np.eye(3) * 20)[None],
              species=np.array([8, 1, 1], np.int32), energy_per_atom=np.zeros(1), forces=np.zeros((3, 3)),
              stress=np.zeros((1, 3, 3)), magmom=np.zeros(3), magmom_mask=np.zeros(3, np.uint8))
    g = build_graph_batch(b, 1.2, 1.2)   # only the two O–H bonds
    assert g.n_angles == 2
    np.testing.assert_allclose(np.arccos(g.cos_theta), ang, atol=1e-9)


def _kdtree_edges(pos, L, rc):
    """Independent enumeration: replicate the cell over a generous image range
    and query a k-d tree (scipy) for all (i, j, n) within rc."""
    w = perpendicular_widths(L)
    f = pos @ np.linalg.inv(L)
    span = f.max(0) - f.min(0)
    lim = np.ceil(span + rc / w).astype(int) + 3
    imgs = np.array([[a, b, c] for a in range(-lim[0], lim[0] + 1) for b in range(-lim[1], lim[1] + 1)
                     for c in range(-lim[2], lim[2] + 1)])
    rep = (pos[None, :, :] + (imgs @ L)[:, None, :]).reshape(-1, 3)
    tree = cKDTree(rep)
    out = {}
    n = pos.shape[0]
    for i in range(n):
        for k in tree.query_ball_point(pos[i], rc + 1e-9):
            im, j = divmod(k, n)
            nvec = imgs[im]
            if i == j and not nvec.any():
                continue
            dvec = pos[i] - rep[k]
            dd = np.linalg.norm(dvec)
            if dd <= rc:
                # d = r_i − (r_j + nL) with the image on j
                out[(i, j, *map(int, nvec))] = dd
    return out


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_against_kdtree(seed):
    b = mptrj_like_batch(3, seed=seed)
    g = build_graph_batch(b, 5.0, 3.0)
    for s in range(b.n_struct):
        a0, a1 = b.atom_ptr[s], b.atom_ptr[s + 1]
        ref = _kdtree_edges(b.positions[a0:a1], b.lattice[s], 5.0)
        sel = (g.center >= a0) & (g.center < a1)
        got = {(int(c - a0), int(n - a0), *map(int, im)): r
               for c, n, im, r in zip(g.center[sel], g.nbr[sel], g.img[sel], g.r[sel])}
        assert set(got) == set(ref)
        for k in got:
            assert abs(got[k] - ref[k]) < 1e-12
    # bonds are exactly the edges within r_bond
    np.testing.assert_array_equal(g.bond_id >= 0, g.r <= 3.0)


def test_skewed_cell_margin_superset():
    """A flat, skewed cell (perpendicular width < cutoff): wider image ranges
    give bit-identical lists (any superset is valid)."""
    rng = np.random.default_rng(5)
    L = np.array([[6.0, 0.0, 0.0], [4.5, 2.2, 0.0], [1.0, 1.5, 2.5]])
    pos = rng.uniform(0, 1, size=(6, 3)) @ L
    b = Batch(atom_ptr=np.array([0, 6]), positions=pos, lattice=L[None],
              species=np.full(6, 14, np.int32), energy_per_atom=np.zeros(1), forces=np.zeros((6, 3)),
              stress=np.zeros((1, 3, 3)), magmom=np.zeros(6), magmom_mask=np.zeros(6, np.uint8))
    g1 = build_graph_batch(b, 5.0, 3.0, margin=1)
    g3 = build_graph_batch(b, 5.0, 3.0, margin=3)
    for k, v in g1.lists().items():
        np.testing.assert_array_equal(v, g3.lists()[k], err_msg=k)
    ref = _kdtree_edges(pos, L, 5.0)
    assert g1.n_edges == len(ref)


def test_directed_symmetry_and_maps():
    b = mptrj_like_batch(4, seed=21)
    g = build_graph_batch(b)
    e = np.arange(g.n_edges)
    np.testing.assert_array_equal(g.rev[g.rev], e)
    np.testing.assert_array_equal(g.center[g.rev], g.nbr)
    np.testing.assert_array_equal(g.img[g.rev], -g.img)
    np.testing.assert_array_equal(g.d[g.rev], -g.d)          # canonical: exact negation
    a = np.arange(g.n_angles)
    np.testing.assert_array_equal(g.swap[g.swap], a)
    np.testing.assert_array_equal(g.angle_b1[g.swap], g.angle_b2)
    # angles pair distinct bonds of the same centre
    c1 = g.center[g.bond_edge[g.angle_b1]]
    c2 = g.center[g.bond_edge[g.angle_b2]]
    np.testing.assert_array_equal(c1, c2)
    assert np.all(g.angle_b1 != g.angle_b2)
    # per-centre angle count m(m-1)
    m = np.bincount(g.center[g.bond_edge], minlength=g.n_atoms)
    assert g.n_angles == int(np.sum(m * (m - 1)))
    # edge order (i, j, n lexicographic)
    key = np.stack([g.center, g.nbr, g.img[:, 0], g.img[:, 1], g.img[:, 2]], 1).astype(np.int64)
    assert np.all(np.diff(np.lexsort(key.T[::-1])) == 1)


def _multisets(g):
    return np.sort(g.r), np.sort(g.cos_theta)


def test_translation_rotation_permutation_invariance():
    b = mptrj_like_batch(2, seed=31)
    g0 = build_graph_batch(b)
    r0, c0 = _multisets(g0)
    rng = np.random.default_rng(0)
    # translation (Cartesian, unwrapped)
    bt = Batch(**{**b.__dict__, "positions": b.positions + rng.normal(size=3) * 3.0})
    rt, ct = _multisets(build_graph_batch(bt))
    np.testing.assert_allclose(rt, r0, atol=1e-9); np.testing.assert_allclose(ct, c0, atol=1e-9)
    # rotation of lattice and positions (row vectors: x -> x R^T)
    R = random_rotation(rng)
    br = Batch(**{**b.__dict__, "positions": b.positions @ R.T, "lattice": b.lattice @ R.T})
    gr = build_graph_batch(br)
    rr, cr = _multisets(gr)
    np.testing.assert_allclose(rr, r0, atol=1e-9); np.testing.assert_allclose(cr, c0, atol=1e-9)
    assert gr.n_edges == g0.n_edges and gr.n_angles == g0.n_angles
    # permutation within each structure
    perm = np.concatenate([b.atom_ptr[s] + rng.permutation(b.atom_ptr[s + 1] - b.atom_ptr[s])
                           for s in range(b.n_struct)])
    bp = Batch(**{**b.__dict__, "positions": b.positions[perm], "species": b.species[perm]})
    rp, cp = _multisets(build_graph_batch(bp))
    np.testing.assert_allclose(rp, r0, atol=1e-12); np.testing.assert_allclose(cp, c0, atol=1e-12)


def test_batched_equals_individual():
    """Alg. 2 ≡ Alg. 1: a batch's per-structure subgraphs equal
    the individually built graphs (offsets applied)."""
    b1 = mptrj_like_batch(1, seed=41)
    b2 = mptrj_like_batch(1, seed=42)
    g = build_graph_batch(concat_batches([b1, b2]))
    g1, g2 = build_graph_batch(b1), build_graph_batch(b2)
    np.testing.assert_array_equal(g.nbr[:g1.n_edges], g1.nbr)
    np.testing.assert_array_equal(g.nbr[g1.n_edges:], g2.nbr + b1.n_atoms)
    np.testing.assert_array_equal(g.d, np.concatenate([g1.d, g2.d]))
    np.testing.assert_array_equal(g.angle_b2[g1.n_angles:], g2.angle_b2 + g1.n_bonds)


def test_errors():
    b = si_diamond()
    with pytest.raises(GeometryError):
        build_graph(b.atom_ptr, b.positions, np.zeros((1, 3, 3)), b.species)
    with pytest.raises(ValueError):
        build_graph(b.atom_ptr, b.positions, b.lattice, np.full(8, 95))
    with pytest.raises(ValueError):
        build_graph(b.atom_ptr, b.positions, b.lattice, b.species, 3.0, 5.0)
    pos = b.positions.copy(); pos[1] = pos[0]
    with pytest.raises(GeometryError):
        build_graph(b.atom_ptr, pos, b.lattice, b.species)
