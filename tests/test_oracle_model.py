"""Pins for oracle O3–O6, O8, O10 (model): census, invariances, extensivity,
site symmetry, closed-form head cases, Jacobian dependency structure of Eq. 4–6
under Eq. 11, energy-derived F/σ against finite differences, parameter
gradients against finite differences.  Cites PAPER.md and SURVEY §8(c)."""
import math

import numpy as np
import pytest
import torch

from chg_inputs import (Batch, concat_batches, dimer, init_flat_params, mptrj_like_batch,
                        random_rotation, si_diamond)
from oracle.graph import build_graph_batch
from oracle.model import (DT, ModelConfig, TGraph, atom_conv, angle_update, bond_conv,
                          derived_force_stress, edge_vectors, forward, param_count, param_layout,
                          run_forward, srbf, unflatten)
from oracle.train import LossConfig, loss_and_grad, loss_terms

CFG = ModelConfig()


def _params(cfg=CFG, seed=0, bias_scale=0.1):
    return init_flat_params(param_layout(cfg), seed=seed, bias_scale=bias_scale)


def _fwd(b, p=None, cfg=CFG, keep=False):
    g = build_graph_batch(b, cfg.r_atom, cfg.r_bond)
    return g, run_forward(g, b.species, b.lattice, _params(cfg) if p is None else p, cfg, keep)


def test_census(golden):
    n = param_count(CFG)
    assert n == golden["census_build"]["value"]
    assert len(param_layout(CFG)) == 151
    paper = golden["census_paper"]["value"]
    assert abs(n - paper) / paper <= golden["census_tolerance_rel"]["value"]


def test_translation_rotation_permutation():
    b = mptrj_like_batch(2, seed=101)
    p = _params()
    _, o = _fwd(b, p)
    rng = np.random.default_rng(3)
    bt = Batch(**{**b.__dict__, "positions": b.positions + rng.normal(size=3) * 2.0})
    _, ot = _fwd(bt, p)
    for k in ("energy", "magmom", "forces", "stress"):
        np.testing.assert_allclose(ot[k].detach().numpy(), o[k].detach().numpy(), atol=1e-9, err_msg=k)
    R = random_rotation(rng)
    br = Batch(**{**b.__dict__, "positions": b.positions @ R.T, "lattice": b.lattice @ R.T})
    _, orr = _fwd(br, p)
    np.testing.assert_allclose(orr["energy"].numpy(), o["energy"].numpy(), atol=1e-9)
    np.testing.assert_allclose(orr["magmom"].numpy(), o["magmom"].numpy(), atol=1e-9)
    # Eq. 8: F(Rx) = R F(x)
    np.testing.assert_allclose(orr["forces"].numpy(), o["forces"].numpy() @ R.T, atol=1e-9)
    perm = np.concatenate([b.atom_ptr[s] + rng.permutation(b.atom_ptr[s + 1] - b.atom_ptr[s])
                           for s in range(b.n_struct)])
    bp = Batch(**{**b.__dict__, "positions": b.positions[perm], "species": b.species[perm]})
    _, op = _fwd(bp, p)
    np.testing.assert_allclose(op["energy"].numpy(), o["energy"].numpy(), atol=1e-9)
    np.testing.assert_allclose(op["magmom"].numpy(), o["magmom"].numpy()[perm], atol=1e-9)
    np.testing.assert_allclose(op["forces"].numpy(), o["forces"].numpy()[perm], atol=1e-9)
    np.testing.assert_allclose(op["stress"].numpy(), o["stress"].numpy(), atol=1e-9)


def test_supercell_extensivity():
    """2×1×1 supercell of a jittered Si cell: E doubles, per-atom outputs equal."""
    b1 = si_diamond(jitter=0.05, seed=7)
    L = b1.lattice[0]
    pos2 = np.concatenate([b1.positions, b1.positions + L[0]])
    b2 = Batch(atom_ptr=np.array([0, 16]), positions=pos2, lattice=(L * np.array([[2.0], [1.0], [1.0]]))[None],
               species=np.full(16, 14, np.int32), energy_per_atom=np.zeros(1), forces=np.zeros((16, 3)),
               stress=np.zeros((1, 3, 3)), magmom=np.zeros(16), magmom_mask=np.zeros(16, np.uint8))
    p = _params()
    _, o1 = _fwd(b1, p)
    _, o2 = _fwd(b2, p)
    assert float(o2["energy"][0]) == pytest.approx(2 * float(o1["energy"][0]), rel=1e-12)
    np.testing.assert_allclose(o2["magmom"].numpy()[:8], o1["magmom"].numpy(), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(o2["magmom"].numpy()[8:], o1["magmom"].numpy(), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(o2["forces"].numpy()[8:], o1["forces"].numpy(), atol=1e-12)


def test_si_ideal_site_symmetry():
    """Ideal diamond: all sites equivalent -> equal magmoms; every neighbour
    shell sums to zero -> F^head = 0 and F^E = 0; σ^E isotropic."""
    b = si_diamond()
    p = _params()
    g, o = _fwd(b, p)
    m = o["magmom"].numpy()
    np.testing.assert_allclose(m, m[0], atol=1e-12)
    assert np.max(np.abs(o["forces"].numpy())) < 1e-12
    d = derived_force_stress(g, b.positions, b.lattice, b.species, p, CFG)
    assert np.max(np.abs(d["forces"].numpy())) < 1e-10
    s = d["stress"].numpy()[0]
    assert np.max(np.abs(s - np.diag(np.diag(s)))) < 1e-9
    np.testing.assert_allclose(np.diag(s), s[0, 0], atol=1e-9)


def test_head_closed_forms():
    b = mptrj_like_batch(2, seed=111)
    p = _params()
    P = unflatten(torch.as_tensor(p.copy()), CFG)
    # energy head: zero last layer, bias c -> E_s = N_s c
    P["head_E.W3"].zero_(); P["head_E.b3"].fill_(0.25)
    P["head_M.W"].zero_(); P["head_M.b"].fill_(-0.5)              # magmom = bias
    P["head_S.W2"].zero_()
    Bm = torch.tensor([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0], [7.0, 8.0, 9.0]], dtype=DT)
    P["head_S.b2"].copy_(Bm.reshape(-1))
    P["head_F.W2"].zero_(); P["head_F.b2"].fill_(0.3)
    flat = torch.cat([P[n].reshape(-1) for n, _ in param_layout(CFG)]).numpy()
    g, o = _fwd(b, flat)
    np.testing.assert_allclose(o["energy"].numpy(), 0.25 * np.diff(b.atom_ptr), rtol=1e-13)
    np.testing.assert_allclose(o["magmom"].numpy(), -0.5, rtol=0, atol=1e-15)
    # Eq. 9 with constant MLP output B: σ = sym(B) ⊙ (Σ_p L̂_p)(Σ_q L̂_q)^T
    for s in range(b.n_struct):
        Lh = b.lattice[s] / np.linalg.norm(b.lattice[s], axis=1, keepdims=True)
        sh = Lh.sum(0)
        exp = 0.5 * (Bm.numpy() + Bm.numpy().T) * np.outer(sh, sh)
        np.testing.assert_allclose(o["stress"].numpy()[s], exp, rtol=1e-12, atol=1e-12)
    # Eq. 7 with constant n: F_i = n Σ_j x̂_ij
    xh = g.d / g.r[:, None]
    F = np.zeros((b.n_atoms, 3)); np.add.at(F, g.center, 0.3 * xh)
    np.testing.assert_allclose(o["forces"].numpy(), F, atol=1e-13)
    # cubic lattice: G = all-ones
    bc = si_diamond()
    _, oc = _fwd(bc, flat)
    np.testing.assert_allclose(oc["stress"].numpy()[0], 0.5 * (Bm.numpy() + Bm.numpy().T), rtol=1e-12)
    # dimer: F_1 = -F_2 exactly (directed-edge antisymmetry)
    _, od = _fwd(dimer(2.0), flat)
    np.testing.assert_array_equal(od["forces"].numpy()[0], -od["forces"].numpy()[1])


def test_empty_graph_and_zero_angles():
    p = _params()
    # no edges at all: the message sum is empty, so each atom conv adds only the
    # bias of 𝓛_v (Eq. 4; = identity at the default zero-bias init)
    _, o = _fwd(dimer(7.0, 30.0), p, keep=True)
    P = unflatten(torch.as_tensor(p), CFG)
    bsum = sum(P[f"atom{t}.out.b"] for t in range(CFG.n_atom_conv)).numpy()
    np.testing.assert_allclose(o["v_final"].numpy(), o["v0"].numpy() + bsum, atol=1e-15)
    assert np.all(o["forces"].numpy() == 0)
    p0 = _params(bias_scale=0.0)
    _, o0 = _fwd(dimer(7.0, 30.0), p0, keep=True)
    np.testing.assert_array_equal(o0["v_final"].numpy(), o0["v0"].numpy())
    # dimer at 2 Å: 2 bond edges, no angles -> e^{t+1} = e^t + b_e (Q16)
    _, o = _fwd(dimer(2.0, 30.0), p, keep=True)
    np.testing.assert_allclose(o["e1"].numpy(), o["e0"].numpy() + P["bond0.out.b"].numpy(), atol=1e-15)


def _block_inputs(b, seed=5):
    g = build_graph_batch(b)
    G = TGraph.from_graph(g)
    P = unflatten(torch.as_tensor(_params()), CFG)
    rng = np.random.default_rng(seed)
    mk = lambda n: torch.as_tensor(rng.normal(size=(n, CFG.d))).requires_grad_(True)  # noqa: E731
    return g, G, P, mk(G.N), mk(G.E), mk(G.A), mk(G.E), mk(G.B)


def _rows(grad):
    return set(np.nonzero(np.abs(grad.numpy()).sum(1) > 0)[0].tolist())


def test_dependency_structure():
    """Jacobian sparsity fixed by Eq. 4, Eq. 5/6 and Eq. 11:
    v'_i depends on v_i, v_j (j ∈ N(i)), e_e and eᵃ_e (e at centre i);
    e'_e depends on v_{i(e)} only, e_e, e_{e2} of angles (e, e2), a of those
    angles, eᵇ of e and the e2's; a'_α on v_i, e_{e1}, e_{e2}, a_α only."""
    b = mptrj_like_batch(1, seed=131)
    g, G, P, v, e, a, ea, eb = _block_inputs(b)
    rng = np.random.default_rng(0)
    i = int(g.center[g.bond_edge[g.angle_b1[0]]])
    vn = atom_conv(0, v, e, ea, G, P, CFG)
    gv, ge, gea = torch.autograd.grad(vn[i].sum(), (v, e, ea))
    row = set(range(g.row_ptr[i], g.row_ptr[i + 1]))
    assert _rows(gv) == {i} | {int(g.nbr[x]) for x in row}
    assert _rows(ge) == row and _rows(gea) == row
    # bond conv on an edge with angles
    b1 = int(g.angle_b1[0]); eid = int(g.bond_edge[b1])
    ang = list(range(g.angle_ptr[b1], g.angle_ptr[b1 + 1]))
    en = bond_conv(0, v, e, a, eb, G, P, CFG)
    gv, ge, ga, geb = torch.autograd.grad(en[eid].sum(), (v, e, a, eb), retain_graph=True)
    assert _rows(gv) == {i}
    assert _rows(ge) == {eid} | {int(g.bond_edge[g.angle_b2[x]]) for x in ang}
    assert _rows(ga) == set(ang)
    assert _rows(geb) == {b1} | {int(g.angle_b2[x]) for x in ang}
    # a non-bond edge only gets the bias path: depends on itself alone
    nb = int(np.nonzero(g.bond_id < 0)[0][0])
    gv, ge, ga = torch.autograd.grad(en[nb].sum(), (v, e, a), allow_unused=True)
    assert _rows(ge) == {nb} and _rows(gv) == set() and _rows(ga) == set()
    # angle update
    al = int(rng.integers(g.n_angles))
    an = angle_update(0, v, e, a, G, P, CFG)
    gv, ge, ga = torch.autograd.grad(an[al].sum(), (v, e, a))
    i_al = int(g.center[g.bond_edge[g.angle_b1[al]]])
    assert _rows(gv) == {i_al}
    assert _rows(ge) == {int(g.bond_edge[g.angle_b1[al]]), int(g.bond_edge[g.angle_b2[al]])}
    assert _rows(ga) == {al}


def test_eq11_order_independence():
    """Eq. 11: bond conv and angle update read only layer-t features, so their
    results do not depend on evaluation order."""
    b = mptrj_like_batch(1, seed=141)
    g, G, P, v, e, a, ea, eb = _block_inputs(b)
    e1 = bond_conv(0, v, e, a, eb, G, P, CFG); a1 = angle_update(0, v, e, a, G, P, CFG)
    a2 = angle_update(0, v, e, a, G, P, CFG); e2 = bond_conv(0, v, e, a, eb, G, P, CFG)
    assert torch.equal(e1, e2) and torch.equal(a1, a2)


def _energy_fixed_graph(G, species, pos, lat, P, cfg, strain=None):
    if strain is not None:
        D = torch.eye(3, dtype=DT) + strain
        pos = pos @ D
        lat = lat @ D
    d = edge_vectors(G, pos, lat)
    return forward(G, species, d, lat, P, cfg)["energy"]


@pytest.mark.parametrize("which", ["si", "c2"])
def test_derived_force_stress_fd(which):
    """O10 against central finite differences (h = 1e-5 Å, strain 1e-6);
    NS bar: ≤ 1e-4 eV/Å and ≤ 1e-4 GPa.  Also σ^E symmetric to 1e-10."""
    b = si_diamond(jitter=0.05, seed=7) if which == "si" else mptrj_like_batch(1, seed=151)
    p = _params()
    g = build_graph_batch(b)
    res = derived_force_stress(g, b.positions, b.lattice, b.species, p, CFG)
    G = TGraph.from_graph(g)
    P = unflatten(torch.as_tensor(p), CFG)
    sp = torch.as_tensor(b.species)
    pos0 = torch.as_tensor(b.positions.copy())
    lat = torch.as_tensor(b.lattice)
    h = 1e-5
    Ffd = np.zeros_like(b.positions)
    for i in range(b.n_atoms):
        for c in range(3):
            pp = pos0.clone(); pp[i, c] += h
            pm = pos0.clone(); pm[i, c] -= h
            Ffd[i, c] = -(float(_energy_fixed_graph(G, sp, pp, lat, P, CFG).sum())
                          - float(_energy_fixed_graph(G, sp, pm, lat, P, CFG).sum())) / (2 * h)
    assert np.max(np.abs(Ffd - res["forces"].numpy())) < 1e-4
    hs = 1e-6
    sfd = np.zeros((3, 3))
    vol = abs(np.linalg.det(b.lattice[0]))
    for a in range(3):
        for c in range(3):
            ep = torch.zeros(3, 3, dtype=DT); ep[a, c] = hs
            Ep = float(_energy_fixed_graph(G, sp, pos0, lat[0:1], P, CFG, ep).sum())
            Em = float(_energy_fixed_graph(G, sp, pos0, lat[0:1], P, CFG, -ep).sum())
            sfd[a, c] = 160.21766208 / vol * (Ep - Em) / (2 * hs)
    s = res["stress"].numpy()[0]
    assert np.max(np.abs(sfd - s)) < 1e-4
    assert np.max(np.abs(s - s.T)) < 1e-10


def test_parameter_gradient_fd():
    """O8 against central finite differences on a d = 8 model (one interaction
    block + final atom conv), 3 atoms, every parameter, h = 1e-5, per-tensor
    relative error < 1e-4."""
    cfg = ModelConfig(d=8, n_radial=5, n_angular=5, n_atom_conv=2, n_bond_conv=1, gmlp_hidden=8,
                      head_hidden=8)
    rng = np.random.default_rng(0)
    L = np.eye(3) * 6.0
    pos = np.array([[0.0, 0.0, 0.0], [1.6, 0.3, 0.1], [0.2, 1.7, -0.3]]) + 1.0
    b = Batch(atom_ptr=np.array([0, 3]), positions=pos, lattice=L[None], species=np.array([8, 1, 26], np.int32),
              energy_per_atom=np.array([-4.0]), forces=rng.normal(0, 0.3, (3, 3)),
              stress=rng.normal(0, 1, (1, 3, 3)), magmom=np.abs(rng.normal(size=3)),
              magmom_mask=np.array([1, 0, 1], np.uint8))
    g = build_graph_batch(b, cfg.r_atom, cfg.r_bond)
    assert g.n_angles > 0
    p = init_flat_params(param_layout(cfg), seed=3, bias_scale=0.3)
    # wide Huber δ so the loss is smooth at the test point
    lc = LossConfig(delta=10.0)
    _, grad, _ = loss_and_grad(g, b, p, cfg, lc)
    G = TGraph.from_graph(g)
    sp, dd, lat = torch.as_tensor(b.species), torch.as_tensor(g.d), torch.as_tensor(b.lattice)

    def L(x):
        with torch.no_grad():
            out = forward(G, sp, dd, lat, unflatten(torch.as_tensor(x), cfg), cfg)
            return float(loss_terms(out, b, lc, 1, 3, int(b.magmom_mask.sum()))["total"])
    # 4-point central stencil, truncation O(h^4)
    h = 1e-3
    fd = np.zeros_like(p)
    for k in range(p.size):
        x = p.copy()
        vals = []
        for s_ in (1, -1, 2, -2):
            x[k] = p[k] + s_ * h
            vals.append(L(x))
        fd[k] = (8 * (vals[0] - vals[1]) - (vals[2] - vals[3])) / (12 * h)
    off = 0
    for name, shape in param_layout(cfg):
        n = int(np.prod(shape))
        gr, f = grad[off:off + n], fd[off:off + n]
        off += n
        if name.startswith("angle0"):       # t = n_bond_conv-1 angle update is dead (Q17)
            assert np.all(gr == 0), name
            continue
        nrm = np.linalg.norm(f)
        assert nrm > 0, name
        assert np.linalg.norm(gr - f) / nrm < 1e-4, name
