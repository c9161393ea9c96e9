"""Closed-form pins of the oracle's GatedMLP, the multiplicative message forms of
Eq. 4 / Eq. 5, the angle update (Eq. 6) and the hidden layers of
the readout heads (Eq. 7, Eq. 9).

Each case is built so that one plausible mistake in the oracle flips a sign or changes a
value by O(1) (VERDICT r01 "What's weak" #1); `tools/oracle_mutations.py` applies those
mistakes to a copy of `oracle/model.py` and checks that this file fails for every one:
  sigma/SiLU swapped between the gate and core branches, LayerNorm dropped, the hidden
  SiLU of the Linear-SiLU-Linear Fc dropped (reading Q12), e^a moved inside phi, one e^b
  factor dropped, the message summed at the neighbour instead of the centre, and a hidden
  SiLU of each readout head dropped.
Expected values come from the scalar definitions of sigmoid / SiLU (math.exp) and from
d = 2 LayerNorm, whose normalised output is exactly +-|h1 - h2| / sqrt((h1 - h2)^2 + 4 eps).
"""
import math

import numpy as np
import torch

from chg_inputs import si_diamond
from oracle.graph import build_graph_batch
from oracle.model import (DT, ModelConfig, TGraph, angle_update, atom_conv, bond_conv, forward, gated_mlp,
                          param_layout, unflatten)

CFG = ModelConfig()
EPS = 1e-5   # LayerNorm epsilon (reading Q14)


def sig(x):
    return 1.0 / (1.0 + math.exp(-x))


def silu(x):
    return x * sig(x)


def ln2(h1, h2, g, b):
    """d = 2 LayerNorm written out: mean (h1+h2)/2, biased variance ((h1-h2)/2)^2."""
    s = (h1 - h2) / math.sqrt((h1 - h2) ** 2 + 4.0 * EPS)
    return g[0] * s + b[0], -g[1] * s + b[1]


def T(x):
    return torch.tensor(x, dtype=DT)


def gmlp_params(prefix, hidden, W1c, b1c, W2c, b2c, W1g, b1g, W2g, b2g, gc, bc, gg, bg):
    P = {}
    for br, (W1, b1, W2, b2) in (("core", (W1c, b1c, W2c, b2c)), ("gate", (W1g, b1g, W2g, b2g))):
        if hidden:
            P.update({f"{prefix}.{br}.W1": T(W1), f"{prefix}.{br}.b1": T(b1),
                      f"{prefix}.{br}.W2": T(W2), f"{prefix}.{br}.b2": T(b2)})
        else:
            P.update({f"{prefix}.{br}.W": T(W1), f"{prefix}.{br}.b": T(b1)})
    P.update({f"{prefix}.ln_core.g": T(gc), f"{prefix}.ln_core.b": T(bc),
              f"{prefix}.ln_gate.g": T(gg), f"{prefix}.ln_gate.b": T(bg)})
    return P


# ---------------------------------------------------------------------------------------
# GatedMLP phi(x) = sigma(LN_g(Fc_g(x))) * SiLU(LN_c(Fc_c(x)))   (Q12-Q14)
# ---------------------------------------------------------------------------------------

def test_gmlp_ln_d2_closed_form():
    """Fc = one Linear (angle-update form): Fc_c(x) = (1, 2) -> LN at d = 2 gives
    (-g1, +g2) + beta up to the epsilon term; the gate branch Fc_g(x) = (3, -4)."""
    x = [[1.0]]
    gc, bc, gg, bg = [1.5, 0.5], [0.2, -0.1], [0.7, 1.3], [0.05, -0.3]
    P = gmlp_params("m", 0, [[1.0, 2.0]], [0.0, 0.0], None, None, [[3.0, -4.0]], [0.0, 0.0], None, None,
                    gc, bc, gg, bg)
    phi = gated_mlp(T(x), P, "m", 0).numpy()[0]
    c1, c2 = ln2(1.0, 2.0, gc, bc)
    g1, g2 = ln2(3.0, -4.0, gg, bg)
    exp = [sig(g1) * silu(c1), sig(g2) * silu(c2)]
    np.testing.assert_allclose(phi, exp, rtol=1e-13)
    # the normalised core output is the sign pattern (-1, +1): gains enter with sign
    assert c1 < 0.2 - 1.49 and c2 > -0.1 + 0.49


def test_gmlp_branches_with_zero_ln_gain():
    """LN gain 0 on both branches: phi = sigma(beta_gate) * SiLU(beta_core) for any x.
    sigma and SiLU swapped between the branches gives sigma(beta_core) * SiLU(beta_gate)."""
    d = 3
    rng = np.random.default_rng(0)
    x = rng.normal(size=(5, 4))
    bc, bg = [1.1, -2.0, 0.4], [0.3, -0.7, 2.5]
    P = gmlp_params("m", 6, rng.normal(size=(4, 6)), rng.normal(size=6), rng.normal(size=(6, d)), rng.normal(size=d),
                    rng.normal(size=(4, 6)), rng.normal(size=6), rng.normal(size=(6, d)), rng.normal(size=d),
                    [0.0] * d, bc, [0.0] * d, bg)
    phi = gated_mlp(T(x), P, "m", 6).numpy()
    exp = np.array([sig(bg[k]) * silu(bc[k]) for k in range(d)])
    np.testing.assert_allclose(phi, np.broadcast_to(exp, phi.shape), rtol=1e-13)


def test_gmlp_hidden_silu_non_monotone():
    """Fc = Linear-SiLU-Linear (reading Q12) with hidden pre-activations (-1, -2):
    SiLU(-1) = -0.2689 < SiLU(-2) = -0.2384, so the core branch's d = 2 LN output is
    (-1, +1); without the hidden SiLU it would be (+1, -1).  Gate: LN gain 0, beta 0
    -> sigma(0) = 1/2."""
    P = gmlp_params("m", 2, [[-1.0, -2.0]], [0.0, 0.0], [[1.0, 0.0], [0.0, 1.0]], [0.0, 0.0],
                    [[0.5, 0.25]], [0.0, 0.0], [[1.0, 0.0], [0.0, 1.0]], [0.0, 0.0],
                    [1.0, 1.0], [0.0, 0.0], [0.0, 0.0], [0.0, 0.0])
    phi = gated_mlp(T([[1.0]]), P, "m", 2).numpy()[0]
    c1, c2 = ln2(silu(-1.0), silu(-2.0), [1.0, 1.0], [0.0, 0.0])
    assert c1 < -0.9 and c2 > 0.9
    np.testing.assert_allclose(phi, [0.5 * silu(c1), 0.5 * silu(c2)], rtol=1e-12)
    # the second linear's bias enters before LN: b2 = (0, -0.1) moves the pair to
    # (-0.2689, -0.3384) and flips the order again
    P["m.core.b2"] = T([0.0, -0.1])
    phi = gated_mlp(T([[1.0]]), P, "m", 2).numpy()[0]
    c1, c2 = ln2(silu(-1.0), silu(-2.0) - 0.1, [1.0, 1.0], [0.0, 0.0])
    assert c1 > 0.9
    np.testing.assert_allclose(phi, [0.5 * silu(c1), 0.5 * silu(c2)], rtol=1e-12)


# ---------------------------------------------------------------------------------------
# Eq. 4 / Eq. 5 / Eq. 6 message forms with a constant phi (LN gains 0)
# ---------------------------------------------------------------------------------------

def _layer_params(bc, bg):
    """Full-size layer parameters (d = 64) with random Fc weights, LN gains 0 (so phi is the
    constant c = sigma(bg) * SiLU(bc)) and identity output linears."""
    rng = np.random.default_rng(11)
    flat = torch.as_tensor(rng.normal(size=sum(int(np.prod(s)) for _, s in param_layout(CFG))) * 0.3)
    P = unflatten(flat, CFG)
    for pre in ("atom0", "bond0", "angle0"):
        P[f"{pre}.ln_core.g"].zero_(); P[f"{pre}.ln_gate.g"].zero_()
        P[f"{pre}.ln_core.b"].copy_(T(bc)); P[f"{pre}.ln_gate.b"].copy_(T(bg))
    for pre in ("atom0", "bond0"):
        P[f"{pre}.out.W"].copy_(torch.eye(CFG.d, dtype=DT)); P[f"{pre}.out.b"].zero_()
    c = np.array([sig(bg[k]) * silu(bc[k]) for k in range(CFG.d)])
    return P, c


def _tiny_graph():
    """4 atoms; edges 0->1, 0->2, 3->0, 2->0 (the first three are bonds b0, b1, b2);
    angles (b0, b1) and (b1, b0) at centre 0."""
    t = lambda x: torch.tensor(x, dtype=torch.int64)  # noqa: E731
    return TGraph(N=4, E=4, B=3, A=2, ctr=t([0, 0, 3, 2]), nbr=t([1, 2, 0, 0]), img=t([[0, 0, 0]] * 4),
                  bond_edge=t([0, 1, 2]), a_b1=t([0, 1]), a_b2=t([1, 0]), struct_of_atom=t([0, 0, 0, 0]),
                  struct_of_edge=t([0, 0, 0, 0]), S=1)


def test_atom_conv_message_is_ea_times_phi():
    """Eq. 4 with constant phi = c and L_v = identity: v'_i - v_i = (sum over edges with
    centre i of e^a_e) * c.  Atom 1 is only a neighbour and receives nothing."""
    rng = np.random.default_rng(1)
    bc, bg = rng.normal(size=CFG.d), rng.normal(size=CFG.d)
    P, c = _layer_params(bc, bg)
    G = _tiny_graph()
    v, e, ea = (T(rng.normal(size=(n, CFG.d))) for n in (4, 4, 4))
    dv = (atom_conv(0, v, e, ea, G, P, CFG) - v).numpy()
    ean = ea.numpy()
    np.testing.assert_allclose(dv[0], (ean[0] + ean[1]) * c, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dv[1], 0.0, atol=0)
    np.testing.assert_allclose(dv[2], ean[3] * c, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dv[3], ean[2] * c, rtol=1e-12, atol=1e-14)


def test_bond_conv_message_is_eb_eb_phi():
    """Eq. 5 with constant phi = c and L_e = identity: the bond row of edge(b1) gains
    e^b_{b1} * e^b_{b2} * c for each angle (b1, b2) whose FIRST bond is b1; bond b2 and the
    non-bond edge 3 are unchanged (Q16 with zero bias)."""
    rng = np.random.default_rng(2)
    bc, bg = rng.normal(size=CFG.d), rng.normal(size=CFG.d)
    P, c = _layer_params(bc, bg)
    G = _tiny_graph()
    v, e, a, eb = T(rng.normal(size=(4, CFG.d))), T(rng.normal(size=(4, CFG.d))), T(rng.normal(size=(2, CFG.d))), \
        T(rng.normal(size=(3, CFG.d)))
    de = (bond_conv(0, v, e, a, eb, G, P, CFG) - e).numpy()
    ebn = eb.numpy()
    np.testing.assert_allclose(de[0], ebn[0] * ebn[1] * c, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(de[1], ebn[1] * ebn[0] * c, rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(de[2], 0.0)
    np.testing.assert_array_equal(de[3], 0.0)


def test_angle_update_adds_phi():
    """Eq. 6: a' = a + phi_a; with LN gains 0, a' - a = sigma(beta_gate) * SiLU(beta_core)."""
    rng = np.random.default_rng(3)
    bc, bg = rng.normal(size=CFG.d), rng.normal(size=CFG.d)
    P, c = _layer_params(bc, bg)
    G = _tiny_graph()
    v, e, a = T(rng.normal(size=(4, CFG.d))), T(rng.normal(size=(4, CFG.d))), T(rng.normal(size=(2, CFG.d)))
    da = (angle_update(0, v, e, a, G, P, CFG) - a).numpy()
    np.testing.assert_allclose(da, np.broadcast_to(c, da.shape), rtol=1e-12)


# ---------------------------------------------------------------------------------------
# readout heads: hidden layers enter (Eq. 7, Eq. 9)
# ---------------------------------------------------------------------------------------

def _head_model():
    """All interaction outputs frozen (L_v = L_e = 0, zero biases) so v^4 = v^0 = W_v[Z-1]
    and e^3 = e^0; every head works on channel 0 only, so each reduces to a scalar chain
    whose hidden pre-activations sit in SiLU's non-monotone region."""
    flat = torch.zeros(sum(int(np.prod(s)) for _, s in param_layout(CFG)), dtype=DT)
    P = unflatten(flat, CFG)
    P["rbf_a.freq"].copy_(torch.arange(1, 32, dtype=DT) * math.pi)
    P["rbf_b.freq"].copy_(torch.arange(1, 32, dtype=DT) * math.pi)
    P["embed.W"][13, 0] = 2.0                                   # Si: v_0 = 2
    # energy head 64 -> 64 -> 64 -> 64 -> 1, SiLU after each hidden linear
    P["head_E.W0"][0, 0] = -1.0; P["head_E.b0"][0] = 0.0         # -2
    P["head_E.W1"][0, 0] = 4.0; P["head_E.b1"][0] = 0.0
    P["head_E.W2"][0, 0] = -3.0; P["head_E.b2"][0] = -1.0
    P["head_E.W3"][0, 0] = 1.5; P["head_E.b3"][0] = 0.1
    # magmom: linear
    P["head_M.W"][0, 0] = 0.75; P["head_M.b"][0] = -0.2
    # force head 64 -> 64 -> 64 -> 1 with W0 = 0: n = W2 . SiLU(W1 . SiLU(b0) + b1) + b2
    P["head_F.b0"][0] = -1.5; P["head_F.b0"][1] = -0.5
    P["head_F.W1"][0, 0] = 2.0; P["head_F.W1"][1, 0] = -1.0; P["head_F.b1"][0] = -0.3
    P["head_F.W2"][0, 0] = -2.5; P["head_F.b2"][0] = 0.05
    # stress head 64 -> 64 -> 64 -> 9 on channel 0 of v: M = m * B (B fixed 3x3)
    P["head_S.W0"][0, 0] = -0.5                                  # -1
    P["head_S.W1"][0, 0] = 3.0; P["head_S.b1"][0] = 0.5
    Bm = np.array([[1.0, -2.0, 0.5], [0.0, 3.0, 1.0], [2.0, -1.0, -0.5]])
    P["head_S.W2"][0, :] = T(Bm.reshape(-1))
    return P, Bm


def test_head_hidden_layers_closed_form():
    b = si_diamond(jitter=0.05, seed=7)
    g = build_graph_batch(b, CFG.r_atom, CFG.r_bond)
    P, Bm = _head_model()
    out = forward(TGraph.from_graph(g), torch.as_tensor(b.species), torch.as_tensor(g.d),
                  torch.as_tensor(b.lattice.reshape(-1, 3, 3)), P, CFG)
    # energy: e_atom = 1.5 * SiLU(-3 * SiLU(4 * SiLU(-2)) - 1) + 0.1 per atom
    h = silu(-2.0); h = silu(4.0 * h); h = silu(-3.0 * h - 1.0)
    e_atom = 1.5 * h + 0.1
    np.testing.assert_allclose(out["energy"].numpy(), [8 * e_atom], rtol=1e-13)
    np.testing.assert_allclose(out["magmom"].numpy(), 0.75 * 2.0 - 0.2, rtol=1e-13)
    # force: F_i = n * sum_{e at i} x_hat_e (Eq. 7) with the hidden chain inside n
    n = -2.5 * silu(2.0 * silu(-1.5) - 1.0 * silu(-0.5) - 0.3) + 0.05
    xh = g.d / np.linalg.norm(g.d, axis=1, keepdims=True)
    F = np.zeros((8, 3)); np.add.at(F, g.center, n * xh)
    np.testing.assert_allclose(out["forces"].numpy(), F, rtol=1e-12, atol=1e-13)
    # stress: sigma = (1/N) sum_i sym(m B) * G with m = SiLU(3 * SiLU(-1) + 0.5)
    m = silu(3.0 * silu(-1.0) + 0.5)
    Lh = b.lattice[0] / np.linalg.norm(b.lattice[0], axis=1, keepdims=True)
    sh = Lh.sum(0)
    exp = m * 0.5 * (Bm + Bm.T) * np.outer(sh, sh)
    np.testing.assert_allclose(out["stress"].numpy()[0], exp, rtol=1e-12, atol=1e-14)


def test_bond_conv_sums_over_the_first_bond():
    """Eq. 5: the sum over k != j runs over the angles whose FIRST bond is ij.  One angle
    (b0, b1) alone: bond b0's edge gains e^b_0 * e^b_1 * c and bond b1's edge nothing."""
    rng = np.random.default_rng(4)
    bc, bg = rng.normal(size=CFG.d), rng.normal(size=CFG.d)
    P, c = _layer_params(bc, bg)
    G = _tiny_graph()
    G.A, G.a_b1, G.a_b2 = 1, G.a_b1[:1], G.a_b2[:1]
    v, e, a, eb = T(rng.normal(size=(4, CFG.d))), T(rng.normal(size=(4, CFG.d))), T(rng.normal(size=(1, CFG.d))), \
        T(rng.normal(size=(3, CFG.d)))
    de = (bond_conv(0, v, e, a, eb, G, P, CFG) - e).numpy()
    ebn = eb.numpy()
    np.testing.assert_allclose(de[0], ebn[0] * ebn[1] * c, rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(de[1], 0.0)
