"""O2–O6, O8, O10 — FastCHGNet model definition in fp64 (oracle; test infrastructure).

Plain PyTorch CPU ops in float64, no fusion, no blocking, in the paper's order
and notation.  Gradients (O8) and energy-derived force/stress (O10) are taken
by torch autograd, i.e. the exact reverse mode of the forward written here.

Paper map (PAPER.md line numbers, readings from SURVEY.md §8(c)):
  envelope u(ξ)        Eq. 12/13; reading Q2 (DimeNet polynomial)
  sRBF                 P:97 (cites DimeNet); reading Q3, Q4 (two bases a/b)
  Fourier basis FT     P:97; reading Q6
  embedding            Eq. 2; readings Q5 (no bias), Q28 (94 rows)
  GatedMLP φ           P:139 (+Fig. 3b); readings Q12, Q13, Q14
  Atom Conv            Eq. 4; reading Q15
  Bond Conv            Eq. 5, P:123-129 with Eq. 11 inputs; Q16
  Angle Update         Eq. 6, P:130-136 with Eq. 11 inputs; Q17 (t=2 dead)
  Energy head          P:141; reading Q18
  Magmom head          P:21/P:93; reading Q19
  Force head           Eq. 7; reading Q20
  Stress head          Eq. 9; reading Q21
  derived F, σ (O10)   P:168 (F = -∂E/∂x, σ = (1/V) ∂E/∂ε); reading Q27
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from .graph import Graph

DT = torch.float64
EV_PER_A3_TO_GPA = 160.21766208


@dataclasses.dataclass
class ModelConfig:
    d: int = 64
    n_radial: int = 31
    n_angular: int = 31
    envelope_p: int = 8
    n_atom_conv: int = 4       # t = 0..3 (three interaction blocks + final atom conv)
    n_bond_conv: int = 3       # t = 0..2 (angle update at t = 2 is dead, Q17)
    gmlp_hidden: int = 64      # Q12: Linear-SiLU-Linear per branch; 0 = single Linear
    n_species: int = 94
    head_hidden: int = 64
    r_atom: float = 5.0
    r_bond: float = 3.0


# ----------------------------------------------------------------------------
# canonical parameter layout (the oracle's own table; the CUDA library reports
# its own through chg_model_layout and a test checks that the two agree)
# ----------------------------------------------------------------------------

def param_layout(cfg: ModelConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    d, h = cfg.d, cfg.gmlp_hidden
    L: List[Tuple[str, Tuple[int, ...]]] = [("embed.W", (cfg.n_species, d)),
                                            ("rbf_a.freq", (cfg.n_radial,)),
                                            ("rbf_b.freq", (cfg.n_radial,)),
                                            ("proj.W0", (cfg.n_radial, d)),
                                            ("proj.Wa", (cfg.n_radial, d)),
                                            ("proj.Wb", (cfg.n_radial, d)),
                                            ("proj.Wtheta", (cfg.n_angular, d))]

    def gmlp(prefix, fan_in, hidden):
        out = []
        for br in ("core", "gate"):
            if hidden:
                out += [(f"{prefix}.{br}.W1", (fan_in, hidden)), (f"{prefix}.{br}.b1", (hidden,)),
                        (f"{prefix}.{br}.W2", (hidden, d)), (f"{prefix}.{br}.b2", (d,))]
            else:
                out += [(f"{prefix}.{br}.W", (fan_in, d)), (f"{prefix}.{br}.b", (d,))]
        out += [(f"{prefix}.ln_core.g", (d,)), (f"{prefix}.ln_core.b", (d,)),
                (f"{prefix}.ln_gate.g", (d,)), (f"{prefix}.ln_gate.b", (d,))]
        return out

    for t in range(cfg.n_atom_conv):
        L += gmlp(f"atom{t}", 3 * d, h)
        L += [(f"atom{t}.out.W", (d, d)), (f"atom{t}.out.b", (d,))]
    for t in range(cfg.n_bond_conv):
        L += gmlp(f"bond{t}", 4 * d, h)
        L += [(f"bond{t}.out.W", (d, d)), (f"bond{t}.out.b", (d,))]
    for t in range(cfg.n_bond_conv):
        L += gmlp(f"angle{t}", 4 * d, 0)
    H = cfg.head_hidden

    def mlp(prefix, dims):
        out = []
        for k in range(len(dims) - 1):
            out += [(f"{prefix}.W{k}", (dims[k], dims[k + 1])), (f"{prefix}.b{k}", (dims[k + 1],))]
        return out

    L += mlp("head_E", [d, H, H, H, 1])
    L += [("head_M.W", (d, 1)), ("head_M.b", (1,))]
    L += mlp("head_F", [d, H, H, 1])
    L += mlp("head_S", [d, H, H, 9])
    return L


def param_count(cfg: ModelConfig) -> int:
    return int(sum(int(np.prod(s)) for _, s in param_layout(cfg)))


def unflatten(flat: torch.Tensor, cfg: ModelConfig) -> Dict[str, torch.Tensor]:
    P, off = {}, 0
    for name, shape in param_layout(cfg):
        n = int(np.prod(shape))
        P[name] = flat[off:off + n].view(shape)
        off += n
    assert off == flat.numel(), (off, flat.numel())
    return P


# ----------------------------------------------------------------------------
# O2 basis
# ----------------------------------------------------------------------------

def envelope(xi: torch.Tensor, p: int) -> torch.Tensor:
    """u(ξ) = 1 − (p+1)(p+2)/2·ξ^p + p(p+2)·ξ^{p+1} − p(p+1)/2·ξ^{p+2}.
    Reading Q2: the DimeNet polynomial (the paper's Eq. 12 third coefficient
    and Eq. 13 signs are garbled; this is the only reading with u(1)=u'(1)=0).
    Evaluated once-ξ^p and factored, the intent of Eq. 13."""
    xp = xi ** p
    return 1.0 - xp * ((p + 1) * (p + 2) / 2.0 - p * (p + 2) * xi + p * (p + 1) / 2.0 * xi * xi)


def srbf(r: torch.Tensor, freq: torch.Tensor, r_cut: float, p: int) -> torch.Tensor:
    """ẽ_n(r) = u(r/r_c)·sqrt(2/r_c)·sin(f_n r / r_c)/r, n = 1..K (Q3; P:97 cites
    DimeNet's smooth radial Bessel basis; f_n trainable, init nπ)."""
    xi = (r / r_cut)[:, None]
    return envelope(xi, p) * math.sqrt(2.0 / r_cut) * torch.sin(freq[None, :] * xi) / r[:, None]


def fourier(theta: torch.Tensor, n: int) -> torch.Tensor:
    """FT(θ) = [1/√(2π), cos θ/√π, sin θ/√π, cos 2θ/√π, sin 2θ/√π, …] (Q6)."""
    cols = [torch.full_like(theta, 1.0 / math.sqrt(2.0 * math.pi))]
    k = 1
    while len(cols) < n:
        cols.append(torch.cos(k * theta) / math.sqrt(math.pi))
        if len(cols) < n:
            cols.append(torch.sin(k * theta) / math.sqrt(math.pi))
        k += 1
    return torch.stack(cols, dim=1)


# ----------------------------------------------------------------------------
# O4 GatedMLP
# ----------------------------------------------------------------------------

def layer_norm(h: torch.Tensor, g: torch.Tensor, b: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    """LN(h) = g ⊙ (h − μ)/sqrt(var + ε) + b, biased variance (Q14)."""
    mu = h.mean(dim=-1, keepdim=True)
    var = ((h - mu) ** 2).mean(dim=-1, keepdim=True)
    return g * (h - mu) / torch.sqrt(var + eps) + b


def silu(x):
    return x * torch.sigmoid(x)


def gated_mlp(x: torch.Tensor, P: Dict[str, torch.Tensor], prefix: str, hidden: int) -> torch.Tensor:
    """φ(x) = (σ ∘ LN ∘ Fc(x)) ⊙ (g ∘ LN ∘ Fc(x)): σ = Sigmoid on the
    gate branch, g = SiLU on the core branch (Q13); Fc = Linear–SiLU–Linear when
    hidden > 0 (Q12), else one Linear."""
    def fc(br):
        if hidden:
            h1 = silu(x @ P[f"{prefix}.{br}.W1"] + P[f"{prefix}.{br}.b1"])
            return h1 @ P[f"{prefix}.{br}.W2"] + P[f"{prefix}.{br}.b2"]
        return x @ P[f"{prefix}.{br}.W"] + P[f"{prefix}.{br}.b"]
    hc = layer_norm(fc("core"), P[f"{prefix}.ln_core.g"], P[f"{prefix}.ln_core.b"])
    hg = layer_norm(fc("gate"), P[f"{prefix}.ln_gate.g"], P[f"{prefix}.ln_gate.b"])
    return torch.sigmoid(hg) * silu(hc)


# ----------------------------------------------------------------------------
# O5 interaction blocks (Eq. 4, 5, 6 with the Eq. 11 inputs)
# ----------------------------------------------------------------------------

@dataclasses.dataclass
class TGraph:
    """Graph index tensors (torch, int64) used by the model."""
    N: int
    E: int
    B: int
    A: int
    ctr: torch.Tensor
    nbr: torch.Tensor
    img: torch.Tensor
    bond_edge: torch.Tensor
    a_b1: torch.Tensor
    a_b2: torch.Tensor
    struct_of_atom: torch.Tensor
    struct_of_edge: torch.Tensor
    S: int

    @staticmethod
    def from_graph(g: Graph) -> "TGraph":
        t = lambda x: torch.as_tensor(np.asarray(x, np.int64))  # noqa: E731
        soa = t(g.struct_of_atom)
        return TGraph(N=g.n_atoms, E=g.n_edges, B=g.n_bonds, A=g.n_angles, ctr=t(g.center),
                      nbr=t(g.nbr), img=t(g.img), bond_edge=t(g.bond_edge), a_b1=t(g.angle_b1),
                      a_b2=t(g.angle_b2), struct_of_atom=soa, struct_of_edge=soa[t(g.center)],
                      S=int(g.counts.shape[0]))


def atom_conv(t: int, v, e, ea, G: TGraph, P, cfg: ModelConfig):
    """Eq. 4: v^{t+1}_i = v^t_i + 𝓛^t_v[ Σ_{j∈N(i)} eᵃ_ij ⊙ φ^t_v([v_i, v_j, e_ij]) ]."""
    x = torch.cat([v[G.ctr], v[G.nbr], e], dim=1)
    m = ea * gated_mlp(x, P, f"atom{t}", cfg.gmlp_hidden)
    agg = torch.zeros(G.N, cfg.d, dtype=DT).index_add(0, G.ctr, m)
    return v + agg @ P[f"atom{t}.out.W"] + P[f"atom{t}.out.b"]


def _angle_input(v, e, a, G: TGraph):
    """f = [v^t_i, e^t_ij, e^t_ik, a^t_ijk] — Eq. 11 inputs shared
    by Bond Conv and Angle Update."""
    e1 = G.bond_edge[G.a_b1]
    e2 = G.bond_edge[G.a_b2]
    return torch.cat([v[G.ctr[e1]], e[e1], e[e2], a], dim=1)


def bond_conv(t: int, v, e, a, eb, G: TGraph, P, cfg: ModelConfig):
    """Eq. 5 with Eq. 11 inputs: e^{t+1}_ij = e^t_ij + 𝓛^t_e[ Σ_{k≠j} eᵇ_ij ⊙ eᵇ_ik ⊙
    φ^t_e([v^t_i, e^t_ij, e^t_ik, a^t_ijk]) ]; 𝓛_e applied to every atom-graph
    edge (empty sum for non-bond edges, Q16)."""
    x = _angle_input(v, e, a, G)
    q = eb[G.a_b1] * eb[G.a_b2] * gated_mlp(x, P, f"bond{t}", cfg.gmlp_hidden)
    aggb = torch.zeros(G.B, cfg.d, dtype=DT).index_add(0, G.a_b1, q)
    agge = torch.zeros(G.E, cfg.d, dtype=DT).index_copy(0, G.bond_edge, aggb)
    return e + agge @ P[f"bond{t}.out.W"] + P[f"bond{t}.out.b"]


def angle_update(t: int, v, e, a, G: TGraph, P, cfg: ModelConfig):
    """Eq. 6 with Eq. 11 inputs: a^{t+1} = a^t + φ^t_a([v^t_i, e^t_ij, e^t_ik, a^t_ijk]),
    φ_a a GatedMLP with one Linear per branch (Q12)."""
    return a + gated_mlp(_angle_input(v, e, a, G), P, f"angle{t}", 0)


# ----------------------------------------------------------------------------
# full forward
# ----------------------------------------------------------------------------

def edge_vectors(G: TGraph, positions: torch.Tensor, lattice: torch.Tensor) -> torch.Tensor:
    """d_e = r_i − (r_j + n_e L_s) (Alg. 1; reading Q11)."""
    Ls = lattice[G.struct_of_edge]                     # [E,3,3]
    shift = torch.einsum("ek,ekc->ec", G.img.to(DT), Ls)
    return positions[G.ctr] - (positions[G.nbr] + shift)


def forward(G: TGraph, species: torch.Tensor, d: torch.Tensor, lattice: torch.Tensor,
            P: Dict[str, torch.Tensor], cfg: ModelConfig, keep: bool = False):
    """Full FastCHGNet forward (Fig. 2a order): embedding (Eq. 2) → three
    interaction blocks t = 0,1,2 (Eq. 3, 4, 5, 6 with Eq. 11) → final atom conv
    t = 3 (Q17) → energy / magmom / force / stress heads.
    `d` [E,3] edge vectors, `lattice` [S,3,3].  Returns dict of outputs (and
    intermediates when keep=True)."""
    out = {}
    r = torch.sqrt((d * d).sum(dim=1))
    # O2 bases
    ea_t = srbf(r, P["rbf_a.freq"], cfg.r_atom, cfg.envelope_p)              # ẽᵃ [E,K]
    rb = r[G.bond_edge]
    eb_t = srbf(rb, P["rbf_b.freq"], cfg.r_bond, cfg.envelope_p)             # ẽᵇ [B,K]
    d1 = d[G.bond_edge[G.a_b1]]
    d2 = d[G.bond_edge[G.a_b2]]
    c = (d1 * d2).sum(dim=1) / (rb[G.a_b1] * rb[G.a_b2])
    theta = torch.arccos(torch.clamp(c, -1.0, 1.0))
    a_t = fourier(theta, cfg.n_angular)                                      # ã [A,K]
    # O3 embedding and projections (Eq. 2; no bias, Q5)
    v = P["embed.W"][species.long() - 1]
    e = ea_t @ P["proj.W0"]
    ea = ea_t @ P["proj.Wa"]
    eb = eb_t @ P["proj.Wb"]
    a = a_t @ P["proj.Wtheta"]
    if keep:
        out.update(r=r, ea_t=ea_t, eb_t=eb_t, cos_theta=c, a_t=a_t, v0=v, e0=e, ea=ea, eb=eb, a0=a)
    # O5 interaction blocks
    for t in range(cfg.n_bond_conv):
        v_n = atom_conv(t, v, e, ea, G, P, cfg)
        e_n = bond_conv(t, v, e, a, eb, G, P, cfg)
        a_n = angle_update(t, v, e, a, G, P, cfg) if t < cfg.n_bond_conv - 1 else a
        v, e, a = v_n, e_n, a_n
        if keep:
            out.update({f"v{t + 1}": v, f"e{t + 1}": e, f"a{t + 1}": a})
    for t in range(cfg.n_bond_conv, cfg.n_atom_conv):
        v = atom_conv(t, v, e, ea, G, P, cfg)
        if keep:
            out[f"v{t + 1}"] = v
    # O6 heads
    S = G.S
    n_atoms = torch.zeros(S, dtype=DT).index_add(0, G.struct_of_atom, torch.ones(G.N, dtype=DT))
    h = v
    for k in range(3):
        h = silu(h @ P[f"head_E.W{k}"] + P[f"head_E.b{k}"])
    e_atom = (h @ P["head_E.W3"] + P["head_E.b3"])[:, 0]
    energy = torch.zeros(S, dtype=DT).index_add(0, G.struct_of_atom, e_atom)
    out["energy"] = energy
    out["energy_per_atom"] = energy / n_atoms
    out["magmom"] = (v @ P["head_M.W"] + P["head_M.b"])[:, 0]
    # Force head (Eq. 7): n_ij = MLP(e_ij); F_i = Σ_j n_ij x̂_ij
    hf = e
    for k in range(2):
        hf = silu(hf @ P[f"head_F.W{k}"] + P[f"head_F.b{k}"])
    n_e = (hf @ P["head_F.W2"] + P["head_F.b2"])[:, 0]
    xhat = d / r[:, None]
    out["forces"] = torch.zeros(G.N, 3, dtype=DT).index_add(0, G.ctr, n_e[:, None] * xhat)
    # Stress head (Eq. 9): σ = Σ_i (scale·MLP(v_i)) ⊙ Σ_{pq} L̂_p ⊗ L̂_q ; scale = 1/N_s,
    # 9 outputs reshaped row-major and symmetrised (Q21)
    hs = v
    for k in range(2):
        hs = silu(hs @ P[f"head_S.W{k}"] + P[f"head_S.b{k}"])
    M = (hs @ P["head_S.W2"] + P["head_S.b2"]).view(-1, 3, 3)
    Msym = 0.5 * (M + M.transpose(1, 2))
    Lhat = lattice / torch.linalg.norm(lattice, dim=2, keepdim=True)
    s_hat = Lhat.sum(dim=1)                                                  # [S,3]
    Gs = s_hat[:, :, None] * s_hat[:, None, :]                              # Σ_pq L̂_p ⊗ L̂_q
    sig = torch.zeros(S, 3, 3, dtype=DT).index_add(0, G.struct_of_atom, Msym)
    out["stress"] = sig * Gs / n_atoms[:, None, None]
    if keep:
        out["v_final"] = v
        out["e_final"] = e
        out["n_e"] = n_e
    return out


# ----------------------------------------------------------------------------
# convenience wrappers
# ----------------------------------------------------------------------------

def run_forward(graph: Graph, species, lattice, flat_params, cfg: ModelConfig, keep=False):
    """Forward from a built oracle graph (uses the graph's canonical fp64 d)."""
    G = TGraph.from_graph(graph)
    flat = torch.as_tensor(np.asarray(flat_params, np.float64))
    P = unflatten(flat, cfg)
    return forward(G, torch.as_tensor(np.asarray(species)), torch.as_tensor(graph.d),
                   torch.as_tensor(np.asarray(lattice, np.float64).reshape(-1, 3, 3)), P, cfg, keep)


def derived_force_stress(graph: Graph, positions, lattice, species, flat_params, cfg: ModelConfig):
    """O10: F^E_i = −∂E/∂r_i and σ^E_s = (160.21766208/V_s)·∂E_s/∂ε_s (P:168,
    reading Q27) with r → r(I+ε), L → L(I+ε) per structure; graph fixed."""
    G = TGraph.from_graph(graph)
    P = unflatten(torch.as_tensor(np.asarray(flat_params, np.float64)), cfg)
    pos = torch.as_tensor(np.asarray(positions, np.float64)).clone().requires_grad_(True)
    lat = torch.as_tensor(np.asarray(lattice, np.float64).reshape(-1, 3, 3))
    eps = torch.zeros(G.S, 3, 3, dtype=DT, requires_grad=True)
    Id = torch.eye(3, dtype=DT)
    defo = Id[None] + eps
    pos_s = torch.einsum("nk,nkc->nc", pos, defo[G.struct_of_atom])
    lat_s = torch.einsum("spk,skc->spc", lat, defo)
    d = edge_vectors(G, pos_s, lat_s)
    out = forward(G, torch.as_tensor(np.asarray(species)), d, lat_s, P, cfg)
    E = out["energy"].sum()
    gpos, geps = torch.autograd.grad(E, (pos, eps))
    vol = torch.abs(torch.linalg.det(lat))
    sigma = EV_PER_A3_TO_GPA * geps / vol[:, None, None]
    return {"energy": out["energy"].detach(), "forces": -gpos, "stress": sigma}
