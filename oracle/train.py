"""O7 loss, O8 parameter gradients, O9 Adam + LR, O11 balance sampler
(oracle; test infrastructure).

  loss       P:370 "Huber loss, with the prefactor defined as 2, 1.5, 0.1, 0.1";
             readings Q22 (δ = 0.1), Q23 (per-atom energy, component means,
             labelled-magmom mean, GLOBAL normalisers)
  Adam       P:370 "'Adam' optimizer"; reading Q24 (PyTorch semantics)
  LR         Eq. 14: init_LR = batch/k × 3e-4, k = 128; cosine
  sampler    P:330-331 (Fig. 4): sort ascending by atoms+bonds+angles, each GPU
             takes the smallest and largest remaining in turn; reading Q25, Q31
  CV         P:425 coefficient of variation of per-GPU feature number
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from .graph import Graph
from .model import DT, ModelConfig, TGraph, forward, unflatten


@dataclasses.dataclass
class LossConfig:
    w_e: float = 2.0
    w_f: float = 1.5
    w_s: float = 0.1
    w_m: float = 0.1
    delta: float = 0.1
    n_struct_global: Optional[int] = None   # S_g (defaults to the batch's)
    n_atoms_global: Optional[int] = None    # N_g
    n_magmom_global: Optional[int] = None   # M_g


def huber(x: torch.Tensor, delta: float) -> torch.Tensor:
    """H(x) = ½x² if |x| < δ else δ(|x| − ½δ)."""
    ax = torch.abs(x)
    return torch.where(ax < delta, 0.5 * x * x, delta * (ax - 0.5 * delta))


def loss_terms(out: Dict[str, torch.Tensor], labels, lc: LossConfig, n_struct: int, n_atoms: int,
               n_mag: int) -> Dict[str, torch.Tensor]:
    """L = (w_e/S_g)ΣH(Δε) + (w_f/(3N_g))ΣH(ΔF) + (w_s/(9S_g))ΣH(Δσ) + (w_m/M_g)Σ_mask H(Δm)."""
    Sg = lc.n_struct_global or n_struct
    Ng = lc.n_atoms_global or n_atoms
    Mg = lc.n_magmom_global if lc.n_magmom_global is not None else n_mag
    d = lc.delta
    eps_hat = torch.as_tensor(np.asarray(labels.energy_per_atom, np.float64))
    f_hat = torch.as_tensor(np.asarray(labels.forces, np.float64))
    s_hat = torch.as_tensor(np.asarray(labels.stress, np.float64)).reshape(-1, 3, 3)
    m_hat = torch.as_tensor(np.asarray(labels.magmom, np.float64))
    mask = torch.as_tensor(np.asarray(labels.magmom_mask, np.float64))
    LE = lc.w_e / Sg * huber(out["energy_per_atom"] - eps_hat, d).sum()
    LF = lc.w_f / (3.0 * Ng) * huber(out["forces"] - f_hat, d).sum()
    LS = lc.w_s / (9.0 * Sg) * huber(out["stress"] - s_hat, d).sum()
    LM = (lc.w_m / Mg * (huber(out["magmom"] - m_hat, d) * mask).sum()) if Mg > 0 else \
        torch.zeros((), dtype=DT)
    return {"total": LE + LF + LS + LM, "E": LE, "F": LF, "S": LS, "M": LM}


def loss_and_grad(graph: Graph, batch, flat_params, cfg: ModelConfig, lc: LossConfig = LossConfig()):
    """O7 + O8: loss terms and dL/dθ for every parameter (flat fp64 vector),
    the exact reverse mode of `oracle.model.forward` via autograd."""
    G = TGraph.from_graph(graph)
    flat = torch.as_tensor(np.asarray(flat_params, np.float64)).clone().requires_grad_(True)
    P = unflatten(flat, cfg)
    out = forward(G, torch.as_tensor(np.asarray(batch.species)), torch.as_tensor(graph.d),
                  torch.as_tensor(np.asarray(batch.lattice, np.float64).reshape(-1, 3, 3)), P, cfg)
    terms = loss_terms(out, batch, lc, G.S, G.N, int(np.asarray(batch.magmom_mask).sum()))
    (g,) = torch.autograd.grad(terms["total"], flat)
    return {k: float(v.detach()) for k, v in terms.items()}, g.numpy(), \
        {k: v.detach().numpy() for k, v in out.items()}


# ----------------------------------------------------------------------------
# O9 Adam and learning rate
# ----------------------------------------------------------------------------

def init_lr(global_batch: int, base: float = 3e-4, k: int = 128) -> float:
    """Eq. 14: init_LR = batch_size / k × 0.0003, k = 128."""
    return global_batch / k * base


def cosine_lr(step: int, total_steps: int, lr0: float) -> float:
    """Cosine annealing, per optimizer step, no warm-up (Q24)."""
    return lr0 * 0.5 * (1.0 + math.cos(math.pi * step / total_steps))


def adam_step(theta, m, v, g, step: int, lr: float, beta1=0.9, beta2=0.999, eps=1e-8):
    """PyTorch Adam (no weight decay).  `step` is the 1-based step count after
    the increment.  Returns new (theta, m, v) as fp64 numpy arrays."""
    theta = np.asarray(theta, np.float64); m = np.asarray(m, np.float64)
    v = np.asarray(v, np.float64); g = np.asarray(g, np.float64)
    m = beta1 * m + (1 - beta1) * g
    v = beta2 * v + (1 - beta2) * g * g
    mhat = m / (1 - beta1 ** step)
    vhat = v / (1 - beta2 ** step)
    theta = theta - lr * mhat / (np.sqrt(vhat) + eps)
    return theta, m, v


# ----------------------------------------------------------------------------
# O11 load-balance sampler
# ----------------------------------------------------------------------------

def balance_assign(loads: Sequence[int], n_ranks: int) -> List[List[int]]:
    """sort ascending (ties by index, Q25); ranks take turns
    round-robin, each turn taking the smallest AND the largest remaining sample
    (one if only one remains).  Returns per-rank lists of sample indices."""
    if n_ranks <= 0:
        raise ValueError("n_ranks must be >= 1")
    order = sorted(range(len(loads)), key=lambda i: (loads[i], i))
    lo, hi = 0, len(order) - 1
    out: List[List[int]] = [[] for _ in range(n_ranks)]
    turn = 0
    while lo <= hi:
        r = turn % n_ranks
        out[r].append(order[lo]); lo += 1
        if lo <= hi:
            out[r].append(order[hi]); hi -= 1
        turn += 1
    return out


def coefficient_of_variation(per_rank_loads: Sequence[float]) -> float:
    """Population std / mean."""
    x = np.asarray(per_rank_loads, np.float64)
    if x.mean() == 0:
        raise ValueError("zero mean")
    return float(x.std() / x.mean())
