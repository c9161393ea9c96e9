"""Training loop around the C-ABI step.

Host-side orchestration only — every step of the computation runs in libchg:
chg_build_graph → chg_forward(train) → chg_backward (global loss normalisers) → chg_step
(NCCL allreduce when the context has a communicator, finite check, fused Adam).

* learning rate: Eq. 14, init_LR = global_batch / 128 × 3e-4, cosine annealing
  per optimizer step over the run, no warm-up (reading Q24);
* epochs over a list of structures, reshuffled per epoch with a seeded generator; with
  world_size > 1 each global batch is dealt to ranks with chg_balance;
* checkpoints: parameters, Adam m / v, the step counter and the shuffle generator state in
  one .npz — resuming reproduces the uninterrupted run bit for bit (the step is deterministic);
* graph prefetch (`prefetch=True`): the next global batch's graph is built
  on a builder context's stream while this step's backward runs (chg_graph_wait orders it).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np

from . import chg


def init_lr(global_batch: int, base: float = 3e-4, k: int = 128) -> float:
    """Eq. 14: init_LR = batch_size / k × 0.0003 with k = 128."""
    return global_batch / k * base


def cosine_lr(step: int, total_steps: int, lr0: float) -> float:
    """Cosine annealing per optimizer step; step counts from 1."""
    return lr0 * 0.5 * (1.0 + math.cos(math.pi * step / max(total_steps, 1)))


def _take(batch, idx):
    """Sub-batch of whole structures (host numpy, order preserved)."""
    idx = list(idx)
    ap = batch.atom_ptr
    atoms = np.concatenate([np.arange(ap[s], ap[s + 1]) for s in idx]) if idx else np.zeros(0, np.int64)
    n_per = [int(ap[s + 1] - ap[s]) for s in idx]
    new_ap = np.zeros(len(idx) + 1, np.int64)
    new_ap[1:] = np.cumsum(n_per)
    return dict(atom_ptr=new_ap, positions=batch.positions[atoms], lattice=batch.lattice[idx],
                species=batch.species[atoms],
                labels=dict(energy_per_atom=batch.energy_per_atom[idx].astype(np.float32),
                            forces=batch.forces[atoms].astype(np.float32),
                            stress=batch.stress[idx].astype(np.float32),
                            magmom=batch.magmom[atoms].astype(np.float32),
                            magmom_mask=batch.magmom_mask[atoms].astype(np.uint8)))


@dataclass
class TrainState:
    step: int = 0
    epoch: int = 0
    history: List[Dict[str, float]] = field(default_factory=list)


class Trainer:
    """Data-parallel trainer (one instance per rank; rank / world_size from the context)."""

    def __init__(self, ctx: chg.Context, model: chg.Model, global_batch: int, total_steps: int,
                 rank: int = 0, world_size: int = 1, seed: int = 0, r_atom: float = 5.0, r_bond: float = 3.0,
                 loss_weights=(2.0, 1.5, 0.1, 0.1), huber_delta: float = 0.1, prefetch: bool = False):
        self.ctx, self.model = ctx, model
        self.global_batch, self.total_steps = global_batch, total_steps
        self.rank, self.world_size = rank, world_size
        self.lr0 = init_lr(global_batch)
        self.rng = np.random.default_rng(seed)
        self.r_atom, self.r_bond = r_atom, r_bond
        self.w, self.delta = loss_weights, huber_delta
        self.state = TrainState()
        self._order: Optional[np.ndarray] = None      # current epoch's shuffled structure order
        self._pos = 0                                 # next global batch in it
        self.builder = chg.Context(ctx.device) if prefetch else None
        self._pending = None                          # (struct ids, local batch, graph) built ahead
        self._loads: Dict[int, int] = {}              # structure id -> atoms + edges + angles (static)

    def _local(self, batch, struct_ids, gctx):
        """This rank's share of a global batch (whole structures, chg_balance over ranks)."""
        glob = _take(batch, struct_ids)
        if self.world_size > 1:
            # the balancer's load (N + E + A) is a property of the structure: counted once per
            # structure of the dataset (one graph build of the not-yet-seen ones), then cached
            missing = sorted({int(k) for k in struct_ids if int(k) not in self._loads})
            if missing:
                part = _take(batch, missing)
                g_new = gctx.build_graph(part["atom_ptr"], part["positions"], part["lattice"], part["species"],
                                         self.r_atom, self.r_bond)
                ps = g_new.per_struct()
                g_new.close()
                for k, sid in enumerate(missing):
                    self._loads[sid] = int(ps[k, 0] + ps[k, 1] + ps[k, 3])
            owner = chg.balance(np.array([self._loads[int(k)] for k in struct_ids], np.int64), self.world_size)
            mine = [struct_ids[k] for k in range(len(struct_ids)) if owner[k] == self.rank]
            return glob, _take(batch, mine)
        return glob, glob

    # ---- one optimizer step on one global batch (whole structures) -------------
    def train_step(self, batch, struct_ids, next_ids=None) -> Dict[str, float]:
        if self._pending is not None and self._pending[0] == list(struct_ids):
            _, glob, local, g = self._pending
        else:
            glob, local = self._local(batch, struct_ids, self.ctx)
            g = self.ctx.build_graph(local["atom_ptr"], local["positions"], local["lattice"], local["species"],
                                     self.r_atom, self.r_bond)
        self._pending = None
        n_atoms = int(glob["atom_ptr"][-1])
        n_mag = int(glob["labels"]["magmom_mask"].sum())
        self.ctx.forward(self.model, g, train=True, host=False)
        if self.builder is not None and next_ids is not None:    # next step's graph, built meanwhile
            nglob, nloc = self._local(batch, next_ids, self.builder)
            ng = self.builder.build_graph(nloc["atom_ptr"], nloc["positions"], nloc["lattice"], nloc["species"],
                                          self.r_atom, self.r_bond)
            self._pending = (list(next_ids), nglob, nloc, ng)
        loss = self.ctx.backward(self.model, g, local["labels"], w=self.w, delta=self.delta,
                                 n_struct_global=len(struct_ids), n_atoms_global=n_atoms,
                                 n_magmom_global=n_mag, sync_loss=True)
        self.state.step += 1
        lr = cosine_lr(self.state.step, self.total_steps, self.lr0)
        self.ctx.step(self.model, lr=lr, step=self.state.step, allreduce=self.world_size > 1)
        if self._pending is not None:
            self.ctx.wait_graph(self._pending[3])
        g.close()
        rec = {"step": self.state.step, "lr": lr, "loss": float(loss[0]), "loss_E": float(loss[1]),
               "loss_F": float(loss[2]), "loss_S": float(loss[3]), "loss_M": float(loss[4])}
        self.state.history.append(rec)
        return rec

    # ---- epochs ------------------------------------------------------------------
    def fit(self, batch, epochs: int, log: Optional[Callable[[Dict[str, float]], None]] = None,
            max_steps: Optional[int] = None):
        """Epochs over the structures of `batch`, shuffled per epoch, global batches of
        `global_batch` structures (the last partial batch of an epoch is dropped).  Resumes
        mid-epoch after `load`."""
        S = batch.n_struct
        while self.state.epoch < epochs:
            if self._order is None:
                self._order, self._pos = self.rng.permutation(S), 0
            while self._pos + self.global_batch <= S:
                if max_steps is not None and self.state.step >= max_steps:
                    return self.state
                ids = self._order[self._pos:self._pos + self.global_batch].tolist()
                self._pos += self.global_batch
                nxt = None
                if self._pos + self.global_batch <= S and (max_steps is None or self.state.step + 1 < max_steps):
                    nxt = self._order[self._pos:self._pos + self.global_batch].tolist()
                rec = self.train_step(batch, ids, nxt)
                if log:
                    log(rec)
            self._order = None
            self.state.epoch += 1
        return self.state

    # ---- checkpoints -------------------------------------------------------------
    def save(self, path: str):
        meta = {"step": self.state.step, "epoch": self.state.epoch, "lr0": self.lr0,
                "total_steps": self.total_steps, "rng": self.rng.bit_generator.state, "pos": self._pos,
                "order": None if self._order is None else self._order.tolist()}
        np.savez(path, params=self.model.get(0), adam_m=self.model.get(2), adam_v=self.model.get(3),
                 meta=np.frombuffer(json.dumps(meta).encode(), np.uint8))

    def load(self, path: str):
        z = np.load(path)
        self.model.set(0, z["params"])
        self.model.set(2, z["adam_m"])
        self.model.set(3, z["adam_v"])
        meta = json.loads(bytes(z["meta"]).decode())
        self.state.step, self.state.epoch = int(meta["step"]), int(meta["epoch"])
        self.lr0, self.total_steps = float(meta["lr0"]), int(meta["total_steps"])
        self.rng.bit_generator.state = meta["rng"]
        self._order = None if meta["order"] is None else np.asarray(meta["order"], np.int64)
        self._pos = int(meta["pos"])
