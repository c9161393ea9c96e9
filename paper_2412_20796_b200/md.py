"""MD inference loop (the paper's Table II regime).

Velocity-Verlet NVE on the GPU.  State lives in device tensors (PyTorch only allocates them);
every step runs in libchg: chg_md_verlet (kick + drift) -> chg_build_graph from the device
positions (cell lists for large cells) -> chg_forward_conservative (F = -dE/dr, on-device
outputs) -> chg_md_verlet (kick).  Units: eV, Å, amu, fs.  Positions are not wrapped into the
cell (the builder accepts any Cartesian positions).

skin > 0: a fixed-topology Verlet list (chg_build_graph_skin: lists with r + skin, bases zero
beyond r) whose geometry is refreshed every step (chg_graph_refresh), so the step has constant
sizes; captured = True records it as one CUDA graph (chg_md_capture) and replays it
(chg_md_run) in chunks of `check_every` steps.  After each chunk the moved-atom flag is read
(set once an atom moved more than skin / 2 since the build) and the lists are rebuilt and the
step re-captured.  The energies and forces equal those of rebuilt-every-step lists while every
atom stays within skin / 2 of its build position; the flag is read every `check_every` steps,
so an atom would have to move faster than (skin / 2) / (check_every · dt) — 0.05 Å/fs (5 km/s)
at the defaults skin = 1 Å, 10 steps, 1 fs — to cross it between two checks.
"""
from __future__ import annotations

import numpy as np

from . import chg

EV_PER_AMU_A2_FS2 = 103.6426965     # 1 amu·Å²/fs² in eV (kinetic energy, monitoring only)
KB_EV = 8.617333262e-5               # Boltzmann constant, eV/K


class NVE:
    def __init__(self, ctx: chg.Context, model: chg.Model, atom_ptr, positions, lattice, species, masses,
                 velocities=None, dt_fs: float = 1.0, r_atom: float = 5.0, r_bond: float = 3.0,
                 skin: float = 0.0, captured: bool = False, check_every: int = 10):
        import torch
        dev = torch.device("cuda", ctx.device)
        self.ctx, self.model, self.dt = ctx, model, float(dt_fs)
        self.r_atom, self.r_bond = r_atom, r_bond
        if captured and skin <= 0:
            raise ValueError("a captured MD step needs a skin graph (skin > 0)")
        self.skin, self.captured, self.check_every = float(skin), bool(captured), max(1, int(check_every))
        self.graph, self.exec, self.rebuilds = None, None, 0
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ap = np.ascontiguousarray(np.asarray(atom_ptr, np.int64))
        n, S = int(self.ap[-1]), self.ap.shape[0] - 1
        f64 = dict(dtype=torch.float64, device=dev)
        self.pos = torch.as_tensor(np.asarray(positions, np.float64).reshape(n, 3), **f64).contiguous()
        self.lat = torch.as_tensor(np.asarray(lattice, np.float64).reshape(S, 3, 3), **f64).contiguous()
        self.spec = torch.as_tensor(np.asarray(species, np.int32), device=dev).contiguous()
        self.mass = np.asarray(masses, np.float64).reshape(n)
        self.inv_m = torch.as_tensor(1.0 / self.mass, **f64).contiguous()
        v = np.zeros((n, 3)) if velocities is None else np.asarray(velocities, np.float64).reshape(n, 3)
        self.vel = torch.as_tensor(v, **f64).contiguous()
        f32 = dict(dtype=torch.float32, device=dev)
        self.out = {"energy": torch.zeros(S, **f32), "energy_per_atom": torch.zeros(S, **f32),
                    "forces": torch.zeros(n, 3, **f32), "stress": torch.zeros(S, 3, 3, **f32),
                    "magmom": torch.zeros(n, **f32)}
        self.steps = 0
        torch.cuda.current_stream(dev).synchronize()   # state tensors written on torch's stream
        if self.skin > 0:
            self._rebuild()
        else:
            self._forces()
        self.ctx.sync()

    def _forces(self):
        if self.skin > 0:                              # fixed topology: refresh the geometry only
            self.ctx.refresh_graph(self.graph, self.pos, self.flag)
            self.ctx.forward_conservative(self.model, self.graph, out=self.out)
            return
        g = self.ctx.build_graph(self.ap, self.pos, self.lat, self.spec, self.r_atom, self.r_bond)
        self.ctx.forward_conservative(self.model, g, out=self.out)
        g.close()

    def _rebuild(self):
        """New skin lists at the current positions (+ forces there, + a new capture)."""
        if self.exec is not None:
            self.exec.close()
            self.exec = None
        if self.graph is not None:
            self.graph.close()
        self.graph = self.ctx.build_graph(self.ap, self.pos, self.lat, self.spec, self.r_atom, self.r_bond,
                                          skin=self.skin)
        self.flag.zero_()
        import torch
        torch.cuda.current_stream(self.flag.device).synchronize()   # zeroed before the ctx stream reads it
        if self.captured:                              # the capture's warm-up pass computes the forces
            self.exec = self.ctx.md_capture(self.model, self.graph, self.pos, self.vel, self.inv_m, self.dt,
                                            self.out, self.flag)
        else:
            self.ctx.forward_conservative(self.model, self.graph, out=self.out)
        self.rebuilds += 1

    def step(self, n: int = 1):
        """n velocity-Verlet steps.  Returns after the work on the ctx stream has finished, so
        pos / vel / out may be read or edited on any stream."""
        done = 0
        while done < n:
            k = min(self.check_every, n - done) if self.skin > 0 else n - done
            if self.captured:
                self.exec.run(k)
            else:
                for _ in range(k):
                    self.ctx.md_verlet(self.pos, self.vel, self.out["forces"], self.inv_m, self.dt, drift=True)
                    self._forces()
                    self.ctx.md_verlet(self.pos, self.vel, self.out["forces"], self.inv_m, self.dt, drift=False)
            done += k
            self.steps += k
            if self.skin > 0:
                self.ctx.sync()
                if int(self.flag.item()):              # an atom left its skin / 2 sphere: new lists
                    self._rebuild()
        self.ctx.sync()

    def close(self):
        if self.exec is not None:
            self.exec.close()
            self.exec = None
        if self.graph is not None:
            self.graph.close()
            self.graph = None

    # ---- observation (host copies; wait for the ctx stream first) -------------------
    def potential_energy(self) -> np.ndarray:
        self.ctx.sync()
        return self.out["energy"].double().cpu().numpy()

    def kinetic_energy(self) -> np.ndarray:
        self.ctx.sync()
        v = self.vel.cpu().numpy()
        ke = 0.5 * self.mass[:, None] * v * v * EV_PER_AMU_A2_FS2
        return np.add.reduceat(ke.sum(1), self.ap[:-1]) if len(self.ap) > 1 else np.zeros(0)

    def total_energy(self) -> np.ndarray:
        return self.potential_energy() + self.kinetic_energy()


def maxwell_boltzmann(masses, temperature_k: float, seed: int = 0) -> np.ndarray:
    """Seeded Maxwell-Boltzmann velocities (Å/fs) with zero total momentum."""
    m = np.asarray(masses, np.float64)
    rng = np.random.default_rng(seed)
    sigma = np.sqrt(KB_EV * temperature_k / (m * EV_PER_AMU_A2_FS2))
    v = rng.normal(size=(m.shape[0], 3)) * sigma[:, None]
    v -= (m[:, None] * v).sum(0) / m.sum()
    return v
