"""MD inference loop (the paper's Table II regime).

Velocity-Verlet NVE on the GPU.  State lives in device tensors (PyTorch only allocates them);
every step runs in libchg: chg_md_verlet (kick + drift) -> chg_build_graph from the device
positions (cell lists for large cells) -> chg_forward_conservative (F = -dE/dr, on-device
outputs) -> chg_md_verlet (kick).  Units: eV, Å, amu, fs.  Positions are not wrapped into the
cell (the builder accepts any Cartesian positions).
"""
from __future__ import annotations

import numpy as np

from . import chg

EV_PER_AMU_A2_FS2 = 103.6426965     # 1 amu·Å²/fs² in eV (kinetic energy, monitoring only)
KB_EV = 8.617333262e-5               # Boltzmann constant, eV/K


class NVE:
    def __init__(self, ctx: chg.Context, model: chg.Model, atom_ptr, positions, lattice, species, masses,
                 velocities=None, dt_fs: float = 1.0, r_atom: float = 5.0, r_bond: float = 3.0):
        import torch
        dev = torch.device("cuda", ctx.device)
        self.ctx, self.model, self.dt = ctx, model, float(dt_fs)
        self.r_atom, self.r_bond = r_atom, r_bond
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
        self._forces()
        self.ctx.sync()

    def _forces(self):
        g = self.ctx.build_graph(self.ap, self.pos, self.lat, self.spec, self.r_atom, self.r_bond)
        self.ctx.forward_conservative(self.model, g, out=self.out)
        g.close()

    def step(self, n: int = 1):
        """n velocity-Verlet steps (graph rebuilt every step).  Returns after the work on the
        ctx stream has finished, so pos / vel / out may be read or edited on any stream."""
        for _ in range(n):
            self.ctx.md_verlet(self.pos, self.vel, self.out["forces"], self.inv_m, self.dt, drift=True)
            self._forces()
            self.ctx.md_verlet(self.pos, self.vel, self.out["forces"], self.inv_m, self.dt, drift=False)
            self.steps += 1
        self.ctx.sync()

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
