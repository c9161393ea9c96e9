"""Per-op device times of one MD step (skin graph, call by call) for the 8-atom Si cell."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from chg_inputs import init_flat_params, make_config_batch  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402
from paper_2412_20796_b200.md import NVE, maxwell_boltzmann  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ctx = chg.Context(0)
cfg = chg.default_model_cfg()
cfg.mlp_precision = prec
m = chg.Model(ctx, cfg)
m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
b = make_config_batch("C1")
mass = np.full(b.n_atoms, 28.0855)
md = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, maxwell_boltzmann(mass, 300.0, 0), 0.5, skin=0.5)
md.step(10)
print("counts", md.graph.counts())
ctx.profile(True)
l0 = ctx.launch_count()
md.step(10)
rep = ctx.profile_report()
ctx.profile(False)
print("launches per step", (ctx.launch_count() - l0) / 10)
tot = sum(v["ms"] for v in rep.values()) / 10
print("sum of op times per step (ms)", round(tot, 4))
for t, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])[:25]:
    print(f"{t:16s} {v['ms'] / 10 * 1e3:8.1f} us/step {v['launches'] // 10:4d} launches {v['ms'] / v['launches'] * 1e3:7.1f} us/launch")
