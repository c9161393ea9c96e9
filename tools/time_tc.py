"""Timing study of the TC row GEMM (profile tags) under CHG_TC_SKIP settings (run once per setting)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from chg_inputs import init_flat_params, make_config_batch
from paper_2412_20796_b200 import chg
b = make_config_batch("C2")
ctx = chg.Context(0)
cfg = chg.default_model_cfg(); cfg.mlp_precision = 2
m = chg.Model(ctx, cfg)
lay = [(n, s) for n, s, _ in m.layout()]
m.set_params(init_flat_params(lay, seed=0).astype(np.float32))
g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
lab = dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
           stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)
for it in range(3):
    ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False)
ctx.profile(True)
for it in range(5):
    ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False)
rep = ctx.profile_report()
r = rep["rowgemm_tc"]
print(json.dumps({"skip": os.environ.get("CHG_TC_SKIP", "0"), "ms_per_launch": r["ms"] / r["launches"] * 1e3,
                  "tflops": r["flops"] / (r["ms"] / 1e3) / 1e12}))
