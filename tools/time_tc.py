"""Timing study of the TC row GEMM (sum over its call sites) under CHG_TC_SKIP debug settings.

  CHG_TC_SKIP=<bits> python tools/time_tc.py [C2|C3]
  bits: 1 no epilogue stores, 2 no gather traffic, 4 no weight traffic, 8 no MMA, 16 no convert
"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from chg_inputs import init_flat_params, make_config_batch
from paper_2412_20796_b200 import chg
TAGS = {"ac_f1", "ac_f2", "bc_f1", "bc_f2", "ac_dZ", "ac_dX", "bc_dZ", "bc_dX"}
os.environ.setdefault("CHG_SERIAL", "1")
b = make_config_batch(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = chg.Context(0)
cfg = chg.default_model_cfg(); cfg.mlp_precision = int(os.environ.get("CHG_PREC", "2"))
m = chg.Model(ctx, cfg)
m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
lab = dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
           stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)
for it in range(3):
    ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False)
ctx.profile(True)
for it in range(5):
    ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False)
rep = ctx.profile_report()
out = {"skip": os.environ.get("CHG_TC_SKIP", "0")}
for t in sorted(TAGS):
    if t in rep:
        out[t] = round(rep[t]["ms"] / rep[t]["launches"] * 1e3, 1)
out["total_ms_per_step"] = round(sum(rep[t]["ms"] for t in TAGS if t in rep) / 5, 3)
print(json.dumps(out))
