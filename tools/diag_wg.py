"""Diagnostic: GatedMLP weight gradients, TF32 tensor-core path vs fp32 path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from chg_inputs import init_flat_params, si_diamond, make_config_batch
from paper_2412_20796_b200 import chg
b = si_diamond(jitter=0.05, seed=7) if len(sys.argv) < 2 else make_config_batch(sys.argv[1])
lab = dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
           stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)
ctx = chg.Context(0)
gr = {}
for prec in (0, 2):
    cfg = chg.default_model_cfg(); cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    lay = m.layout()
    m.set_params(init_flat_params([(n, s) for n, s, _ in lay], seed=0, bias_scale=0.1).astype(np.float32))
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    ctx.forward(m, g, train=True, host=False)
    ctx.backward(m, g, lab)
    gr[prec] = m.grads()
for n, s, o in lay:
    if not any(n.startswith(p) for p in ("atom0.core", "atom0.gate", "bond0.core", "bond0.gate", "angle0.core")):
        continue
    k = int(np.prod(s))
    a, t = gr[0][o:o + k].reshape(s), gr[2][o:o + k].reshape(s)
    print(n, s, "|fp32|", np.linalg.norm(a), "|tf32|", np.linalg.norm(t), "rel", np.linalg.norm(a - t) / max(np.linalg.norm(a), 1e-30))
    if n == "atom0.core.W1":
        print(" fp32[0:3,0:4]", a[0:3, 0:4]); print(" tf32[0:3,0:4]", t[0:3, 0:4])
        print(" ratio stats", np.nanmedian(t / a))
