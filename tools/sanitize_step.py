"""One small training step per precision mode, for compute-sanitizer.

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_step.py
Runs build_graph + forward + backward + step (+ a captured replay) on a 3-structure C2 subset
in fp32 (CUDA cores), 3xTF32 and TF32 (tcgen05: TMA, mbarrier, TMEM paths) and the
conservative-force pass; prints one line per mode.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from chg_inputs import init_flat_params, make_config_batch  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402

b = make_config_batch("C2", 0, n_struct=3)
lab = dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
           stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)
ctx = chg.Context(0)
for prec in sorted(chg.PRECISION_MODES):
    cfg = chg.default_model_cfg()
    cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0, bias_scale=0.1).astype(np.float32))
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    out = ctx.forward(m, g, train=True)
    loss = ctx.backward(m, g, lab)
    ctx.step(m, lr=3e-4, step=1)
    cons = ctx.forward_conservative(m, g)
    ctx.sync()
    print(f"{chg.PRECISION_MODES[prec]}: E/atom {out['energy_per_atom'][0]:.6f} loss {loss[0]:.6f} "
          f"|F_cons| {np.abs(cons['forces']).max():.4f}", flush=True)
    g.close()
    m.close()
ctx.close()
print("sanitize step ok")
