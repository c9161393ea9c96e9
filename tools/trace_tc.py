"""One forward+backward with the row-GEMM trace on (CHG_TC_SKIP=32): per launch, CTA 0's timeline."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from chg_inputs import init_flat_params, make_config_batch
from paper_2412_20796_b200 import chg
os.environ.setdefault("CHG_SERIAL", "1")
b = make_config_batch(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = chg.Context(0)
cfg = chg.default_model_cfg(); cfg.mlp_precision = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m = chg.Model(ctx, cfg)
m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
lab = dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
           stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)
print(g.counts())
ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False)
import torch; torch.cuda.synchronize()
