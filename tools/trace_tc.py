import sys, os
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
ctx.forward(m, g, train=True, host=False)
ctx.sync()
