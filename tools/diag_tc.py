"""Diagnostic: compare TF32 tensor-core GEMM outputs with the fp32 path, row/col-wise."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from chg_inputs import init_flat_params, si_diamond, make_config_batch
from paper_2412_20796_b200 import chg

b = si_diamond(jitter=0.05, seed=7) if len(sys.argv) < 2 else make_config_batch(sys.argv[1])
ctx = chg.Context(0)
res = {}
for prec in (0, 2):
    cfg = chg.default_model_cfg(); cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    lay = [(n, s) for n, s, _ in m.layout()]
    m.set_params(init_flat_params(lay, seed=0, bias_scale=0.1).astype(np.float32))
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    ctx.forward(m, g, train=True)
    res[prec] = {k: ctx.debug(k) for k in ["ac_z1_0", "ac_y_0", "v1", "bc_z1_0", "bc_yb_0", "bc_ya_0"]}
for k in res[0]:
    a, t = res[0][k], res[2][k]
    d = np.abs(a - t)
    rel = np.linalg.norm(a - t) / np.linalg.norm(a)
    rowerr = d.max(1)
    colerr = d.max(0)
    bad_rows = np.nonzero(rowerr > 1e-2 * np.abs(a).max())[0]
    bad_cols = np.nonzero(colerr > 1e-2 * np.abs(a).max())[0]
    print(k, a.shape, 'rel', rel, 'nbad rows', len(bad_rows), bad_rows[:20], 'nbad cols', len(bad_cols), bad_cols[:40])
