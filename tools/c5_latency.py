"""C5 (one 4,096-atom LiFePO4-like cell) forward latency: graph build + forward (inference path)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from chg_inputs import init_flat_params, make_config_batch
from paper_2412_20796_b200 import chg
b = make_config_batch("C5")
ctx = chg.Context(0)
cfg = chg.default_model_cfg(); cfg.mlp_precision = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = chg.Model(ctx, cfg)
m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
pos = torch.as_tensor(b.positions, device="cuda"); lat = torch.as_tensor(b.lattice, device="cuda")
sp = torch.as_tensor(b.species, device="cuda")
for _ in range(3):
    g = ctx.build_graph(b.atom_ptr, pos, lat, sp); ctx.forward(m, g, train=False, host=False); g.close()
ctx.sync()
tb, tf = [], []
for _ in range(10):
    t0 = time.perf_counter(); g = ctx.build_graph(b.atom_ptr, pos, lat, sp); ctx.sync(); t1 = time.perf_counter()
    ctx.forward(m, g, train=False, host=False); ctx.sync(); t2 = time.perf_counter()
    tb.append(t1 - t0); tf.append(t2 - t1); c = g.counts(); g.close()
print("C5 N,E,B,A", c, "graph build ms median", round(1e3 * np.median(tb), 3), "forward ms median", round(1e3 * np.median(tf), 3))
ctx.profile(True)
g = ctx.build_graph(b.atom_ptr, pos, lat, sp); ctx.forward(m, g, train=False, host=False); ctx.sync()
rep = ctx.profile_report()
for t, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])[:8]:
    print(f"  {t:14s} {v['ms']:.3f} ms")
