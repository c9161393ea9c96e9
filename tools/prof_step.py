"""Per-op device-time breakdown of one training step (profile tags)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from chg_inputs import init_flat_params, make_config_batch
from paper_2412_20796_b200 import chg
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 2
b = make_config_batch(cfgname)
ctx = chg.Context(0)
cfg = chg.default_model_cfg(); cfg.mlp_precision = prec
m = chg.Model(ctx, cfg)
m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
lab = dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
           stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)
def step(k):
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False); ctx.step(m, 3e-4, k)
    g.close()
for k in range(3): step(k + 1)
ctx.profile(True)
for k in range(5): step(k + 4)
rep = ctx.profile_report()
ctx.profile(False)                 # wall-clock timing below runs the concurrent schedule
tot = sum(v["ms"] for v in rep.values())
print(cfgname, "prec", prec, "sum of op times per step (ms):", round(tot / 5, 3))
for t, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{t:14s} {v['ms']/5:8.3f} ms/step  {v['launches']//5:4d} launches  {v['ms']/v['launches']*1e3:8.1f} us/launch  "
          f"{(v['flops']/(v['ms']/1e3)/1e12) if v['flops'] else 0:7.1f} TF/s  {(v['bytes']/(v['ms']/1e3)/1e9):8.1f} GB/s")
import time
g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False); ctx.sync()
ts = []
for k in range(5):
    t0 = time.perf_counter()
    ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False)
    t1 = time.perf_counter()
    ctx.sync()
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t0))
print("host enqueue fwd+bwd (ms):", [round(a * 1e3, 2) for a, _ in ts], " enqueue+sync (ms):", [round(b_ * 1e3, 2) for _, b_ in ts])
n0 = ctx.launch_count(); ctx.forward(m, g, train=True, host=False); ctx.backward(m, g, lab, sync_loss=False); ctx.sync()
print("launches fwd+bwd:", ctx.launch_count() - n0)
