"""One training step bracketed by cudaProfilerStart/Stop, for ncu --profile-from-start off.

  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/step.csv python tools/ncu_step.py C2 tf32
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from chg_inputs import init_flat_params, make_config_batch
from paper_2412_20796_b200 import chg

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = {"tf32": 2, "3xtf32": 1, "fp32": 0, "bf16": 3}[sys.argv[2] if len(sys.argv) > 2 else "tf32"]
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


for k in range(3):
    step(k + 1)
ctx.sync()
n0 = ctx.launch_count()
torch.cuda.profiler.start()
step(4)
ctx.sync()
torch.cuda.profiler.stop()
print("launches in the profiled step:", ctx.launch_count() - n0)
