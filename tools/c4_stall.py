"""Diagnose per-step stalls at C4 (one GPU): host time per phase and device time per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from chg_inputs import init_flat_params, make_config_batch  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402

ctx = chg.Context(0)
cfg = chg.default_model_cfg()
cfg.mlp_precision = 1
m = chg.Model(ctx, cfg)
m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
bs = [make_config_batch("C4", k, n_struct=128) for k in range(4)]
dev = []
for b in bs:
    lab = dict(energy_per_atom=torch.as_tensor(b.energy_per_atom.astype(np.float32), device="cuda"),
               forces=torch.as_tensor(b.forces.astype(np.float32), device="cuda"),
               stress=torch.as_tensor(b.stress.astype(np.float32), device="cuda"),
               magmom=torch.as_tensor(b.magmom.astype(np.float32), device="cuda"),
               magmom_mask=torch.as_tensor(b.magmom_mask.astype(np.uint8), device="cuda"))
    dev.append((torch.as_tensor(b.positions, device="cuda"), torch.as_tensor(b.lattice, device="cuda"),
                torch.as_tensor(b.species, device="cuda"), lab))
torch.cuda.synchronize()
for it in range(24):
    k = it % 4
    b = bs[k]
    pos, lat, sp, lab = dev[k]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    tb0 = time.perf_counter()
    g = ctx.build_graph(b.atom_ptr, pos, lat, sp)
    t1 = time.perf_counter()
    g_counts = g.counts()
    ctx.forward(m, g, train=True, host=False)
    t2 = time.perf_counter()
    ctx.backward(m, g, lab, sync_loss=False)
    t3 = time.perf_counter()
    ctx.step(m, 3e-4, it + 1, defer_check=True)
    g.close()
    e1.record()
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    free, total = torch.cuda.mem_get_info()
    print(f"it {it} batch {k} counts {g_counts} | host build {1e3*(t1-t0):7.1f} fwd {1e3*(t2-t1):7.1f} "
          f"bwd {1e3*(t3-t2):7.1f} step {1e3*(t4-t3):7.1f} sync {1e3*(t5-t4):7.1f} | free {free/2**30:.1f} GiB of {total/2**30:.1f}", flush=True)
