"""Graph-build timing for a named config (device-resident inputs, CUDA events), with counts."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from chg_inputs import make_config_batch
from paper_2412_20796_b200 import chg
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
b = make_config_batch(cfgname)
ctx = chg.Context(0)
pos = torch.as_tensor(b.positions, device="cuda"); lat = torch.as_tensor(b.lattice, device="cuda")
spec = torch.as_tensor(b.species, device="cuda")
ts = []
for k in range(reps):
    ctx.sync(); t0 = time.perf_counter()
    g = ctx.build_graph(b.atom_ptr, pos, lat, spec)
    ctx.sync(); ts.append(time.perf_counter() - t0)
    if k < reps - 1:
        g.close()
ps = g.per_struct()
n = np.diff(b.atom_ptr)
print(cfgname, "S", b.n_struct, "N", b.n_atoms, "E/B/A", ps[:, 1].sum(), ps[:, 2].sum(), ps[:, 3].sum(),
      "max atoms", n.max(), "build ms", [round(t * 1e3, 2) for t in ts])
o = np.argsort(-ps[:, 3])[:5]
print("largest angle counts (struct, atoms, edges, angles):", [(int(i), int(n[i]), int(ps[i, 1]), int(ps[i, 3])) for i in o])
