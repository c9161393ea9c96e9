"""Oracle (CPU, fp64) timings on the host cores, SURVEY §8(d) "Oracle timing": seconds per
training step for C1, structures/s for C2 and C3 (forward + backward + Adam on the whole batch),
seconds per forward for C5.  Test infrastructure; writes one JSON object to stdout.

  python tools/oracle_timing.py [--c3-structures 128]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from chg_inputs import init_flat_params, make_config_batch, split_batch  # noqa: E402
from oracle.graph import build_graph_batch  # noqa: E402
from oracle.model import ModelConfig, param_layout, run_forward  # noqa: E402
from oracle.train import LossConfig, adam_step, loss_and_grad  # noqa: E402


def step(b, p, cfg, st):
    g = build_graph_batch(b)
    _, grad, _ = loss_and_grad(g, b, p, cfg, LossConfig())
    st["t"] += 1
    p, st["m"], st["v"] = adam_step(p, st["m"], st["v"], grad, st["t"], 3e-4)
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3-structures", type=int, default=64)
    a = ap.parse_args()
    cfg = ModelConfig()
    p0 = init_flat_params(param_layout(cfg), seed=0).astype(np.float32).astype(np.float64)
    out = {"threads": torch.get_num_threads(), "host_cores": os.cpu_count(), "kind": "oracle (fp64 torch CPU)"}
    for name, n in (("C1", None), ("C2", None), ("C3", a.c3_structures)):
        b = make_config_batch(name, 0) if n is None else make_config_batch(name, 0, n_struct=n)
        st = {"t": 0, "m": np.zeros_like(p0), "v": np.zeros_like(p0)}
        p = step(b, p0, cfg, st)                       # warm-up
        t0 = time.time()
        p = step(b, p, cfg, st)
        dt = time.time() - t0
        out[name] = {"structures": b.n_struct, "atoms": b.n_atoms, "s_per_step": dt, "structures_per_s": b.n_struct / dt}
        print(json.dumps({name: out[name]}), file=sys.stderr, flush=True)
    b5 = make_config_batch("C5")
    t0 = time.time()
    g5 = build_graph_batch(b5)
    t1 = time.time()
    run_forward(g5, b5.species, b5.lattice, p0, cfg)
    t2 = time.time()
    out["C5"] = {"atoms": b5.n_atoms, "graph_s": t1 - t0, "forward_s": t2 - t1, "edges": g5.n_edges, "angles": g5.n_angles}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
