"""MD step timings (NEXT-2, Table II regime P:446-465): device ms per velocity-Verlet step for the
8-atom Si cell (C1) and the 4,096-atom C5 cell — graph rebuilt every step, skin graph refreshed
every step (call by call), and the captured step (chg_md_run).  Writes one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from chg_inputs import init_flat_params, make_config_batch  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402
from paper_2412_20796_b200.md import NVE, maxwell_boltzmann  # noqa: E402


def main():
    prec = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    ctx = chg.Context(0)
    cfg = chg.default_model_cfg()
    cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
    out = {"mlp_precision": chg.PRECISION_MODES[prec], "skin": float(os.environ.get("MD_SKIN", "0.5"))}
    for name, b, mass_v in (("C1_Si8", make_config_batch("C1"), 28.0855), ("C5_4096", make_config_batch("C5"), 30.0)):
        mass = np.full(b.n_atoms, mass_v)
        res = {}
        skin = float(os.environ.get("MD_SKIN", "0.5"))
        for mode, kw in (("rebuild_every_step", {}), ("skin_refresh", dict(skin=skin)),
                         ("captured", dict(skin=skin, captured=True))):
            md = NVE(ctx, m, b.atom_ptr, b.positions, b.lattice, b.species, mass, maxwell_boltzmann(mass, 300.0, 0),
                     dt_fs=0.5, **kw)
            md.step(20)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                md.step(20)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 20)
            res[mode] = {"ms_per_step_median": float(np.median(ts)), "rebuilds": md.rebuilds}
            md.close()
        out[name] = res
        print(json.dumps({name: res}), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
