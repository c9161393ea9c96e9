"""Graph prefetch: a builder context builds the next batch's graph on its
own stream while the training context runs; results must equal the inline-built path bit for
bit (same arrays, same deterministic kernels), and the ownership rules of include/chg.h hold."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from chg_inputs import init_flat_params, make_config_batch  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return 0


def _labels(b):
    return dict(energy_per_atom=b.energy_per_atom.astype(np.float32), forces=b.forces.astype(np.float32),
                stress=b.stress.astype(np.float32), magmom=b.magmom.astype(np.float32), magmom_mask=b.magmom_mask)


def _run(prec, batches, prefetch):
    ctx = chg.Context(0)
    builder = chg.Context(0) if prefetch else None
    cfg = chg.default_model_cfg(); cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    m.set_params(init_flat_params([(n, s) for n, s, _ in m.layout()], seed=0).astype(np.float32))
    losses = []
    gnext = None
    for k, b in enumerate(batches):
        g = gnext if gnext is not None else ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
        ctx.forward(m, g, train=True, host=False)
        gnext = None
        if prefetch and k + 1 < len(batches):
            nb = batches[k + 1]
            gnext = builder.build_graph(nb.atom_ptr, nb.positions, nb.lattice, nb.species)
        losses.append(ctx.backward(m, g, _labels(b), sync_loss=True))
        ctx.step(m, lr=3e-4, step=k + 1)
        if gnext is not None:
            ctx.wait_graph(gnext)
        g.close()
    p = m.params()
    m.close()
    if builder:
        builder.close()
    ctx.close()
    return np.array(losses), p


@pytest.mark.parametrize("prec", [0, 2])
def test_prefetched_graphs_reproduce_inline_training(dev, prec):
    batches = [make_config_batch("C2", seed) for seed in range(4)]
    l_in, p_in = _run(prec, batches, False)
    l_pf, p_pf = _run(prec, batches, True)
    np.testing.assert_array_equal(l_in, l_pf)
    np.testing.assert_array_equal(p_in, p_pf)


def test_graph_user_rules(dev):
    b = make_config_batch("C2", 0)
    a, c, d = chg.Context(0), chg.Context(0), chg.Context(0)
    g = a.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    c.wait_graph(g)                                   # second context: allowed
    with pytest.raises(chg.ChgError):
        d.wait_graph(g)                               # a third context: CHG_ERR_ARG
    g.close()
    for x in (a, c, d):
        x.close()
