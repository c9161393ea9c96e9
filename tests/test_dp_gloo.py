"""Data-parallel host logic on CPU with torch.distributed gloo, world_size 2.

Each rank takes its structures from the load-balance sampler (chg_balance,
P:330-331 — the C-ABI host routine, identical on every rank), computes the fp64
oracle gradient of its shard with GLOBAL loss normalisers (reading Q23), and the
gradients are summed with an allreduce.  The sum must equal the
single-process full-batch gradient (SPEC S:524 data-parallel equivalence)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from chg_inputs import init_flat_params, mptrj_like_batch, split_batch
    from oracle.graph import build_graph_batch
    from oracle.model import ModelConfig, param_layout
    from oracle.train import LossConfig, loss_and_grad
    from paper_2412_20796_b200 import chg
    cfg = ModelConfig(d=64)
    b = mptrj_like_batch(6, seed=501)
    p = init_flat_params(param_layout(cfg), seed=1, bias_scale=0.1)
    g_all = build_graph_batch(b)
    loads = g_all.counts[:, 0] + g_all.counts[:, 1] + g_all.counts[:, 3]
    rank_of = chg.balance(loads, world)
    mine = np.nonzero(rank_of == rank)[0].tolist()
    lc = LossConfig(n_struct_global=b.n_struct, n_atoms_global=b.n_atoms,
                    n_magmom_global=int(b.magmom_mask.sum()))
    sb = split_batch(b, mine)
    terms, grad, _ = loss_and_grad(build_graph_batch(sb), sb, p, cfg, lc)
    t = torch.as_tensor(np.concatenate([grad, [terms["total"]]]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(os.path.join(out_dir, "dp_grad.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.slow
def test_dp_allreduce_equals_full_batch(tmp_path):
    pytest.importorskip("torch.distributed")
    from paper_2412_20796_b200 import chg
    try:
        chg.load()
    except ImportError:
        import __graft_entry__
        __graft_entry__.build()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    dp = np.load(tmp_path / "dp_grad.npy")
    from chg_inputs import init_flat_params, mptrj_like_batch
    from oracle.graph import build_graph_batch
    from oracle.model import ModelConfig, param_layout
    from oracle.train import LossConfig, loss_and_grad
    cfg = ModelConfig(d=64)
    b = mptrj_like_batch(6, seed=501)
    p = init_flat_params(param_layout(cfg), seed=1, bias_scale=0.1)
    terms, grad, _ = loss_and_grad(build_graph_batch(b), b, p, cfg, LossConfig())
    assert dp[-1] == pytest.approx(terms["total"], rel=1e-12)
    np.testing.assert_allclose(dp[:-1], grad, rtol=1e-9, atol=1e-14)
