"""Errors of one precision mode against the fp64 oracle (test infrastructure): outputs, loss
terms and every gradient tensor (per-tensor L2 and element-wise, the measures of
tests/test_gpu_parity_ext.py) on the C2 batch, the first C3 batch and the edge-case batch.
Used to state the bars of a mode from measurement.

  python tools/mode_errors.py 3 > gpurun_out/mode_errors_bf16.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from chg_inputs import init_flat_params, make_config_batch  # noqa: E402
from oracle.graph import build_graph_batch  # noqa: E402
from oracle.model import ModelConfig, param_layout  # noqa: E402
from oracle.train import LossConfig, loss_and_grad  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402
from test_gpu_parity import _labels32, _labels64  # noqa: E402
from test_gpu_parity_ext import _edge_batch  # noqa: E402


def main():
    prec = int(sys.argv[1])
    cfg = ModelConfig()
    params = init_flat_params(param_layout(cfg), seed=0, bias_scale=0.1).astype(np.float32).astype(np.float64)
    ctx = chg.Context(0)
    res = {"mode": chg.PRECISION_MODES[prec]}
    cases = {"C2": make_config_batch("C2"), "C3": make_config_batch("C3", 0, n_struct=128), "edge": _edge_batch()}
    for name, b0 in cases.items():
        b = _labels64(b0)
        terms, gref, ref = loss_and_grad(build_graph_batch(b), b, params, cfg, LossConfig())
        mc = chg.default_model_cfg()
        mc.mlp_precision = prec
        m = chg.Model(ctx, mc)
        m.set_params(params.astype(np.float32))
        g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
        out = ctx.forward(m, g, train=True)
        loss = ctx.backward(m, g, _labels32(b))
        eps = np.asarray(ref["energy_per_atom"])
        r = {"epa": float(np.max(np.abs(out["energy_per_atom"] - eps) / np.maximum(np.abs(eps), 1.0))),
             "forces": float(np.max(np.abs(out["forces"] - np.asarray(ref["forces"])))),
             "stress": float(np.max(np.abs(out["stress"] - np.asarray(ref["stress"])))),
             "magmom": float(np.max(np.abs(out["magmom"] - np.asarray(ref["magmom"]))))}
        r["loss_rel"] = {k: float(abs(loss[i] - terms[k]) / max(abs(terms[k]), 1e-6))
                         for i, k in enumerate(["total", "E", "F", "S", "M"])}
        grads, off, tens = m.grads(), 0, []
        for pname, shape, _ in m.layout():
            n = int(np.prod(shape))
            gr, gx = gref[off:off + n], grads[off:off + n].astype(np.float64)
            off += n
            if np.all(gr == 0):
                continue
            l2 = float(np.linalg.norm(gx - gr) / np.linalg.norm(gr))
            el = float(np.max(np.abs(gx - gr) / (np.abs(gr) + 0.01 * np.max(np.abs(gr)))))
            tens.append((l2, el, pname))
        tens.sort(reverse=True)
        r["grad_worst_l2"] = tens[:5]
        r["grad_worst_elem"] = sorted(tens, key=lambda t: -t[1])[:5]
        r["grad_median_l2"] = float(np.median([t[0] for t in tens]))
        res[name] = r
        print(json.dumps({name: {k: r[k] for k in ("epa", "forces", "stress", "magmom")},
                          "worst_l2": tens[0]}), file=sys.stderr, flush=True)
        g.close()
        m.close()
    gem = {}
    for M, K, N in [(1000, 64, 128), (4097, 256, 256), (777, 128, 192)]:
        rng = np.random.default_rng(M + K + N)
        A = rng.normal(size=(M, K)).astype(np.float32)
        W = (rng.normal(size=(K, N)) / np.sqrt(K)).astype(np.float32)
        o = ctx.debug_gemm(0, prec, A, W)
        refm = A.astype(np.float64) @ W.astype(np.float64)
        D = rng.normal(size=(M, N)).astype(np.float32)
        ow = ctx.debug_gemm(1, prec, A, D)
        refw = A.astype(np.float64).T @ D.astype(np.float64)
        gem[f"{M}x{K}x{N}"] = {"row": float(np.linalg.norm(o - refm) / np.linalg.norm(refm)),
                               "wgrad": float(np.linalg.norm(ow - refw) / np.linalg.norm(refw))}
    res["debug_gemm"] = gem
    ctx.close()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
