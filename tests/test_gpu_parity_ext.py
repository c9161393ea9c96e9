"""GPU parity, widened, every precision mode against the fp64 oracle.

* Full-C3 backward: the whole first C3 batch (128 MPtrj-shaped structures, bench's per-GPU
  work of the N > 1 runs) through forward + backward on the GPU, loss terms and all 151
  gradient tensors against the oracle of the same batch.
* Sampled C4 gradients at full size: the whole C4 batch (128 skewed oxides) runs on the GPU;
  every structure except the sampled one gets labels equal to its own GPU prediction, so its
  Huber residuals and seeds are exactly 0 and the full-batch gradient is the sampled
  structure's alone — computed inside the full-size launches (large-M GEMM plans).  The
  oracle runs that structure alone with the same global normalisers (reading Q23).
* Edge cases through forward + backward: an isolated atom (no edges), a dimer at 2 A (bond
  edges, no angles), a 1-atom simple-cubic cell (self-image neighbours; theta = pi at the
  bond cutoff, the clamp), mixed into C2 structures, at cutoffs 5/3 and 6/3 A.
* Gradient bars: per tensor ||dg|| / ||g|| (NS: 1e-4 strict, 2e-3 TF32) AND element-wise
  e_i = |dg_i| / (|g_i| + 0.01 max|g|) — a wrong row of one species or one channel gives
  e ~ 1 and cannot hide in a large tensor.  Element-wise bars (measured worst in brackets):
  fp32 CUDA cores 5e-4 [1.2e-4, C4]; 3xTF32 5e-3 [1.2e-3, C4 bond W1: the tensor core's
  accumulation is not IEEE round-to-nearest, ~10x the SIMT error, while its per-tensor error
  2.9e-5 meets the NS 1e-4]; TF32 0.15 [0.061, C4: single elements that are sums of
  cancelling TF32 products]; BF16 1.0 [0.59, C2] with per-tensor 1.5e-2 [7.3e-3]: BF16 does
  NOT meet the NS 2e-3 per-tensor bar on the angle-update tensors (reported), and
  its element-wise bar is no localisation check — the fp32 / 3xTF32 / TF32 modes carry that.
* Output bars (NS): E/atom 1e-5 max(|eps|, 1 eV), F 1e-4 eV/A, sigma 1e-4 GPa in
  every mode; magmom 1e-5 muB (fp32 strict, 3xTF32), 2e-4 muB (TF32: m is a linear map of v^4,
  whose TF32 feature error is ~1e-5 relative; measured 5.9e-5, profiles/r01_tf32_parity_errors.json),
  2e-3 muB (BF16, measured 5.9e-4).
* Labels: a NULL label array skips its task (chg_labels), all NULL is CHG_ERR_ARG.
"""
import json
import os

import numpy as np
import pytest

from chg_inputs import Batch, concat_batches, dimer, init_flat_params, make_config_batch, simple_cubic, split_batch

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle.graph import build_graph_batch  # noqa: E402
from oracle.model import ModelConfig, param_layout, run_forward  # noqa: E402
from oracle.train import LossConfig, loss_and_grad  # noqa: E402
from paper_2412_20796_b200 import chg  # noqa: E402

from test_gpu_parity import _labels32, _labels64  # noqa: E402

CFG = ModelConfig()
# mlp_precision -> bars: per-tensor gradient (NS), element-wise gradient, magmom
MODES = {0: dict(name="fp32", grad=1e-4, elem=5e-4, mag=1e-5),
         2: dict(name="tf32", grad=2e-3, elem=0.15, mag=2e-4)}
if 1 in chg.PRECISION_MODES:
    MODES[1] = dict(name="3xtf32", grad=1e-4, elem=5e-3, mag=1e-5)
if 3 in chg.PRECISION_MODES:
    # BF16 operands (8-bit significand): the NS 2e-3 per-tensor bar fails on the angle-update
    # GatedMLP tensors (measured worst 7.3e-3, median 1.7e-3: profiles/r02_mode_errors_bf16.json);
    # the bars below are the measured worst x ~2, stated in DESIGN §6; loss terms 1e-3 relative
    MODES[3] = dict(name="bf16", grad=1.5e-2, elem=1.0, mag=2e-3, loss=1e-3)
REPORT = {}
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(scope="module")
def ctx():
    c = chg.Context(0)
    yield c
    c.close()
    if os.path.isdir(OUT):
        with open(os.path.join(OUT, "parity_ext_errors.json"), "w") as f:
            json.dump(REPORT, f, indent=1)


@pytest.fixture(scope="module")
def params():
    return init_flat_params(param_layout(CFG), seed=0, bias_scale=0.1).astype(np.float32).astype(np.float64)


def _model(ctx, params, prec):
    cfg = chg.default_model_cfg()
    cfg.mlp_precision = prec
    m = chg.Model(ctx, cfg)
    m.set_params(params.astype(np.float32))
    return m


def _check_grads(g, gref, bars, key):
    rep, off, bad = {}, 0, {}
    worst_l2, worst_el = 0.0, 0.0
    for name, shape in param_layout(CFG):
        n = int(np.prod(shape))
        gr, gx = gref[off:off + n], g[off:off + n].astype(np.float64)
        off += n
        if np.all(gr == 0):
            if not np.all(gx == 0):
                bad[name] = "nonzero where the oracle is exactly zero"
            continue
        l2 = float(np.linalg.norm(gx - gr) / np.linalg.norm(gr))
        el = float(np.max(np.abs(gx - gr) / (np.abs(gr) + 0.01 * np.max(np.abs(gr)))))
        worst_l2, worst_el = max(worst_l2, l2), max(worst_el, el)
        if l2 > bars["grad"] or el > bars["elem"]:
            bad[name] = (l2, el)
    rep["worst_l2"], rep["worst_elementwise"] = worst_l2, worst_el
    REPORT[key] = rep
    assert not bad, bad


def _check_outputs(out, ref, bars, sl=None):
    """sl: (structures, atoms) index arrays of the GPU outputs to compare, default all."""
    s_ix, a_ix = sl if sl is not None else (slice(None), slice(None))
    eps = ref["energy_per_atom"].detach().numpy()
    de = np.abs(out["energy_per_atom"][s_ix] - eps) / np.maximum(np.abs(eps), 1.0)
    df = np.max(np.abs(out["forces"][a_ix] - ref["forces"].detach().numpy()), initial=0.0)
    ds = np.max(np.abs(out["stress"][s_ix] - ref["stress"].detach().numpy()), initial=0.0)
    dm = np.max(np.abs(out["magmom"][a_ix] - ref["magmom"].detach().numpy()), initial=0.0)
    errs = dict(epa=float(np.max(de, initial=0.0)), forces=float(df), stress=float(ds), magmom=float(dm))
    assert errs["epa"] <= 1e-5 and errs["forces"] <= 1e-4 and errs["stress"] <= 1e-4, errs
    assert errs["magmom"] <= bars["mag"], errs
    return errs


# ---------------------------------------------------------------------------------------
# full-C3 backward parity
# ---------------------------------------------------------------------------------------
_C3 = {}


def _c3_ref(params):
    if "ref" not in _C3:
        b = _labels64(make_config_batch("C3", 0, n_struct=128))
        og = build_graph_batch(b)
        terms, gref, out = loss_and_grad(og, b, params, CFG, LossConfig())
        _C3.update(b=b, terms=terms, gref=gref, out=out)
    return _C3


@pytest.mark.parametrize("prec", sorted(MODES))
def test_c3_full_backward(ctx, params, prec):
    R = _c3_ref(params)
    b, bars = R["b"], MODES[prec]
    m = _model(ctx, params, prec)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    out = ctx.forward(m, g, train=True)
    loss = ctx.backward(m, g, _labels32(b))
    errs = _check_outputs(out, {k: torch.as_tensor(v) for k, v in R["out"].items()}, bars)
    REPORT[f"c3_outputs_{bars['name']}"] = errs
    for k, key in enumerate(["total", "E", "F", "S", "M"]):
        assert abs(loss[k] - R["terms"][key]) <= bars.get("loss", 1e-5) * max(abs(R["terms"][key]), 1e-6), key
    _check_grads(m.grads(), R["gref"], bars, f"c3_grads_{bars['name']}")
    g.close(); m.close()


# ---------------------------------------------------------------------------------------
# sampled C4 gradients at full size (zero-residual masking of the other structures)
# ---------------------------------------------------------------------------------------
_C4 = {}


def _c4():
    if "b" not in _C4:
        _C4["b"] = _labels64(make_config_batch("C4", 0, n_struct=128))
    return _C4["b"]


def _c4_samples(b):
    n = np.diff(b.atom_ptr)
    o = np.argsort(n, kind="stable")
    return [int(o[len(o) // 2]), int(o[int(len(o) * 0.9)]), int(o[-1])]


@pytest.mark.parametrize("prec", sorted(MODES))
def test_c4_sampled_gradients_fullsize(ctx, params, prec):
    b, bars = _c4(), MODES[prec]
    m = _model(ctx, params, prec)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    n_mag = int(b.magmom_mask.sum())
    gl = dict(n_struct_global=b.n_struct, n_atoms_global=b.n_atoms, n_magmom_global=n_mag)
    lc = LossConfig(n_struct_global=b.n_struct, n_atoms_global=b.n_atoms, n_magmom_global=n_mag)
    for s in _c4_samples(b):
        pred = ctx.forward(m, g, train=True)
        a0, a1 = int(b.atom_ptr[s]), int(b.atom_ptr[s + 1])
        lab = dict(energy_per_atom=pred["energy_per_atom"].copy(), forces=pred["forces"].copy(),
                   stress=pred["stress"].copy(), magmom=pred["magmom"].copy(),
                   magmom_mask=b.magmom_mask.astype(np.uint8))
        own = _labels32(b)
        lab["energy_per_atom"][s] = own["energy_per_atom"][s]
        lab["forces"][a0:a1] = own["forces"][a0:a1]
        lab["stress"][s] = own["stress"][s]
        lab["magmom"][a0:a1] = own["magmom"][a0:a1]
        m.set(1, np.zeros(m.P, np.float32))
        ctx.backward(m, g, lab, **gl)
        sb = split_batch(b, [s])
        terms, gref, out = loss_and_grad(build_graph_batch(sb), sb, params, CFG, lc)
        errs = _check_outputs(pred, {k: torch.as_tensor(v) for k, v in out.items()}, bars,
                              sl=(slice(s, s + 1), slice(a0, a1)))
        REPORT[f"c4_s{s}_outputs_{bars['name']}"] = errs
        _check_grads(m.grads(), gref, bars, f"c4_s{s}_grads_{bars['name']}")
    g.close(); m.close()


# ---------------------------------------------------------------------------------------
# edge cases through forward + backward
# ---------------------------------------------------------------------------------------

def _isolated_atom():
    return Batch(atom_ptr=np.array([0, 1], np.int64), positions=np.array([[5.0, 5.0, 5.0]]),
                 lattice=(np.eye(3) * 30.0)[None], species=np.array([26], np.int32),
                 energy_per_atom=np.array([-3.0]), forces=np.zeros((1, 3)), stress=np.zeros((1, 3, 3)),
                 magmom=np.array([2.0]), magmom_mask=np.ones(1, np.uint8))


def _edge_batch():
    c2 = make_config_batch("C2")
    sc = simple_cubic(3.0, Z=3)
    sc.magmom_mask = np.ones(1, np.uint8)
    return concat_batches([split_batch(c2, [0, 1]), _isolated_atom(), dimer(2.0, 30.0), sc,
                           split_batch(c2, [2, 3])])


@pytest.mark.parametrize("cut", [(5.0, 3.0), (6.0, 3.0)])
@pytest.mark.parametrize("prec", sorted(MODES))
def test_edge_cases_forward_backward(ctx, params, prec, cut):
    b, bars = _labels64(_edge_batch()), MODES[prec]
    cfg = ModelConfig(r_atom=cut[0], r_bond=cut[1])
    og = build_graph_batch(b, cut[0], cut[1])
    ps = og.counts
    assert ps[2, 1] == 0 and ps[3, 3] == 0 and ps[3, 2] == 2 and ps[4, 3] > 0   # no edges / no angles / 1-atom cell
    terms, gref, ref = loss_and_grad(og, b, params, cfg, LossConfig())
    m = _model(ctx, params, prec)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species, cut[0], cut[1])
    assert tuple(g.counts()) == (og.n_atoms, og.n_edges, og.n_bonds, og.n_angles)
    out = ctx.forward(m, g, train=True)
    loss = ctx.backward(m, g, _labels32(b))
    REPORT[f"edge_{cut[0]}_outputs_{bars['name']}"] = _check_outputs(
        out, {k: torch.as_tensor(v) for k, v in ref.items()}, bars)
    for k, key in enumerate(["total", "E", "F", "S", "M"]):
        assert abs(loss[k] - terms[key]) <= bars.get("loss", 1e-5) * max(abs(terms[key]), 1e-6), key
    _check_grads(m.grads(), gref, bars, f"edge_{cut[0]}_grads_{bars['name']}")
    g.close(); m.close()


# ---------------------------------------------------------------------------------------
# NULL labels skip their task (chg_labels)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("drop", ["forces", "stress", "magmom", "energy_per_atom", "magmom_mask"])
def test_missing_labels_skip_task(ctx, params, drop):
    b = _labels64(make_config_batch("C2"))
    w = dict(energy_per_atom=2.0, forces=1.5, stress=0.1, magmom=0.1)
    if drop in w:
        w[drop] = 0.0
    lb = b
    if drop == "magmom_mask":                      # NULL mask = every magmom labelled
        lb = Batch(**{**b.__dict__, "magmom_mask": np.ones_like(b.magmom_mask)})
    terms, gref, _ = loss_and_grad(build_graph_batch(b), lb, params, CFG,
                                   LossConfig(w_e=w["energy_per_atom"], w_f=w["forces"], w_s=w["stress"],
                                              w_m=w["magmom"]))
    m = _model(ctx, params, 0)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    ctx.forward(m, g, train=True, host=False)
    lab = _labels32(b)
    lab[drop] = None
    loss = ctx.backward(m, g, lab)
    for k, key in enumerate(["total", "E", "F", "S", "M"]):
        assert abs(loss[k] - terms[key]) <= 1e-5 * max(abs(terms[key]), 1e-6), (drop, key, loss[k], terms[key])
    _check_grads(m.grads(), gref, MODES[0], f"missing_{drop}")
    g.close(); m.close()


def test_all_labels_missing_is_arg_error(ctx, params):
    b = make_config_batch("C2")
    m = _model(ctx, params, 0)
    g = ctx.build_graph(b.atom_ptr, b.positions, b.lattice, b.species)
    ctx.forward(m, g, train=True, host=False)
    with pytest.raises(chg.ChgError) as e:
        ctx.backward(m, g, dict(magmom_mask=b.magmom_mask))
    assert e.value.name == "CHG_ERR_ARG"
    g.close(); m.close()
