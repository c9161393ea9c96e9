"""Thin ctypes binding of libchg (include/chg.h) — argument marshalling only.

Every computation happens in libchg.so (CUDA, sm_100a).  PyTorch is used only
for device memory / streams by callers that pass device tensors.  There is no
CPU fallback: importing this module on a machine without the library raises.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from typing import Dict, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHG_LIB_PATH") or os.path.join(_PKG, "libchg.so")   # override: A/B timing builds

CHG_OK = 0
STATUS = {0: "CHG_OK", 1: "CHG_ERR_ARG", 2: "CHG_ERR_GEOMETRY", 3: "CHG_ERR_SPECIES", 4: "CHG_ERR_CAPACITY",
          5: "CHG_ERR_NONFINITE", 6: "CHG_ERR_CUDA", 7: "CHG_ERR_NCCL", 8: "CHG_ERR_STATE"}


class ChgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class Cutoffs(C.Structure):
    _fields_ = [("r_atom", C.c_double), ("r_bond", C.c_double)]


class ModelCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("d", "n_radial", "n_angular", "envelope_p", "n_atom_conv", "n_bond_conv",
                                       "gmlp_hidden", "n_species", "head_hidden", "mlp_precision")]


class Pred(C.Structure):
    _fields_ = [("energy", C.c_void_p), ("energy_per_atom", C.c_void_p), ("forces", C.c_void_p),
                ("stress", C.c_void_p), ("magmom", C.c_void_p), ("on_device", C.c_int)]


class Labels(C.Structure):
    _fields_ = [("energy_per_atom", C.c_void_p), ("forces", C.c_void_p), ("stress", C.c_void_p),
                ("magmom", C.c_void_p), ("magmom_mask", C.c_void_p), ("on_device", C.c_int)]


class LossCfg(C.Structure):
    _fields_ = [("w_e", C.c_float), ("w_f", C.c_float), ("w_s", C.c_float), ("w_m", C.c_float),
                ("huber_delta", C.c_float), ("n_struct_global", C.c_int64), ("n_atoms_global", C.c_int64),
                ("n_magmom_global", C.c_int64)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("step", C.c_int64), ("allreduce", C.c_int), ("defer_check", C.c_int)]


# every symbol include/chg.h declares (checked by tests/test_abi_symbols.py)
SYMBOLS = ["chg_ctx_create", "chg_ctx_destroy", "chg_last_error", "chg_sync", "chg_launch_count",
           "chg_nccl_unique_id", "chg_ctx_set_nccl", "chg_build_graph", "chg_graph_counts", "chg_graph_export",
           "chg_graph_destroy", "chg_graph_wait", "chg_md_verlet", "chg_model_create", "chg_model_destroy", "chg_model_layout",
           "chg_model_num_params", "chg_model_set", "chg_model_get", "chg_model_device_ptr", "chg_forward",
           "chg_forward_conservative",
           "chg_backward", "chg_step", "chg_balance", "chg_profile", "chg_profile_query", "chg_debug_gemm", "chg_debug_get",
           "chg_capture_step", "chg_exec_step", "chg_exec_destroy", "chg_ctx_set_grad_overlap",
           "chg_build_graph_skin", "chg_graph_refresh", "chg_md_capture", "chg_md_run", "chg_md_exec_destroy"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libchg.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libchg.so not built at {path}; run __graft_entry__.build()")
    lib = C.CDLL(path)
    vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
    sig = {
        "chg_ctx_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
        "chg_ctx_destroy": (None, [vp]),
        "chg_last_error": (C.c_char_p, [vp]),
        "chg_sync": (C.c_int, [vp]),
        "chg_launch_count": (i64, [vp]),
        "chg_nccl_unique_id": (C.c_int, [vp]),
        "chg_ctx_set_nccl": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "chg_build_graph": (C.c_int, [vp, i32, vp, vp, vp, vp, Cutoffs, C.c_int, C.POINTER(vp)]),
        "chg_graph_counts": (C.c_int, [vp, vp, vp]),
        "chg_graph_export": (C.c_int, [vp] + [vp] * 11),
        "chg_graph_destroy": (None, [vp]),
        "chg_graph_wait": (C.c_int, [vp, vp]),
        "chg_md_verlet": (C.c_int, [vp, i64, vp, vp, vp, vp, C.c_double, C.c_int]),
        "chg_model_create": (C.c_int, [vp, C.POINTER(ModelCfg), C.POINTER(vp)]),
        "chg_model_destroy": (None, [vp]),
        "chg_model_layout": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_char_p)),
                                       C.POINTER(C.POINTER(i64)), C.POINTER(C.POINTER(i32))]),
        "chg_model_num_params": (i64, [vp]),
        "chg_model_set": (C.c_int, [vp, C.c_int, vp, i64]),
        "chg_model_get": (C.c_int, [vp, C.c_int, vp, i64]),
        "chg_model_device_ptr": (vp, [vp, C.c_int]),
        "chg_forward": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(Pred)]),
        "chg_forward_conservative": (C.c_int, [vp, vp, vp, C.POINTER(Pred)]),
        "chg_backward": (C.c_int, [vp, vp, vp, C.POINTER(Labels), C.POINTER(LossCfg), dp]),
        "chg_step": (C.c_int, [vp, vp, C.POINTER(AdamCfg)]),
        "chg_balance": (C.c_int, [vp, i32, i32, vp]),
        "chg_debug_get": (C.c_int, [vp, C.c_char_p, vp, i64, C.POINTER(i64), C.POINTER(i64)]),
        "chg_profile": (C.c_int, [vp, C.c_int]),
        "chg_debug_gemm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
        "chg_profile_query": (C.c_int, [vp, C.c_int, C.c_char_p, dp, C.POINTER(i64), dp, dp]),
        "chg_capture_step": (C.c_int, [vp, vp, vp, C.POINTER(Labels), C.POINTER(LossCfg), C.POINTER(AdamCfg),
                                       C.POINTER(vp)]),
        "chg_exec_step": (C.c_int, [vp, vp, C.POINTER(AdamCfg)]),
        "chg_exec_destroy": (None, [vp]),
        "chg_ctx_set_grad_overlap": (C.c_int, [vp, C.c_int]),
        "chg_build_graph_skin": (C.c_int, [vp, i32, vp, vp, vp, vp, Cutoffs, C.c_double, C.c_int, C.POINTER(vp)]),
        "chg_graph_refresh": (C.c_int, [vp, vp, vp, vp]),
        "chg_md_capture": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_double, C.POINTER(Pred), vp, C.POINTER(vp)]),
        "chg_md_run": (C.c_int, [vp, vp, C.c_int]),
        "chg_md_exec_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(x) -> Optional[int]:
    """Pointer of a numpy array (host) or torch tensor (host/device)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous()
        return x.data_ptr()
    raise TypeError(type(x))


def _on_device(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


# chg_model_cfg.mlp_precision values this build implements (include/chg.h)
PRECISION_MODES = {0: "fp32", 1: "3xtf32", 2: "tf32", 3: "bf16"}


def default_model_cfg() -> ModelCfg:
    """d = 64, 31 radial / angular bases, p = 8; three interaction blocks
    plus a final atom conv (reading Q17); GatedMLP hidden 64 (Q12); 94 species (Q28)."""
    return ModelCfg(d=64, n_radial=31, n_angular=31, envelope_p=8, n_atom_conv=4, n_bond_conv=3,
                    gmlp_hidden=64, n_species=94, head_hidden=64, mlp_precision=0)


class Context:
    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.lib = load()
        h = C.c_void_p()
        self._check(self.lib.chg_ctx_create(device, stream, C.byref(h)), None)
        self.h = h
        self.device = device
        self._children = weakref.WeakSet()   # graphs / models bound to this ctx

    def _check(self, st: int, h=None):
        if st != CHG_OK:
            msg = self.lib.chg_last_error(h if h is not None else getattr(self, "h", None))
            raise ChgError(st, (msg or b"").decode())

    def close(self):
        """Destroys the ctx; graphs and models bound to it are released first."""
        if getattr(self, "h", None):
            for ch in list(self._children):
                ch.close()
            self.lib.chg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self._check(self.lib.chg_sync(self.h))

    def launch_count(self) -> int:
        return int(self.lib.chg_launch_count(self.h))

    def set_nccl(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, 128)
        self._check(self.lib.chg_ctx_set_nccl(self.h, buf, nranks, rank))

    def set_grad_overlap(self, on: bool = True):
        """chg_ctx_set_grad_overlap: bucketed gradient allreduce during the backward (NEXT-3)."""
        self._check(self.lib.chg_ctx_set_grad_overlap(self.h, int(on)))

    # ---- graph
    def wait_graph(self, graph: "Graph"):
        """This context's stream waits for `graph`'s build (graph prefetch: built by another
        Context of the same device on its own stream; chg_forward also waits implicitly)."""
        self._check(self.lib.chg_graph_wait(self.h, graph.h))

    def md_verlet(self, positions, velocities, forces, inv_mass, dt_fs: float, drift: bool):
        """chg_md_verlet: one velocity-Verlet half step on device tensors (fp64 positions /
        velocities [n,3], fp32 forces [n,3], fp64 inverse masses [n]; eV, Å, amu, fs)."""
        n = int(positions.shape[0])
        self._check(self.lib.chg_md_verlet(self.h, n, _ptr(positions), _ptr(velocities), _ptr(forces), _ptr(inv_mass),
                                           float(dt_fs), int(bool(drift))))

    def build_graph(self, atom_ptr, positions, lattice, species, r_atom: float = 5.0, r_bond: float = 3.0,
                    skin: float = 0.0) -> "Graph":
        """chg_build_graph; skin > 0: chg_build_graph_skin (lists with r + skin, model cutoffs r:
        a fixed-topology graph for chg_graph_refresh / captured MD steps)."""
        ap = np.ascontiguousarray(np.asarray(atom_ptr, np.int64))
        dev = _on_device(positions)
        if not dev:
            positions = np.ascontiguousarray(np.asarray(positions, np.float64))
            lattice = np.ascontiguousarray(np.asarray(lattice, np.float64))
            species = np.ascontiguousarray(np.asarray(species, np.int32))
        h = C.c_void_p()
        if skin > 0:
            self._check(self.lib.chg_build_graph_skin(self.h, ap.shape[0] - 1, _ptr(ap), _ptr(positions),
                                                      _ptr(lattice), _ptr(species), Cutoffs(r_atom, r_bond),
                                                      float(skin), int(dev), C.byref(h)))
        else:
            self._check(self.lib.chg_build_graph(self.h, ap.shape[0] - 1, _ptr(ap), _ptr(positions), _ptr(lattice),
                                                 _ptr(species), Cutoffs(r_atom, r_bond), int(dev), C.byref(h)))
        return Graph(self, h, ap.shape[0] - 1)

    def refresh_graph(self, graph: "Graph", positions, flag=None):
        """chg_graph_refresh: the skin graph's edge geometry from new DEVICE positions; flag (device
        int32 tensor, optional) is set to 1 when an atom moved more than skin / 2 since the build."""
        self._check(self.lib.chg_graph_refresh(self.h, graph.h, _ptr(positions), _ptr(flag)))

    def md_capture(self, model: "Model", graph: "Graph", positions, velocities, inv_mass, dt_fs: float, out: Dict,
                   flag=None) -> "MDExec":
        """chg_md_capture: one velocity-Verlet step on a skin graph (kick + drift, geometry refresh,
        conservative forces into `out` — dict of device tensors, forces required — kick) as a CUDA
        graph; .run(n) replays it."""
        p = Pred(*(_ptr(out.get(k)) for k in ("energy", "energy_per_atom", "forces", "stress", "magmom")), 1)
        h = C.c_void_p()
        self._check(self.lib.chg_md_capture(self.h, model.h, graph.h, _ptr(positions), _ptr(velocities),
                                            _ptr(inv_mass), float(dt_fs), C.byref(p), _ptr(flag), C.byref(h)))
        return MDExec(self, h, (positions, velocities, inv_mass, out, flag, graph, model))

    # ---- compute
    def forward(self, model: "Model", graph: "Graph", train: bool = True, out: Optional[Dict] = None,
                host: bool = True) -> Optional[Dict[str, np.ndarray]]:
        """Runs chg_forward.  host=True returns numpy outputs; host=False writes
        into `out` (dict of device tensors) or returns nothing."""
        N, E, B, A = graph.counts()
        S = graph.n_struct
        if host:
            res = {"energy": np.zeros(S, np.float32), "energy_per_atom": np.zeros(S, np.float32),
                   "forces": np.zeros((N, 3), np.float32), "stress": np.zeros((S, 3, 3), np.float32),
                   "magmom": np.zeros(N, np.float32)}
            p = Pred(*(_ptr(res[k]) for k in ("energy", "energy_per_atom", "forces", "stress", "magmom")), 0)
            self._check(self.lib.chg_forward(self.h, model.h, graph.h, int(train), C.byref(p)))
            return res
        if out:
            p = Pred(*(_ptr(out.get(k)) for k in ("energy", "energy_per_atom", "forces", "stress", "magmom")), 1)
            self._check(self.lib.chg_forward(self.h, model.h, graph.h, int(train), C.byref(p)))
        else:
            self._check(self.lib.chg_forward(self.h, model.h, graph.h, int(train), None))
        return None

    def forward_conservative(self, model: "Model", graph: "Graph", out: Optional[Dict] = None):
        """chg_forward_conservative: energy-head forces F = -dE/dr and stress (160.2/V) dE/deps
        (the reference-CHGNet output) plus energy / magmom, as numpy arrays — or written into
        `out` (dict of device tensors, nothing returned)."""
        if out is not None:
            p = Pred(*(_ptr(out.get(k)) for k in ("energy", "energy_per_atom", "forces", "stress", "magmom")), 1)
            self._check(self.lib.chg_forward_conservative(self.h, model.h, graph.h, C.byref(p)))
            return None
        N, E, B, A = graph.counts()
        S = graph.n_struct
        res = {"energy": np.zeros(S, np.float32), "energy_per_atom": np.zeros(S, np.float32),
               "forces": np.zeros((N, 3), np.float32), "stress": np.zeros((S, 3, 3), np.float32),
               "magmom": np.zeros(N, np.float32)}
        p = Pred(*(_ptr(res[k]) for k in ("energy", "energy_per_atom", "forces", "stress", "magmom")), 0)
        self._check(self.lib.chg_forward_conservative(self.h, model.h, graph.h, C.byref(p)))
        return res

    def backward(self, model: "Model", graph: "Graph", labels: Dict, w=(2.0, 1.5, 0.1, 0.1), delta: float = 0.1,
                 n_struct_global: int = 0, n_atoms_global: int = 0, n_magmom_global: int = 0,
                 sync_loss: bool = True):
        """labels: dict energy_per_atom [S], forces [N,3], stress [S,3,3], magmom [N],
        magmom_mask [N] (numpy → host copy, or CUDA tensors).  A missing / None entry
        skips that task (chg_labels NULL field)."""
        lab, keep = self._labels(labels)
        cfg = LossCfg(w[0], w[1], w[2], w[3], delta, n_struct_global, n_atoms_global, n_magmom_global)
        out = (C.c_double * 5)()
        self._check(self.lib.chg_backward(self.h, model.h, graph.h, C.byref(lab), C.byref(cfg),
                                          out if sync_loss else None))
        return list(out) if sync_loss else None

    def step(self, model: "Model", lr: float, step: int, allreduce: bool = False, beta1=0.9, beta2=0.999, eps=1e-8,
             defer_check: bool = False):
        cfg = AdamCfg(lr, beta1, beta2, eps, step, int(allreduce), int(defer_check))
        self._check(self.lib.chg_step(self.h, model.h, C.byref(cfg)))

    def _labels(self, labels: Dict):
        names = ("energy_per_atom", "forces", "stress", "magmom", "magmom_mask")
        present = [labels[k] for k in names if labels.get(k) is not None]
        dev = _on_device(present[0]) if present else False
        keep = {}
        for k, dt in zip(names, (np.float32, np.float32, np.float32, np.float32, np.uint8)):
            x = labels.get(k)
            keep[k] = None if x is None else (x if dev else np.ascontiguousarray(np.asarray(x, dt)))
        return Labels(*(_ptr(keep[k]) for k in names), int(dev)), keep

    def capture_step(self, model: "Model", graph: "Graph", labels: Dict, w=(2.0, 1.5, 0.1, 0.1), delta: float = 0.1,
                     n_struct_global: int = 0, n_atoms_global: int = 0, n_magmom_global: int = 0,
                     allreduce: bool = False, beta1=0.9, beta2=0.999, eps=1e-8) -> "Exec":
        """chg_capture_step: forward + backward + [allreduce] + Adam on `graph` as one CUDA graph.
        labels: CUDA tensors (kept alive by the returned Exec)."""
        lab, keep = self._labels(labels)
        cfg = LossCfg(w[0], w[1], w[2], w[3], delta, n_struct_global, n_atoms_global, n_magmom_global)
        acfg = AdamCfg(1e-3, beta1, beta2, eps, 1, int(allreduce), 1)
        h = C.c_void_p()
        self._check(self.lib.chg_capture_step(self.h, model.h, graph.h, C.byref(lab), C.byref(cfg), C.byref(acfg),
                                              C.byref(h)))
        return Exec(self, h, (keep, graph, model), (beta1, beta2, eps, allreduce))

    def profile(self, on: bool):
        """Clear and enable/disable per-op device timing (chg_profile)."""
        self._check(self.lib.chg_profile(self.h, int(on)))

    def profile_report(self) -> Dict[str, Dict[str, float]]:
        """{tag: {ms, launches, flops, bytes}} since the last profile(True)."""
        out = {}
        i = 0
        while True:
            tag = C.create_string_buffer(64)
            ms, fl, by = C.c_double(), C.c_double(), C.c_double()
            n = C.c_int64()
            st = self.lib.chg_profile_query(self.h, i, tag, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by))
            if st != CHG_OK:
                break
            out[tag.value.decode()] = {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}
            i += 1
        return out

    def debug_gemm(self, kind: int, engine: int, A: np.ndarray, W: np.ndarray) -> np.ndarray:
        """Kernel unit test: kind 0 -> A @ W, kind 1 -> A.T @ W (W = D), on the
        fp32 CUDA-core engine (0) or the tcgen05 TF32 engine (2)."""
        A = np.ascontiguousarray(A, np.float32)
        W = np.ascontiguousarray(W, np.float32)
        M, K = A.shape
        N = W.shape[1]
        out = np.zeros((M, N) if kind == 0 else (K, N), np.float32)
        self._check(self.lib.chg_debug_gemm(self.h, kind, engine, M, K, N, _ptr(A), _ptr(W), _ptr(out)))
        return out

    def debug(self, name: str) -> np.ndarray:
        r, c = C.c_int64(), C.c_int64()
        self._check(self.lib.chg_debug_get(self.h, name.encode(), None, 0, C.byref(r), C.byref(c)))
        out = np.zeros((r.value, c.value), np.float32)
        self._check(self.lib.chg_debug_get(self.h, name.encode(), _ptr(out), out.size, C.byref(r), C.byref(c)))
        return out


class Graph:
    def __init__(self, ctx: Context, h, n_struct: int):
        self.ctx, self.h, self.n_struct = ctx, h, n_struct
        ctx._children.add(self)
        t = (C.c_int64 * 4)()
        ctx._check(ctx.lib.chg_graph_counts(h, t, None))
        self._counts = tuple(int(x) for x in t)

    def counts(self):
        """(N, E, B, A): atoms, directed edges, bond edges, ordered angles."""
        return self._counts

    def per_struct(self) -> np.ndarray:
        """[S, 4] per-structure (N, E, B, A)."""
        t = (C.c_int64 * 4)()
        ps = np.zeros((self.n_struct, 4), np.int64)
        self.ctx._check(self.ctx.lib.chg_graph_counts(self.h, t, _ptr(ps) if ps.size else None))
        return ps

    def export(self) -> Dict[str, np.ndarray]:
        N, E, B, A = self._counts
        out = {"row_ptr": np.zeros(N + 1, np.int32), "nbr": np.zeros(E, np.int32), "img": np.zeros((E, 3), np.int8),
               "vec": np.zeros((E, 4), np.float32), "bond_id": np.zeros(E, np.int32),
               "bond_edge": np.zeros(B, np.int32), "angle_ptr": np.zeros(B + 1, np.int32),
               "angle_b1": np.zeros(A, np.int32), "angle_b2": np.zeros(A, np.int32), "rev": np.zeros(E, np.int32),
               "swap": np.zeros(A, np.int32)}
        keys = ["row_ptr", "nbr", "img", "vec", "bond_id", "bond_edge", "angle_ptr", "angle_b1", "angle_b2", "rev",
                "swap"]
        self.ctx._check(self.ctx.lib.chg_graph_export(self.h, *[_ptr(out[k]) for k in keys]))
        return out

    def close(self):
        if getattr(self, "h", None) and getattr(self.ctx, "h", None):
            self.ctx.lib.chg_graph_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MDExec:
    """A captured MD step (chg_md_exec); .run(n) replays it n times on the ctx stream."""

    def __init__(self, ctx: "Context", h, keep):
        self.ctx, self.h, self._keep = ctx, h, keep

    def run(self, n: int = 1):
        self.ctx._check(self.ctx.lib.chg_md_run(self.ctx.h, self.h, int(n)))

    def close(self):
        if self.h:
            self.ctx.lib.chg_md_exec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Exec:
    """A captured training step (chg_exec); .step(lr, step) replays it on the ctx stream."""

    def __init__(self, ctx: "Context", h, keep, adam):
        self.ctx, self.h, self._keep, self._adam = ctx, h, keep, adam

    def step(self, lr: float, step: int):
        b1, b2, eps, ar = self._adam
        cfg = AdamCfg(lr, b1, b2, eps, step, int(ar), 1)
        self.ctx._check(self.ctx.lib.chg_exec_step(self.ctx.h, self.h, C.byref(cfg)))

    def close(self):
        if self.h:
            self.ctx.lib.chg_exec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Model:
    def __init__(self, ctx: Context, cfg: Optional[ModelCfg] = None):
        self.ctx = ctx
        self.cfg = cfg or default_model_cfg()
        h = C.c_void_p()
        ctx._check(ctx.lib.chg_model_create(ctx.h, C.byref(self.cfg), C.byref(h)))
        self.h = h
        self.P = int(ctx.lib.chg_model_num_params(h))
        ctx._children.add(self)

    def layout(self):
        n = C.c_int()
        names = C.POINTER(C.c_char_p)()
        offs = C.POINTER(C.c_int64)()
        shp = C.POINTER(C.c_int32)()
        self.ctx._check(self.ctx.lib.chg_model_layout(self.h, C.byref(n), C.byref(names), C.byref(offs),
                                                      C.byref(shp)))
        out = []
        for i in range(n.value):
            r, c = shp[2 * i], shp[2 * i + 1]
            out.append((names[i].decode(), (r, c) if c else (r,), int(offs[i])))
        return out

    def set(self, which: int, flat: np.ndarray):
        a = np.ascontiguousarray(np.asarray(flat, np.float32))
        self.ctx._check(self.ctx.lib.chg_model_set(self.h, which, _ptr(a), a.size))

    def get(self, which: int) -> np.ndarray:
        a = np.zeros(self.P, np.float32)
        self.ctx._check(self.ctx.lib.chg_model_get(self.h, which, _ptr(a), a.size))
        return a

    def set_params(self, flat):
        self.set(0, flat)

    def params(self):
        return self.get(0)

    def grads(self):
        return self.get(1)

    def device_ptr(self, which: int) -> int:
        return int(self.ctx.lib.chg_model_device_ptr(self.h, which))

    def close(self):
        if getattr(self, "h", None) and getattr(self.ctx, "h", None):
            self.ctx.lib.chg_model_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def balance(loads: Sequence[int], n_ranks: int) -> np.ndarray:
    lib = load()
    a = np.ascontiguousarray(np.asarray(loads, np.int64))
    out = np.zeros(a.shape[0], np.int32)
    st = lib.chg_balance(_ptr(a) if a.size else None, a.shape[0], n_ranks, _ptr(out) if a.size else None)
    if st != CHG_OK:
        raise ChgError(st, "chg_balance")
    return out


def nccl_unique_id() -> bytes:
    lib = load()
    buf = C.create_string_buffer(128)
    st = lib.chg_nccl_unique_id(buf)
    if st != CHG_OK:
        raise ChgError(st, "chg_nccl_unique_id")
    return buf.raw
