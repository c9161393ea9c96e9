#!/usr/bin/env python
"""Benchmark of the FastCHGNet training step on B200 (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Step = chg_build_graph (A1) + chg_forward(train) (A2-A6) + chg_backward (A7-A8)
+ chg_step (A9: NCCL allreduce when N > 1, finite check, fused Adam) on one
synthetic batch.  Workload: N = 1 -> C2 (40 MPtrj-shaped structures, BASELINE
configs[1]); N > 1 -> C3 (128 structures per GPU, load-balanced with
chg_balance, weak scaling).  `value` is device-timed (CUDA events on the
library stream, inputs resident in HBM, L2 flushed between steps, max over
ranks); `e2e` is the same step through the C ABI from pinned HOST buffers with
the H2D copies and the loss D2H inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train structures/s (fwd+bwd) at 1/2/4/8 B200; gather-scatter HBM GB/s"
PEAKS = {"hbm_gbs": 6547.5, "sm_max_mhz": 1965.0}
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        PEAKS.update(json.load(f))
    PEAK_SRC = "measured (MEASURED_PEAKS.json)"
except Exception:
    PEAK_SRC = "fallback (B200_PROFILING.md)"
# FP32 CUDA-core peak: 148 SMs x 128 FMA/clk x 2 flop x max SM clock
FP32_PEAK_TFLOPS = 148 * 128 * 2 * PEAKS.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
# TF32 dense tensor peak: measured bf16 cuBLAS peak (sustained: kernels timed inside a long step)
# x the nominal tf32:bf16 ratio 1.1 : 2.25 PF/s (B200_PROFILING.md)
TF32_PEAK_TFLOPS = PEAKS.get("bf16_tflops_sustained", PEAKS.get("bf16_tflops", 1590.0)) * 1.1 / 2.25
# 3xTF32 (mlp_precision 1): every fp32 product is three TF32 MMAs (A_lo·B_hi + A_hi·B_lo + A_hi·B_hi),
# so the tensor roof for the algorithmic flops is a third of the TF32 peak
PREC_CODE = {"fp32": 0, "3xtf32": 1, "tf32": 2, "bf16": 3}
DTYPE = {"fp32": "f32", "3xtf32": "f32 (3xTF32)", "tf32": "tf32+f32", "bf16": "bf16+f32"}
BF16_PEAK_TFLOPS = PEAKS.get("bf16_tflops_sustained", PEAKS.get("bf16_tflops", 1590.0))


def tensor_peak(precision: str) -> float:
    return {"tf32": TF32_PEAK_TFLOPS, "3xtf32": TF32_PEAK_TFLOPS / 3.0,
            "bf16": BF16_PEAK_TFLOPS}.get(precision, FP32_PEAK_TFLOPS)


def step_roofline(counts, precision: str):
    """whole-step roof from the batch's N, E, B, A (per GPU).
    GEMM flops fwd = 286,592 E + 380,800 A + 28,544 B + 75,136 N, step = 3 x fwd;
    compulsory bytes fwd = 256 (14E + 6A + 7B + 12N) + 24E + 12A, step = 3 x fwd."""
    N, E, B, A = (float(x) for x in counts)
    flops = 3.0 * (286592 * E + 380800 * A + 28544 * B + 75136 * N)
    byts = 3.0 * (256 * (14 * E + 6 * A + 7 * B + 12 * N) + 24 * E + 12 * A)
    t_tensor = flops / (tensor_peak(precision) * 1e12)
    t_hbm = byts / (PEAKS["hbm_gbs"] * 1e9)
    return flops, byts, t_tensor, t_hbm
# profile tags (chg_profile call sites) of the GatedMLP contractions: on tcgen05 in tf32 mode (NS)
TC_ROW_TAGS = {"ac_f1", "ac_f2", "bc_f1", "bc_f2", "ac_dZ", "ac_dX", "bc_dZ", "bc_dX", "ac_P", "bc_P", "ac_dvS",
               "bc_dvS", "bc_deS"}
TC_WG_TAGS = {"ac_W1_wg", "ac_W2_wg", "bc_W1_wg", "bc_W2_wg", "ac_W1v_wg", "bc_W1p_wg"}
WG_TAGS = TC_WG_TAGS | {"ac_out_wg", "bc_out_wg", "bc_outb_wg", "head_wg", "headM_wg", "proj_wg"}
ROW_TAGS = TC_ROW_TAGS | {"ac_fout", "bc_fout", "head_f", "proj_f", "headM_f", "ac_dagg", "bc_daggb", "head_b",
                          "headM_b", "dbasis"}


def kernel_of(tag: str, precision: str) -> str:
    """CUDA kernel (ncu name) that a profile tag times; the roofline is taken per kernel."""
    if tag.startswith("segsum"):
        return "k_segsum"
    if tag.endswith("_red"):
        return "k_wgrad_reduce"
    if tag in TC_ROW_TAGS:
        return "k_rowgemm_tc" if precision != "fp32" else "k_rowgemm"
    if tag in TC_WG_TAGS:
        return "k_wgrad_tc" if precision != "fp32" else "k_wgrad"
    if tag in ROW_TAGS:
        return "k_rowgemm"
    if tag in WG_TAGS:
        return "k_wgrad"
    if tag in ("head_mlp_f", "head_mlp_b", "head_reduce", "species_grad", "proj_basis", "proj_bwd", "proj_reduce"):
        return {"head_mlp_f": "k_head_fwd", "head_mlp_b": "k_head_bwd", "head_reduce": "k_head_reduce",
                "species_grad": "k_species_grad", "proj_basis": "k_proj_fwd", "proj_bwd": "k_proj_bwd",
                "proj_reduce": "k_proj_reduce"}[tag]
    return {"segsum": "k_segsum", "gate_fwd": "k_gate_fwd", "gate_bwd": "k_gate_bwd", "wgrad_reduce": "k_wgrad_reduce",
            "tc_pack": "k_pack_b", "rows_add": "k_rows_add"}.get(tag, tag)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batches", type=int, default=4, help="distinct pre-generated batches cycled through")
    ap.add_argument("--prefetch", default="auto", choices=["auto", "e2e", "all", "off"],
                    help="graph prefetch on a builder context (SURVEY NEXT-3): all = the next step's graph is "
                         "built on a high-priority stream during this step in every pass (measured +1.7 %% at C2, "
                         "+1.2 %% at C3 on one GPU, +1.2 %% at N = 2, but a 20 %% outlier at N = 4 next to NCCL); "
                         "e2e = in the e2e pass only; off = every build inline; auto (default) = all at N = 1, off "
                         "at N > 1 (DESIGN.md §12)")
    ap.add_argument("--workload", default="auto", choices=["auto", "C2", "C3", "C4"],
                    help="auto: C2 at N=1, C3 at N>1; C4: skewed 4-400-atom oxides (BASELINE configs[3])")
    ap.add_argument("--per-gpu", type=int, default=0, help="structures per GPU (default: 40 at N=1, 128 at N>1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32", "bf16", "fp32"],
                    help="GatedMLP GEMM engine (headline mode): 3xtf32 = tcgen05 split-operand fp32 (strict "
                         "parity, the paper's fp32, P:473), tf32 = tcgen05 TF32 (NS loosened), fp32 = CUDA cores")
    ap.add_argument("--no-side-modes", action="store_true", help="skip timing the two other precision modes")
    ap.add_argument("--grad-overlap", default="on", choices=["on", "off"],
                    help="N > 1: bucketed gradient allreduce during the backward (SURVEY NEXT-3, P:353)")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


WL_DESC = {"C2": "MPtrj-shaped synthetic batch", "C3": "MPtrj-shaped synthetic batch",
           "C4": "skewed synthetic oxides (4-400 atoms, O/Li/Mn/Fe/Co/Ni)"}


def _workload(n_gpus: int, per_gpu: int, name: str = "auto"):
    if name != "auto":
        return name, per_gpu or (40 if name == "C2" else 128)
    if n_gpus == 1 and per_gpu in (0, 40):
        return "C2", 40
    return "C3", per_gpu or 128


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampled every 25 ms from before the timed passes to after them; only samples
    whose timestamp falls inside a timed window (mark_begin / mark_end) are kept."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None
        self.windows = []

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "25", "-i", str(self.device)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def mark_begin(self):
        self.windows.append([time.time(), None])

    def mark_end(self):
        self.windows[-1][1] = time.time()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": PEAKS.get("sm_max_mhz"), "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=5)
        import datetime
        sm, mx, reasons, total = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                clk, mxv = float(f[2]), float(f[3])
            except ValueError:
                continue
            total += 1
            if not any(w0 - 0.03 <= ts <= (w1 or w0) + 0.03 for w0, w1 in self.windows):
                continue
            sm.append(clk)
            mx = mxv
            for k, v in zip(names, f[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "samples_total": total, "reasons": sorted(reasons),
                "window": "samples inside the timed passes (device-resident + e2e), 25 ms period"}


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the fp64 oracle on the host cores
# ---------------------------------------------------------------------------
def _oracle_step(batch, params, cfg, lc, state):
    from oracle.graph import build_graph_batch
    from oracle.train import adam_step, loss_and_grad
    g = build_graph_batch(batch)
    _, grad, _ = loss_and_grad(g, batch, params, cfg, lc)
    state["t"] += 1
    p, state["m"], state["v"] = adam_step(params, state["m"], state["v"], grad, state["t"], 3e-4)
    return p


def _oracle_sample(wl: str, per: int, budget_s: float):
    """Largest prefix of the workload's first batch whose oracle step fits the budget."""
    import torch
    from chg_inputs import init_flat_params, make_config_batch, split_batch
    from oracle.model import ModelConfig, param_layout
    from oracle.train import LossConfig
    cfg = ModelConfig()
    full = make_config_batch(wl, 0, n_struct=per)
    params = init_flat_params(param_layout(cfg), seed=0).astype(np.float32).astype(np.float64)
    lc = LossConfig()
    n = full.n_struct
    sample = full
    state = {"t": 0, "m": np.zeros_like(params), "v": np.zeros_like(params)}
    t0 = time.time()
    _oracle_step(split_batch(full, list(range(min(4, n)))), params, cfg, lc, state)
    per_struct = (time.time() - t0) / min(4, n)
    fit = max(1, min(n, int(budget_s / max(per_struct, 1e-3))))
    if fit < n:
        sample = split_batch(full, list(range(fit)))
    return sample, params, cfg, lc, torch.get_num_threads()


def cpu_baseline(wl: str, per: int, seconds: float):
    sample, params, cfg, lc, cores = _oracle_sample(wl, per, seconds / 2)
    state = {"t": 0, "m": np.zeros_like(params), "v": np.zeros_like(params)}
    t0 = time.time()
    done = 0
    while True:
        params = _oracle_step(sample, params, cfg, lc, state)
        done += sample.n_struct
        if time.time() - t0 >= seconds / 2:
            break
    dt = time.time() - t0
    return {"value": done / dt, "unit": "structures/s", "cores": cores, "host_cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{sample.n_struct} of the {wl} batch's {per} structures, fp64 torch CPU oracle fwd+bwd+Adam "
                      f"({done} structure-steps in {dt:.1f} s)"}


def run_reference(a, ws, rank):
    if rank != 0:
        return
    wl, per = _workload(ws, a.per_gpu, a.workload)
    sample, params, cfg, lc, cores = _oracle_sample(wl, per, 8.0)
    state = {"t": 0, "m": np.zeros_like(params), "v": np.zeros_like(params)}
    for _ in range(a.warmup):
        params = _oracle_step(sample, params, cfg, lc, state)
    t0 = time.time()
    for _ in range(a.steps):
        params = _oracle_step(sample, params, cfg, lc, state)
    dt = time.time() - t0
    v = sample.n_struct * a.steps / dt
    cb = {"value": v, "unit": "structures/s", "cores": cores, "host_cores": os.cpu_count(), "kind": "oracle",
          "sample": f"{sample.n_struct} structures of the {wl} batch per step (fp64 torch CPU oracle fwd+bwd+Adam)"}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "structures/s", "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * dt / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "structures_per_step": sample.n_struct, "host_threads": cores},
        "cpu_baseline": cb, "e2e": {"value": v, "unit": "structures/s", "h2d_bytes_per_step": 0,
                                    "d2h_bytes_per_step": 0}}), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    a = _args()
    ws, rank, local = _dist()
    if a.impl == "reference":
        run_reference(a, ws, rank)
        return
    import torch
    import torch.distributed as dist
    from chg_inputs import init_flat_params, make_config_batch, split_batch
    from paper_2412_20796_b200 import chg

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl, per = _workload(ws, a.per_gpu, a.workload)
    stream = torch.cuda.Stream()
    ctx = chg.Context(local, stream=stream.cuda_stream)
    if ws > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(chg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ctx.set_nccl(bytes(uid.cpu().numpy()), ws, rank)
        ctx.set_grad_overlap(a.grad_overlap == "on")
    def make_model(prec):
        cfg = chg.default_model_cfg()
        cfg.mlp_precision = PREC_CODE[prec]
        mm = chg.Model(ctx, cfg)
        lay = [(n, s) for n, s, _ in mm.layout()]         # the library's own layout table
        mm.set_params(init_flat_params(lay, seed=0).astype(np.float32))
        return mm
    others = [] if a.no_side_modes else [p for p in PREC_CODE if p != a.precision]
    models = {p: make_model(p) for p in [a.precision] + others}
    model = models[a.precision]

    # ---- batches: global batch per index, balanced over ranks
    def make_batches(wl, per, nbatches):
        out = []
        for bi in range(nbatches):
            glob = make_config_batch(wl, bi, n_struct=per * ws)
            if ws > 1:
                g_all = ctx.build_graph(glob.atom_ptr, glob.positions, glob.lattice, glob.species)
                ps = g_all.per_struct()
                g_all.close()
                loads = ps[:, 0] + ps[:, 1] + ps[:, 3]              # atoms + edges + angles (Q31)
                rank_of = chg.balance(loads, ws)
                mine = split_batch(glob, np.nonzero(rank_of == rank)[0].tolist())
                per_rank_load = np.bincount(rank_of, weights=loads, minlength=ws)
                contiguous = loads.reshape(ws, -1).sum(1) if glob.n_struct % ws == 0 else per_rank_load
                cv = (float(per_rank_load.std() / per_rank_load.mean()), float(contiguous.std() / contiguous.mean()))
                imb = (float(per_rank_load.max() / per_rank_load.mean()), float(contiguous.max() / contiguous.mean()))
            else:
                mine, cv, imb = glob, (0.0, 0.0), (1.0, 1.0)
            gc = ctx.build_graph(mine.atom_ptr, mine.positions, mine.lattice, mine.species)
            counts = tuple(int(x) for x in gc.counts())              # this rank's N, E, B, A
            gc.close()
            gl = dict(S=glob.n_struct, N=glob.n_atoms, M=int(glob.magmom_mask.sum()))
            dev = dict(pos=torch.as_tensor(mine.positions, device="cuda"),
                       lat=torch.as_tensor(mine.lattice, device="cuda"),
                       spec=torch.as_tensor(mine.species, device="cuda"),
                       lab=dict(energy_per_atom=torch.as_tensor(mine.energy_per_atom, dtype=torch.float32, device="cuda"),
                                forces=torch.as_tensor(mine.forces, dtype=torch.float32, device="cuda"),
                                stress=torch.as_tensor(mine.stress, dtype=torch.float32, device="cuda"),
                                magmom=torch.as_tensor(mine.magmom, dtype=torch.float32, device="cuda"),
                                magmom_mask=torch.as_tensor(mine.magmom_mask, device="cuda")))

            def pinned(x, dt):
                t = torch.empty(x.shape, dtype=dt, pin_memory=True)
                t.copy_(torch.as_tensor(np.ascontiguousarray(x)).to(dt))
                return t.numpy()
            host = dict(pos=pinned(mine.positions, torch.float64), lat=pinned(mine.lattice, torch.float64),
                        spec=pinned(mine.species, torch.int32),
                        lab=dict(energy_per_atom=pinned(mine.energy_per_atom, torch.float32),
                                 forces=pinned(mine.forces, torch.float32),
                                 stress=pinned(mine.stress, torch.float32),
                                 magmom=pinned(mine.magmom, torch.float32),
                                 magmom_mask=pinned(mine.magmom_mask, torch.uint8)))
            h2d = sum(v.nbytes for k, v in host.items() if k != "lab") + sum(v.nbytes for v in host["lab"].values()) \
                + mine.atom_ptr.nbytes
            out.append(dict(ap=mine.atom_ptr, dev=dev, host=host, gl=gl, S=mine.n_struct, cv=cv, imb=imb, h2d=h2d,
                            counts=counts))
        return out

    batches = make_batches(wl, per, a.batches)

    lr0 = (per * ws) / 128 * 3e-4                      # Eq. 14
    total_steps = 2 * (a.warmup + a.steps) + 8
    step_no = [0]

    # graph prefetch: a builder context builds the next step's graph on its own
    # stream while this step's forward / backward run; the step's end waits for that build, so
    # every build stays inside a timed step window (the first step builds its own inline)
    # (high-priority stream: its short kernels are scheduled first whenever SMs free up)
    if a.prefetch == "auto":
        a.prefetch = "all" if ws == 1 else "off"
    bstream = None if a.prefetch == "off" else torch.cuda.Stream(device=local, priority=-5)
    builder = None if a.prefetch == "off" else chg.Context(local, stream=bstream.cuda_stream)

    def build(b, on_host: bool, bctx=None):
        src = b["host"] if on_host else b["dev"]
        return (bctx or ctx).build_graph(b["ap"], src["pos"], src["lat"], src["spec"], 5.0, 3.0)

    def one_step(b, on_host: bool, model=None, g=None, nxt=None, keep_graph=False):
        model = model or models[a.precision]
        step_no[0] += 1
        lr = lr0 * 0.5 * (1 + math.cos(math.pi * step_no[0] / total_steps))   # cosine
        src = b["host"] if on_host else b["dev"]
        if g is None:
            g = build(b, on_host)
        ctx.forward(model, g, train=True, host=False)
        # the build's host part (count readback on the builder stream) is issued once this
        # step's work is queued: after the forward when the loss readback blocks the host
        # (e2e), after the Adam step otherwise — the training stream never runs dry
        gn = build(nxt, on_host, builder) if (nxt is not None and on_host) else None
        loss = ctx.backward(model, g, src["lab"], n_struct_global=b["gl"]["S"], n_atoms_global=b["gl"]["N"],
                            n_magmom_global=b["gl"]["M"], sync_loss=on_host)
        # device-resident pass: no host synchronisation in the step (finite flag checked by a later call)
        ctx.step(model, lr=lr, step=step_no[0], allreduce=ws > 1, defer_check=not on_host)
        if nxt is not None and not on_host:
            gn = build(nxt, on_host, builder)
        if gn is not None:
            ctx.wait_graph(gn)
        if not keep_graph:
            g.close()
        return loss, gn

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")     # 256 MiB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(on_host: bool, profile: bool = False, model=None, bl=None, cached=None, execs=None, inline=False):
        """K steps; cached = prebuilt graphs per batch (graph build outside);
        execs = captured steps per batch (chg_capture_step: one CUDA graph replay per step)."""
        bl = bl or batches
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        if profile:
            ctx.profile(True)
        l0 = ctx.launch_count()
        lb0 = builder.launch_count() if builder else 0
        barrier()
        gnext = None
        for k in range(a.steps):
            b = bl[k % len(bl)]
            use = builder is not None and not profile and not inline and (on_host or a.prefetch == "all")
            nxt = bl[(k + 1) % len(bl)] if (use and k + 1 < a.steps) else None
            ev[k][0].record(stream)
            if execs is not None:
                step_no[0] += 1
                lr = lr0 * 0.5 * (1 + math.cos(math.pi * step_no[0] / total_steps))
                execs[k % len(bl)].step(lr, step_no[0])
            elif cached is not None:
                one_step(b, on_host, model, g=cached[k % len(bl)], keep_graph=True)
            else:
                _, gnext = one_step(b, on_host, model, g=gnext, nxt=nxt)
            ev[k][1].record(stream)
            with torch.cuda.stream(stream):
                flush.zero_()                              # L2 flush outside the timed events
        barrier()
        launches = ctx.launch_count() - l0 + ((builder.launch_count() - lb0) if builder else 0)
        per_step = [s.elapsed_time(e) for s, e in ev]
        ms = sum(per_step)
        rep = ctx.profile_report() if profile else None
        if profile:
            ctx.profile(False)
        rank_ms = [ms]
        if ws > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            allt = [torch.zeros_like(t) for _ in range(ws)]
            dist.all_gather(allt, t)
            rank_ms = [float(x.item()) for x in allt]
            ms = max(rank_ms)
        stats[id(bl), on_host, profile, id(model), cached is not None] = dict(per_step=per_step, rank_ms=rank_ms)
        last_stats[0] = stats[id(bl), on_host, profile, id(model), cached is not None]
        return ms, launches, rep

    stats, last_stats = {}, [None]
    # warm-up covers every cycled batch at least once (its graph / workspace sizes are then known
    # to the memory pool before timing), and at least --warmup steps
    # (with graph prefetch the warm-up runs the prefetching loop too: the builder context's own
    # workspaces and pinned buffers are sized before timing — else the first timed step pays them)
    nwu = max(a.warmup, len(batches))
    for on_host in (False, True):
        gnext = None
        for k in range(nwu):
            nxt = batches[(k + 1) % len(batches)] if (builder is not None and k + 1 < nwu) else None
            _, gnext = one_step(batches[k % len(batches)], on_host, g=gnext, nxt=nxt)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)                                   # nvidia-smi's first sample lands before the timing
    clocks.mark_begin()
    ms, launches, _ = timed(False)
    clocks.mark_end()
    main_stats = last_stats[0]
    clocks.mark_begin()
    ms_e2e, _, _ = timed(True)                        # clocks sampled across both timed passes
    clocks.mark_end()
    clk = clocks.stop()
    # cached-graph variant: graphs built once outside the timed region (training graphs are static
    # per dataset)
    cached = [build(b, False) for b in batches]
    for k in range(a.warmup):
        one_step(batches[k % len(batches)], False, g=cached[k % len(batches)], keep_graph=True)
    ms_cached, _, _ = timed(False, cached=cached)
    # captured variant: the cached graph's whole step (forward + backward + allreduce + Adam) as one
    # CUDA graph per batch, replayed with this step's lr (no host synchronisation inside the step)
    ms_capt, capt_launches, capt_err = None, None, None
    try:
        if ws > 1:     # measured: the capture's first launch fails ("invalid device function") once NCCL
            raise RuntimeError("captured step measured at N = 1 only (multi-rank stream capture fails on this stack)")
        execs = [ctx.capture_step(model, cached[i], b["dev"]["lab"], n_struct_global=b["gl"]["S"],
                                  n_atoms_global=b["gl"]["N"], n_magmom_global=b["gl"]["M"], allreduce=ws > 1)
                 for i, b in enumerate(batches)]
        for k in range(a.warmup):
            execs[k % len(execs)].step(lr0, step_no[0] + 1)
            step_no[0] += 1
        ms_capt, capt_launches, _ = timed(False, execs=execs)
        ctx.sync()
        for x in execs:
            x.close()
    except Exception as ex:          # reported in the line, never silently
        capt_err = f"{type(ex).__name__}: {ex}"
    for g_ in cached:
        g_.close()
    _, _, rep = timed(False, profile=True)
    side = {}
    for other in others:
        for k in range(a.warmup):
            one_step(batches[k % len(batches)], False, models[other])
        ms_o, _, _ = timed(False, model=models[other])
        side[other] = ms_o

    # weak-scaling base: the per-GPU workload of the N > 1 runs (C3, 128 structures) on this one GPU,
    # so value(N) / (N * c3_value(1)) compares equal per-GPU work (the headline N = 1 line stays C2)
    weak_base = None
    if ws == 1 and wl == "C2":
        c3 = make_batches("C3", 128, 2)
        for k in range(a.warmup):
            one_step(c3[k % len(c3)], False)
        ms_c3, _, _ = timed(False, bl=c3, inline=True)    # graph builds inline, as in the N > 1 runs
        s_c3 = sum(c3[k % len(c3)]["gl"]["S"] for k in range(a.steps))
        roof_c3 = [step_roofline(c3[k % len(c3)]["counts"], a.precision) for k in range(a.steps)]
        weak_base = {"workload": "C3: 128 MPtrj-shaped structures on 1 GPU (the per-GPU work of the N > 1 runs; "
                                 "graph builds inline as at N > 1)",
                     "value": s_c3 / (ms_c3 / 1e3), "unit": "structures/s", "ms_per_step": ms_c3 / a.steps,
                     "whole_step_frac": sum(max(r[2], r[3]) for r in roof_c3) / (ms_c3 / 1e3)}
        _, _, rep_c3 = timed(False, profile=True, bl=c3)         # gather-scatter GB/s at C3 (§8(d) item 7)

    # C5 (BASELINE configs[4]): one 4,096-atom LiFePO4-like cell, graph build + forward with the
    # force / stress readout (inference path), device-timed latency
    c5 = None
    if ws == 1 and wl == "C2":
        b5 = make_config_batch("C5")
        d5 = (torch.as_tensor(b5.positions, device="cuda"), torch.as_tensor(b5.lattice, device="cuda"),
              torch.as_tensor(b5.species, device="cuda"))
        model5 = models[a.precision]

        def inf5():
            g5 = ctx.build_graph(b5.atom_ptr, d5[0], d5[1], d5[2], 5.0, 3.0)
            ctx.forward(model5, g5, train=False, host=False)
            return g5
        for _ in range(a.warmup):
            inf5().close()
        ev5 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        barrier()
        for k in range(a.steps):
            ev5[k][0].record(stream)
            g5 = inf5()
            ev5[k][1].record(stream)
            g5.close()
        barrier()
        t5 = sorted(s.elapsed_time(e) for s, e in ev5)
        # the same cell through chg_forward_conservative (F = -dE/dr, stress from dE/deps: the
        # reference-CHGNet output)
        for _ in range(a.warmup):
            g5 = ctx.build_graph(b5.atom_ptr, d5[0], d5[1], d5[2], 5.0, 3.0)
            ctx.forward_conservative(model5, g5)
            g5.close()
        ev6 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        barrier()
        for k in range(a.steps):
            ev6[k][0].record(stream)
            g5 = ctx.build_graph(b5.atom_ptr, d5[0], d5[1], d5[2], 5.0, 3.0)
            ctx.forward_conservative(model5, g5)
            ev6[k][1].record(stream)
            g5.close()
        barrier()
        t6 = sorted(s.elapsed_time(e) for s, e in ev6)
        # NEXT-2 MD loop: one velocity-Verlet NVE step (kick+drift, graph rebuild, conservative
        # forces on device, kick), device-timed, for the C5 cell and an 8-atom cell (Table II size)
        from paper_2412_20796_b200.md import NVE, maxwell_boltzmann

        def md_ms(b, mass, per=1, **kw):
            """median device ms per MD step; per steps per timed call (captured: one chunk of
            replays between two moved-atom checks)"""
            md = NVE(ctx, model5, b.atom_ptr, b.positions, b.lattice, b.species, mass,
                     maxwell_boltzmann(mass, 300.0, 0), dt_fs=0.5, **kw)
            md.step(max(a.warmup, per))
            evm = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
            barrier()
            for k in range(a.steps):
                evm[k][0].record(stream)
                md.step(per)
                evm[k][1].record(stream)
            barrier()
            tm = sorted(s.elapsed_time(e) / per for s, e in evm)
            md.close()
            return tm[len(tm) // 2]
        b8 = make_config_batch("C1")
        c5 = {"workload": "C5: one 4,096-atom LiFePO4-like cell (graph build + forward + force/stress readout)",
              "atoms": int(b5.n_atoms), "latency_ms_median": t5[len(t5) // 2], "latency_ms_min": t5[0],
              "conservative_latency_ms_median": t6[len(t6) // 2],
              "conservative_note": "chg_forward_conservative: forward + energy-seeded backward + basis derivatives "
                                   "(includes the host copy of the outputs)",
              "md_step_ms_median": {"C5_4096_atoms": md_ms(b5, np.full(b5.n_atoms, 30.0)),
                                    "C1_Si8": md_ms(b8, np.full(b8.n_atoms, 28.0855))},
              "md_step_ms_median_captured": {
                  "C5_4096_atoms": md_ms(b5, np.full(b5.n_atoms, 30.0), per=10, skin=0.5, captured=True),
                  "C1_Si8": md_ms(b8, np.full(b8.n_atoms, 28.0855), per=10, skin=0.5, captured=True)},
              "md_captured_note": "skin graph (lists r + 0.5 Å, bases zero beyond r) refreshed every step; "
                                  "the step (kick+drift, geometry refresh, conservative forces, kick) replayed "
                                  "as one CUDA graph, 10 replays between moved-atom checks (pays off for small "
                                  "cells only: the skin enlarges the angle list ~2.5x)",
              "md_note": "NEXT-2 velocity-Verlet NVE step: chg_md_verlet kick+drift, graph rebuild from device "
                         "positions, chg_forward_conservative (device outputs), kick; dt 0.5 fs"}

    structs = sum(batches[k % len(batches)]["gl"]["S"] for k in range(a.steps))
    value = structs / (ms / 1e3)
    e2e = structs / (ms_e2e / 1e3)
    h2d = int(np.mean([batches[k % len(batches)]["h2d"] for k in range(a.steps)]))

    # ---- roofline of the dominant kernel (live CUDA events, profiled pass of the same steps)
    kern = {}
    for t, v in rep.items():
        k = kernel_of(t, a.precision)
        d = kern.setdefault(k, {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0, "tags": []})
        for f in ("ms", "launches", "flops", "bytes"):
            d[f] += v[f]
        d["tags"].append(t)
    dom = max(kern, key=lambda k: kern[k]["ms"])
    # shares are of the summed kernel time of the profiled steps, the quantity ncu's launch list sums
    # (the profiled pass itself is slowed by its per-launch events, so its wall time is not the base)
    ms_sum = sum(v["ms"] for v in rep.values()) or 1e-9
    r = kern[dom]
    per_launch_s = r["ms"] / 1e3 / max(r["launches"], 1)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
            tr = tj.get(f"{a.precision}_{wl}", tj.get(a.precision, {})).get(dom)
            traffic = tr["dram_bytes_per_launch"] if tr else None
    except Exception:
        pass
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9
    tfs = r["flops"] / (r["ms"] / 1e3) / 1e12
    on_tc = dom.endswith("_tc")
    flop_peak = tensor_peak(a.precision) if on_tc else FP32_PEAK_TFLOPS
    # binding roof by arithmetic intensity: below the ridge flop_peak / hbm_peak the kernel is HBM-bound
    if r["bytes"] > 0 and (r["flops"] / r["bytes"]) < flop_peak * 1e3 / PEAKS["hbm_gbs"]:
        roof = {"bound": "hbm", "achieved": gbs, "peak": PEAKS["hbm_gbs"], "unit": "GB/s", "peak_source": PEAK_SRC}
        per_launch_alg = r["bytes"] / max(r["launches"], 1)
    elif on_tc:
        roof = {"bound": "tensor", "achieved": tfs, "peak": flop_peak, "unit": "TFLOP/s",
                "peak_source": (PEAK_SRC + " bf16_tflops_sustained") if a.precision == "bf16" else
                               ("tf32 = " + PEAK_SRC + " bf16_tflops_sustained x (1.1/2.25 nominal ratio)"
                                + (" / 3 (3xTF32: three MMAs per fp32 product)" if a.precision == "3xtf32" else ""))}
        per_launch_alg = r["flops"] / max(r["launches"], 1)
    else:
        roof = {"bound": "alu", "achieved": tfs, "peak": flop_peak, "unit": "TFLOP/s",
                "peak_source": "FP32 CUDA cores: 148 SM x 128 FMA/clk x 2 x sm_max_mhz (DESIGN.md)"}
        per_launch_alg = r["flops"] / max(r["launches"], 1)
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": traffic, "kernel": dom, "call_sites": sorted(r["tags"]),
                 "algorithmic_per_launch": per_launch_alg, "algorithmic_unit": "bytes" if roof["bound"] == "hbm" else "flop",
                 "avg_launch_us": per_launch_s * 1e6, "share_of_step": r["ms"] / ms_sum, "share_base": "summed kernel time of the step",
                 "profiled_pass": "same steps with per-launch CUDA events; the concurrent branches run serially "
                                  "while profiling, so each launch's time is its own",
                 "intensity_flop_per_byte": r["flops"] / max(r["bytes"], 1.0),
                 "tensor_frac": tfs / flop_peak if on_tc else None, "hbm_frac": gbs / PEAKS["hbm_gbs"]})
    def gather_of(rp, wl_name):
        gs = {"bytes": sum(v["bytes"] for t, v in rp.items() if t.startswith("segsum")),
              "ms": sum(v["ms"] for t, v in rp.items() if t.startswith("segsum")) or 1e-9}
        return {"kernel": "segsum (atomic-free CSR / rev / swap segmented gather-reduce)", "workload": wl_name,
                "achieved_gbs": gs["bytes"] / (gs["ms"] / 1e3) / 1e9,
                "frac": gs["bytes"] / (gs["ms"] / 1e3) / 1e9 / PEAKS["hbm_gbs"], "peak_gbs": PEAKS["hbm_gbs"],
                "bytes": "algorithmic: each summed row (256 B) + index read once, each target written once"}
    gather = gather_of(rep_c3, "C3") if (ws == 1 and wl == "C2") else gather_of(rep, wl)
    if ws == 1 and wl == "C2":
        gather["at_headline_workload"] = gather_of(rep, wl)
    # whole-step roof from each timed batch's N, E, B, A
    roofs = [step_roofline(batches[k % len(batches)]["counts"], a.precision) for k in range(a.steps)]
    whole = {"flop_per_step": float(np.mean([r[0] for r in roofs])), "bytes_per_step": float(np.mean([r[1] for r in roofs])),
             "t_tensor_ms": 1e3 * float(np.mean([r[2] for r in roofs])), "t_hbm_ms": 1e3 * float(np.mean([r[3] for r in roofs])),
             "tensor_peak_tflops": tensor_peak(a.precision), "hbm_peak_gbs": PEAKS["hbm_gbs"],
             "frac": sum(max(r[2], r[3]) for r in roofs) / (ms / 1e3),
             "note": "max(t_tensor, t_HBM) / measured step time; SURVEY §8(d) algorithmic GEMM flops and compulsory "
                     "bytes of the batch's counts (3 x forward); 3xtf32 roof = TF32 peak / 3"}
    ps_ = sorted(main_stats["per_step"])
    q = lambda f: ps_[min(len(ps_) - 1, int(round(f * (len(ps_) - 1))))]   # noqa: E731
    step_ms = {"median": q(0.5), "p10": q(0.1), "p90": q(0.9), "mean": float(np.mean(ps_))}
    rank_ms = main_stats["rank_ms"]
    ops = {t: {"ms_per_step": v["ms"] / a.steps, "launches_per_step": v["launches"] / a.steps,
               "share": v["ms"] / ms_sum, "kernel": kernel_of(t, a.precision)}
           for t, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])}
    kernels = {k: {"ms_per_step": v["ms"] / a.steps, "share": v["ms"] / ms_sum,
                   "gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9, "tflops": v["flops"] / (v["ms"] / 1e3) / 1e12}
               for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])}

    if rank == 0:
        cb = None
        if not a.no_cpu_baseline and ws == 1:
            cb = cpu_baseline(wl, per, a.cpu_seconds)
        b0 = batches[0]
        line = {
            "metric": METRIC, "value": value, "unit": "structures/s", "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE[a.precision], "data": "synthetic",
            "precision": {"mode": a.precision,
                          "note": "3xtf32: GatedMLP GEMMs on tcgen05 with split operands (hi + lo TF32, three MMAs, "
                                  "fp32 accumulate: strict 1e-4 gradient parity); tf32: tcgen05 TF32 (NS-loosened "
                                  "2e-3); bf16: tcgen05 kind::f16 with BF16 operands rounded as they are staged, fp32 "
                                  "features in HBM (bars in DESIGN §6); fp32: everything on CUDA cores (strict); heads, "
                                  "projections, output linears and all non-GEMM kernels are fp32 in every mode",
                          **{o: {"value": structs / (side[o] / 1e3), "ms_per_step": side[o] / a.steps,
                                 "dtype": DTYPE[o],
                                 "whole_step_frac": sum(max(r[2], r[3]) for r in
                                                        [step_roofline(batches[k % len(batches)]["counts"], o)
                                                         for k in range(a.steps)]) / (side[o] / 1e3),
                                 "whole_step_hbm_frac": sum(r[3] for r in
                                                            [step_roofline(batches[k % len(batches)]["counts"], o)
                                                             for k in range(a.steps)]) / (side[o] / 1e3)}
                             for o in others}},
            "step_ms": step_ms,
            "per_step_ms": [round(x, 4) for x in main_stats["per_step"]],
            "whole_step_roofline": whole,
            "cached_graph": {"value": structs / (ms_cached / 1e3), "unit": "structures/s",
                             "ms_per_step": ms_cached / a.steps,
                             "note": "graphs built once outside the timed region (static per dataset); "
                                     "forward + backward + allreduce + Adam timed"},
            "captured_step": ({"value": structs / (ms_capt / 1e3), "unit": "structures/s",
                               "ms_per_step": ms_capt / a.steps, "kernels_per_step": capt_launches / a.steps,
                               "note": "cached graph + chg_capture_step: the whole step replayed as ONE CUDA graph "
                                       "(no host synchronisation inside; finite flag checked by a later call)"}
                              if ms_capt is not None else {"error": capt_err}),
            "config": {"workload": f"{wl}: {WL_DESC[wl]}, {per} structures per GPU "
                                   f"(5/3 Å cutoffs, d=64, 4 atom-conv / 3 bond-conv)",
                       "structures_per_gpu": per, "global_batch": per * ws, "parallelism": f"dp{ws}",
                       "step": "build_graph + forward + backward + allreduce + Adam",
                       "allreduce": ("bucketed during the backward (NEXT-3)" if a.grad_overlap == "on" else
                                     "one call before Adam") if ws > 1 else "none (1 GPU)",
                       "graph_build": {"value": "prefetched on a builder context during the previous step" if a.prefetch == "all"
                                       else "inline",
                                       "e2e": "inline" if a.prefetch == "off" else
                                       "prefetched on a builder context during the previous step"},
                       "l2": "flushed between steps (256 MiB write, outside the timed events)",
                       "batches_cycled": len(batches), "cv_balanced_vs_contiguous": b0["cv"],
                       "max_over_mean_rank_load_balanced_vs_contiguous": b0["imb"],
                       "counts_first_batch_NEBA": list(b0["counts"]),
                       "per_rank_ms_max_over_mean": max(rank_ms) / (sum(rank_ms) / len(rank_ms))},
            "e2e": {"value": e2e, "unit": "structures/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 40 + 4},
            "gpu_launches": int(launches),
            "weak_scaling_base": weak_base,
            "c5_inference": c5,
            "clocks": clk,
            "roofline": roof,
            "gather_scatter": gather,
            "kernels": kernels,
            "ops": ops,
            "cpu_baseline": cb,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
