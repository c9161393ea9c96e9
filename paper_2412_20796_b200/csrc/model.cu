// model.cu — forward / backward / step orchestration of the FastCHGNet
// training step (A2–A9 of DESIGN.md §"Hot path").
//
// Forward (Fig. 2a): basis (Alg. 2) → embedding + projections (Eq. 2) → for
// t = 0..T-1 { atom conv (Eq. 4) ∥ bond conv (Eq. 5) ∥ angle update (Eq. 6),
// all reading layer-t features (Eq. 11) } → final atom conv → energy, magmom,
// force (Eq. 7) and stress (Eq. 9) heads.
// Backward: first-order reverse mode only (the decomposed heads need no
// derivative of E); gather adjoints are segmented reductions
// through the CSR rows, the reverse-edge map (rev) and the angle swap map
// (swap) — no atomics, fixed order, deterministic.
#include <nccl.h>

#include <cmath>

#include "gemm.cuh"
#include "ops.cuh"

namespace {

struct Fwd {
  chg_ctx *ctx;
  chg_model *m;
  chg_graph *g;
  int train;                       // train-mode forward (activations kept for chg_backward)
  float *buf(const std::string &n, int64_t rows, int cols) {
    float *q = ctx->getf(n, (size_t)std::max<int64_t>(rows, 1) * cols);
    ctx->dbg[n] = {q, rows, cols, cols};
    return q;
  }
  GateLN ln(const std::string &pre) {
    return GateLN{m->p(pre + ".ln_core.g"), m->p(pre + ".ln_core.b"), m->p(pre + ".ln_gate.g"),
                  m->p(pre + ".ln_gate.b")};
  }
};

// Run f() on the ctx's second stream, forked from the library stream (the caller joins with
// join_side before consuming f's outputs).  Without a side stream f runs inline.
template <class Fn>
void on_side(chg_ctx *ctx, Fn &&f) {
  if (!ctx->concurrent()) { f(); return; }
  cudaStream_t main_stream = ctx->stream;
  CUDA_OK(cudaEventRecord(ctx->ev_fork, main_stream));
  CUDA_OK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
  ctx->forked = true;
  ctx->stream = ctx->side;
  try {
    f();
  } catch (...) {
    ctx->stream = main_stream;
    throw;
  }
  ctx->stream = main_stream;
  CUDA_OK(cudaEventRecord(ctx->ev_join, ctx->side));
}
void join_side(chg_ctx *ctx) {
  if (ctx->concurrent()) CUDA_OK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
  ctx->forked = false;
}

// First GatedMLP layer, factorised: the input rows are concatenations of per-atom,
// per-bond and per-row features, so x·W1 = Σ_parts part·W1[part rows]: the per-atom / per-bond
// products are computed once per atom / bond (P tables) and added by the per-row GEMM's
// epilogue through the gather indices — the per-row GEMM contracts only the row's own part
// (K = 64: e_ij for atom conv, a_ijk for bond conv / angle update).  Exact up to rounding order.
// P[rows, 64·nw] = X · [W_0[r_0:r_0+64] | W_1[r_1:r_1+64] | ...] (one 64-column chunk per weight
// block; r == nullptr: all blocks at row r0)
static void part_product(chg_ctx *ctx, const ASeg &x, int64_t rows, const float *const *W, int nw, int r0, float *P,
                         int ldP, const char *tag, const int *r = nullptr, const float *add = nullptr,
                         const int32_t *add_idx = nullptr) {
  if (rows <= 0) return;
  RowGemm G;
  G.A.seg[0] = x;
  G.A.nseg = 1;
  G.M = (int)rows; G.K = 64; G.nchunk = nw; G.tc = 1;
  for (int c = 0; c < nw; ++c) {
    G.ch[c] = chunk1(W[c] + (size_t)(r ? r[c] : r0) * 64, 64, 64, nullptr, P + 64 * c, ldP);
    if (add) {   // + add[add_idx[row]] (a per-atom product carried into a per-bond one)
      G.ch[c].gadd[0] = add + 64 * c; G.ch[c].gidx[0] = add_idx; G.ch[c].ldga[0] = ldP; G.ch[c].ngadd = 1;
    }
  }
  G.tag = tag;
  rowgemm(ctx, G);
}

// --- Atom Conv (Eq. 4) ------------------------------------------------------
void atom_conv_fwd(Fwd &F, int t, const float *v, const float *e, const float *ea, float *v_out) {
  chg_ctx *ctx = F.ctx;
  chg_model *m = F.m;
  chg_graph *g = F.g;
  const int64_t N = g->N, E = g->E;
  std::string pre = "atom" + std::to_string(t);
  float *z1 = F.buf("ac_z1_" + std::to_string(t), E, 128);
  float *y = F.buf("ac_y_" + std::to_string(t), E, 128);
  float *agg = F.buf("ac_agg_" + std::to_string(t), N, 64);
  float *msg = ctx->getf("msg_edge", std::max<int64_t>(E, 1) * 64);
  const float *W1c = m->p(pre + ".core.W1"), *W1g = m->p(pre + ".gate.W1");
  static const bool fact_full = getenv("CHG_FACT_FULL") != nullptr;   // A/B knob: both v parts as tables
  if (fact_full) {  // per atom: Pa = v · [W1c_i | W1g_i | W1c_j | W1g_j]  (rows 0..63: v_i part, 64..127: v_j part)
    float *Pa = ctx->getf(ctx->ws_name("ac_P"), (size_t)std::max<int64_t>(N, 1) * 256);
    const float *Wi[4] = {W1c, W1g, W1c, W1g};
    const int ri[4] = {0, 0, 64, 64};
    part_product(ctx, aseg(v, 64, 64), N, Wi, 4, 0, Pa, 256, "ac_P", ri);
    // per edge: z1 = e·W1[128:192] + b1 + Pa[i] (v_i part) + Pa[j] (v_j part)
    RowGemm G;
    G.A.seg[0] = aseg(e, 64, 64);
    G.A.nseg = 1;
    G.M = (int)E; G.K = 64; G.nchunk = 2; G.tc = 1;
    G.ch[0] = chunk1(W1c + 128 * 64, 64, 64, m->p(pre + ".core.b1"), z1, 128);
    G.ch[1] = chunk1(W1g + 128 * 64, 64, 64, m->p(pre + ".gate.b1"), z1 + 64, 128);
    for (int c = 0; c < 2; ++c) {
      Chunk &C = G.ch[c];
      C.gadd[0] = Pa + 64 * c; C.gidx[0] = g->center; C.ldga[0] = 256;
      C.gadd[1] = Pa + 128 + 64 * c; C.gidx[1] = g->nbr; C.ldga[1] = 256;
      C.ngadd = 2;
    }
    G.tag = "ac_f1";
    rowgemm(ctx, G);
  } else {  // per atom: Pa = v · [W1c_i | W1g_i] (the centre part: rows of one centre are contiguous
            // in the CSR edge order, so the epilogue's gathered addition is an L1 broadcast)
    float *Pa = ctx->getf(ctx->ws_name("ac_P"), (size_t)std::max<int64_t>(N, 1) * 128);
    const float *Wi[2] = {W1c, W1g};
    part_product(ctx, aseg(v, 64, 64), N, Wi, 2, 0, Pa, 128, "ac_P");
    // per edge: z1 = [e | v_j] · [W1[128:192] ; W1[64:128]] + b1 + Pa[i]: the neighbour rows (random
    // gathers) are A operand rows, loaded asynchronously by the loader warps
    RowGemm G;
    G.A.seg[0] = aseg(e, 64, 64);
    G.A.seg[1] = aseg(v, 64, 64, g->nbr, N);
    G.A.nseg = 2;
    G.M = (int)E; G.K = 128; G.nchunk = 2; G.tc = 1;
    const float *W1[2] = {W1c, W1g};
    const float *b1[2] = {m->p(pre + ".core.b1"), m->p(pre + ".gate.b1")};
    for (int c = 0; c < 2; ++c) {
      Chunk &C = G.ch[c];
      C = chunk1(W1[c] + 128 * 64, 64, 64, b1[c], z1 + 64 * c, 128);
      C.W[1] = W1[c] + 64 * 64; C.ldw[1] = 64;
      C.wk0[0] = 0; C.wk0[1] = 64; C.wk0[2] = 128; C.nwb = 2;
      C.gadd[0] = Pa + 64 * c; C.gidx[0] = g->center; C.ldga[0] = 128;
      C.ngadd = 1;
    }
    G.tag = "ac_f1";
    rowgemm(ctx, G);
  }
  {  // SiLU(z1) · blockdiag(W2_core, W2_gate) + b2
    RowGemm G;
    G.A.seg[0] = aseg(z1, 128, 128);
    G.A.nseg = 1; G.A.act = 1;
    G.M = (int)E; G.K = 64; G.nchunk = 2; G.tc = 1;
    G.ch[0] = chunk1(m->p(pre + ".core.W2"), 64, 64, m->p(pre + ".core.b2"), y, 128);
    G.ch[1] = chunk1(m->p(pre + ".gate.W2"), 64, 64, m->p(pre + ".gate.b2"), y + 64, 128);
    G.ch[1].a_k0 = 64;
    G.tag = "ac_f2";
    rowgemm(ctx, G);
  }
  // m_e = eᵃ_e ⊙ σ(LN_g(y_g)) ⊙ SiLU(LN_c(y_c))
  gate_fwd(ctx, E, y, 128, F.ln(pre), GATE_MUL_W, ea, nullptr, nullptr, nullptr, msg);
  // agg_i = Σ_{e at centre i} m_e and v' = v + agg · W_out + b_out in one pass
  SegSrc s;
  s.in = msg; s.ptr = g->row_ptr; s.rows = E;
  segsum_linear(ctx, N, 1, &s, agg, m->p(pre + ".out.W"), m->p(pre + ".out.b"), v, v_out, "segsum_ac");
}

// --- Bond Conv (Eq. 5) + Angle Update (Eq. 6) with Eq. 11 inputs ------------
// first-layer weights of the shared input [v_i, e_ij, e_ik, a_ijk] (Fig. 3a packing):
// bond core / gate hidden, angle core / gate (rows 0..63 v_i, 64..127 e_ij, 128..191 e_ik, 192..255 a)
static int bc_first_weights(chg_model *m, int t, bool angle_branch, const float **W, const float **b) {
  const std::string bp = "bond" + std::to_string(t), ap = "angle" + std::to_string(t);
  W[0] = m->p(bp + ".core.W1"); b[0] = m->p(bp + ".core.b1");
  W[1] = m->p(bp + ".gate.W1"); b[1] = m->p(bp + ".gate.b1");
  if (!angle_branch) return 2;
  W[2] = m->p(ap + ".core.W"); b[2] = m->p(ap + ".core.b");
  W[3] = m->p(ap + ".gate.W"); b[3] = m->p(ap + ".gate.b");
  return 4;
}

void bond_conv_fwd(Fwd &F, int t, bool angle_branch, const float *v, const float *e, const float *a, const float *eb,
                   float *e_out, float *a_out) {
  chg_ctx *ctx = F.ctx;
  chg_model *m = F.m;
  chg_graph *g = F.g;
  const int64_t N = g->N, E = g->E, B = g->B, A = g->A;
  std::string bp = "bond" + std::to_string(t), ap = "angle" + std::to_string(t), ts = std::to_string(t);
  float *z1 = F.buf("bc_z1_" + ts, A, 128);
  float *yb = F.buf("bc_yb_" + ts, A, 128);
  float *ya = angle_branch ? F.buf("bc_ya_" + ts, A, 128) : nullptr;
  float *aggb = F.buf("bc_aggb_" + ts, B, 64);
  float *q = ctx->getf("msg_angle", std::max<int64_t>(A, 1) * 64);
  if (A > 0) {
    const float *W[4], *bias[4];
    const int nw = bc_first_weights(m, t, angle_branch, W, bias);
    const int ldP = 64 * nw;
    // per atom (v_i part) and per bond (e_ij, e_ik parts) products of the packed first layers
    float *Pv = ctx->getf(ctx->ws_name("bc_Pv"), (size_t)std::max<int64_t>(N, 1) * ldP);
    float *P1 = ctx->getf(ctx->ws_name("bc_P1"), (size_t)std::max<int64_t>(B, 1) * ldP);
    part_product(ctx, aseg(v, 64, 64), N, W, nw, 0, Pv, ldP, "bc_P");
    // Q1[b] = e_b·W[64:128] + Pv[centre of b]: the v_i part rides on the first bond (the angles
    // of a first bond are contiguous, so the per-angle GEMM gathers Q1 with L1 reuse)
    part_product(ctx, aseg(e, 64, 64, g->bond_edge, E), B, W, nw, 64, P1, ldP, "bc_P", nullptr, Pv, g->bond_ctr);
    static const bool fact_full = getenv("CHG_FACT_FULL") != nullptr;   // A/B knob (atom_conv_fwd)
    RowGemm G;
    if (fact_full) {
      // per angle: [z1_bond | y_angle] = a·W[192:256] + b + Q1[b1] + P2[b2]
      float *P2 = ctx->getf(ctx->ws_name("bc_P2"), (size_t)std::max<int64_t>(B, 1) * ldP);
      part_product(ctx, aseg(e, 64, 64, g->bond_edge, E), B, W, nw, 128, P2, ldP, "bc_P");
      G.A.seg[0] = aseg(a, 64, 64);
      G.A.nseg = 1;
      G.M = (int)A; G.K = 64; G.nchunk = nw; G.tc = 1;
      for (int c = 0; c < nw; ++c) {
        float *dst = c < 2 ? z1 + 64 * c : ya + 64 * (c - 2);
        G.ch[c] = chunk1(W[c] + 192 * 64, 64, 64, bias[c], dst, 128);
        Chunk &C = G.ch[c];
        C.gadd[0] = P1 + 64 * c; C.gidx[0] = g->angle_b1; C.ldga[0] = ldP;
        C.gadd[1] = P2 + 64 * c; C.gidx[1] = g->angle_b2; C.ldga[1] = ldP;
        C.ngadd = 2;
      }
    } else {
      // per angle: [z1_bond | y_angle] = [a | e_ik] · [W[192:256] ; W[128:192]] + b + Q1[b1]: the
      // second bond's edge rows (random gathers) are A operand rows, loaded by the loader warps
      G.A.seg[0] = aseg(a, 64, 64);
      G.A.seg[1] = aseg(e, 64, 64, g->angle_e2, E);
      G.A.nseg = 2;
      G.M = (int)A; G.K = 128; G.nchunk = nw; G.tc = 1;
      for (int c = 0; c < nw; ++c) {
        float *dst = c < 2 ? z1 + 64 * c : ya + 64 * (c - 2);
        G.ch[c] = chunk1(W[c] + 192 * 64, 64, 64, bias[c], dst, 128);
        Chunk &C = G.ch[c];
        C.W[1] = W[c] + 128 * 64; C.ldw[1] = 64;
        C.wk0[0] = 0; C.wk0[1] = 64; C.wk0[2] = 128; C.nwb = 2;
        C.gadd[0] = P1 + 64 * c; C.gidx[0] = g->angle_b1; C.ldga[0] = ldP;
        C.ngadd = 1;
      }
    }
    G.tag = "bc_f1";
    rowgemm(ctx, G);
    RowGemm H;
    H.A.seg[0] = aseg(z1, 128, 128);
    H.A.nseg = 1; H.A.act = 1;
    H.M = (int)A; H.K = 64; H.nchunk = 2; H.tc = 1;
    H.ch[0] = chunk1(m->p(bp + ".core.W2"), 64, 64, m->p(bp + ".core.b2"), yb, 128);
    H.ch[1] = chunk1(m->p(bp + ".gate.W2"), 64, 64, m->p(bp + ".gate.b2"), yb + 64, 128);
    H.ch[1].a_k0 = 64;
    H.tag = "bc_f2";
    rowgemm(ctx, H);
    // q = eᵇ_ij ⊙ eᵇ_ik ⊙ φ_e
    gate_fwd(ctx, A, yb, 128, F.ln(bp), GATE_MUL_W1W2, eb, g->angle_b1, g->angle_b2, nullptr, q);
  }
  {  // e' = e + 𝓛_e(agg) on all E edges (Q16): agg = Σ over the angles whose first bond is the
     // edge's bond (empty for non-bond edges -> bias only); aggb (per bond) kept for the backward
    SegSrc s;
    s.in = q; s.ptr = g->angle_ptr; s.segmap = g->bond_id; s.rows = A;
    segsum_linear(ctx, E, 1, &s, aggb, m->p(bp + ".out.W"), m->p(bp + ".out.b"), e, e_out, "segsum_bc", 1);
  }
  if (angle_branch && A > 0)   // a' = a + φ_a
    gate_fwd(ctx, A, ya, 128, F.ln(ap), GATE_RESID, nullptr, nullptr, nullptr, a, a_out);
}

// --- MLP heads: hidden layers Linear+SiLU, last Linear (fused, head_mlp.cu) --------
void mlp_fwd(Fwd &F, const std::string &pre, int nl, const float *x, int64_t rows, int nout, float *out, int ldo) {
  float *Z[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k + 1 < nl; ++k) Z[k] = F.buf(pre + "_z" + std::to_string(k), rows, 64);
  head_mlp_fwd(F.ctx, nl, nout, x, rows, F.m->p(pre + ".W0"), Z, out, ldo);
}

void copy_out(chg_ctx *ctx, float *dst, const float *src, int64_t n, int on_device) {
  if (!dst || n <= 0) return;
  CUDA_OK(cudaMemcpyAsync(dst, src, 4 * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                          ctx->stream));
}

}  // namespace

void forward_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, int train, chg_pred *out) {
  Fwd F{ctx, m, g, train};
  const int64_t N = g->N, E = g->E, B = g->B, A = g->A;
  const int T = m->cfg.n_bond_conv;
  const int p = m->cfg.envelope_p;
  ctx->dbg.clear();
  ctx->fwd_train = false;
  ctx->set_precision(m->cfg.mlp_precision);
  ctx->cur_model = m;
  ctx->cur_wt = nullptr;
  if (ctx->use_tc) {   // K-major weight copy for the tensor-core operands
    if (!m->wt) CUDA_OK(cudaMalloc(&m->wt, 4 * (size_t)std::max<int64_t>(m->P, 1)));   // per model: images cache its addresses
    float *wt = m->wt;
    transpose_params(ctx, m, wt);
    ctx->cur_wt = wt;
    tc_repack_all(ctx, m);
  }
  // A2 + A3: fused basis expansion and projection (Eq. 2; no bias, Q5); the bases (and
  // ∂basis/∂f in train mode) are saved for the backward
  float *ea_t = F.buf("ea_t", E, 32), *eb_t = F.buf("eb_t", B, 32), *a_t = F.buf("a_t", A, 32);
  float *ea_g = train ? F.buf("ea_g", E, 32) : nullptr, *eb_g = train ? F.buf("eb_g", B, 32) : nullptr;
  std::vector<float *> v(T + 2), e(T + 1), a(T);
  v[0] = F.buf("v0", N, 64);
  embed_fwd(ctx, N, g->species, m->p("embed.W"), v[0]);
  e[0] = F.buf("e0", E, 64);
  float *ea = F.buf("ea", E, 64), *eb = F.buf("eb", B, 64);
  a[0] = F.buf("a0", A, 64);
  proj_radial_fwd(ctx, E, g->vec64, nullptr, m->p("rbf_a.freq"), g->r_atom, p, m->p("proj.W0"), m->p("proj.Wa"),
                  e[0], ea, ea_t, ea_g);
  proj_radial_fwd(ctx, B, g->vec64, g->bond_edge, m->p("rbf_b.freq"), g->r_bond, p, m->p("proj.Wb"), nullptr, eb,
                  nullptr, eb_t, eb_g);
  proj_angle_fwd(ctx, A, g->vec64, g->angle_e1, g->angle_e2, m->p("proj.Wtheta"), a[0], a_t);
  // A4/A5 interaction blocks
  // Eq. 11: atom conv (writes v^{t+1}) and bond conv + angle update (write e^{t+1}, a^{t+1})
  // of a layer read only layer-t features, so they run concurrently: the bond branch on a
  // second stream forked from / joined into the library stream (CHG_SERIAL=1 disables)
  static const bool serial = getenv("CHG_SERIAL") != nullptr;
  if (!serial && !ctx->side) {
    CUDA_OK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  for (int t = 0; t < T; ++t) {
    v[t + 1] = F.buf("v" + std::to_string(t + 1), N, 64);
    e[t + 1] = F.buf("e" + std::to_string(t + 1), E, 64);
    bool ab = t + 1 < T;
    if (ab) a[t + 1] = F.buf("a" + std::to_string(t + 1), A, 64);
    if (!ctx->concurrent()) {
      atom_conv_fwd(F, t, v[t], e[t], ea, v[t + 1]);
      bond_conv_fwd(F, t, ab, v[t], e[t], a[t], eb, e[t + 1], ab ? a[t + 1] : nullptr);
      continue;
    }
    cudaStream_t main_stream = ctx->stream;
    CUDA_OK(cudaEventRecord(ctx->ev_fork, main_stream));
    CUDA_OK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    ctx->forked = true;
    ctx->stream = ctx->side;
    try {
      bond_conv_fwd(F, t, ab, v[t], e[t], a[t], eb, e[t + 1], ab ? a[t + 1] : nullptr);
    } catch (...) {
      ctx->stream = main_stream;
      throw;
    }
    ctx->stream = main_stream;
    CUDA_OK(cudaEventRecord(ctx->ev_join, ctx->side));
    atom_conv_fwd(F, t, v[t], e[t], ea, v[t + 1]);
    CUDA_OK(cudaStreamWaitEvent(main_stream, ctx->ev_join, 0));
    ctx->forked = false;
  }
  v[T + 1] = F.buf("v" + std::to_string(T + 1), N, 64);
  // A6 heads: the force head reads e^T only, so it runs beside the final atom conv
  float *vf = v[T + 1], *ef = e[T];
  float *e_atom = F.buf("e_atom", N, 1), *mag = F.buf("magmom", N, 1), *n_e = F.buf("n_e", E, 1);
  float *M9 = F.buf("M9", N, 9);
  float *Zf[2] = {F.buf("head_F_z0", E, 64), F.buf("head_F_z1", E, 64)};
  on_side(ctx, [&] { head_mlp_fwd(ctx, 3, 1, ef, E, m->p("head_F.W0"), Zf, n_e, 1); });
  atom_conv_fwd(F, T, v[T], e[T], ea, v[T + 1]);
  mlp_fwd(F, "head_E", 4, vf, N, 1, e_atom, 1);
  {
    RowGemm G;
    G.A.seg[0] = aseg(vf, 64, 64);
    G.A.nseg = 1;
    G.M = (int)N; G.K = 64;
    G.ch[0] = chunk1(m->p("head_M.W"), 1, 64, m->p("head_M.b"), mag, 1, 1);
    G.tag = "headM_f";
    rowgemm(ctx, G);
  }
  mlp_fwd(F, "head_S", 3, vf, N, 9, M9, 9);
  join_side(ctx);
  float *energy = F.buf("energy", g->S, 1), *epa = F.buf("energy_per_atom", g->S, 1);
  float *forces = F.buf("forces", N, 3), *stress = F.buf("stress", g->S, 9);
  heads_forces(ctx, g, n_e, forces);
  heads_struct(ctx, g, e_atom, M9, energy, epa, stress);
  if (out) {
    copy_out(ctx, out->energy, energy, g->S, out->on_device);
    copy_out(ctx, out->energy_per_atom, epa, g->S, out->on_device);
    copy_out(ctx, out->forces, forces, 3 * N, out->on_device);
    copy_out(ctx, out->stress, stress, 9 * (int64_t)g->S, out->on_device);
    copy_out(ctx, out->magmom, mag, N, out->on_device);
    if (!out->on_device) CUDA_OK(cudaStreamSynchronize(ctx->stream));
  }
  ctx->fwd_graph = g;
  ctx->fwd_graph_id = g->id;
  ctx->fwd_train = train != 0;
}

// ===========================================================================
// backward
// ===========================================================================
namespace {

struct Bwd {
  chg_ctx *ctx;
  chg_model *m;
  chg_graph *g;
  float *wt;   // transposed copy of every 2-D weight at its own flat offset
  const float *WT(const std::string &n) const { return wt + m->off(n); }
  float *G(const std::string &n) const { return m->g(n); }
  const float *act(const std::string &n) const {
    auto it = ctx->dbg.find(n);
    if (it == ctx->dbg.end()) CHG_THROW(CHG_ERR_STATE, "missing forward activation %s", n.c_str());
    return it->second.p;
  }
  GateLN ln(const std::string &pre) const {
    return GateLN{m->p(pre + ".ln_core.g"), m->p(pre + ".ln_core.b"), m->p(pre + ".ln_gate.g"),
                  m->p(pre + ".ln_gate.b")};
  }
  GateLNGrad lng(const std::string &pre) const {
    return GateLNGrad{G(pre + ".ln_core.g"), G(pre + ".ln_core.b"), G(pre + ".ln_gate.g"), G(pre + ".ln_gate.b")};
  }
  float *scratch(const char *n, int64_t rows, int cols) {
    return ctx->getf(n, (size_t)std::max<int64_t>(rows, 1) * cols);
  }
};

// dx accumulation and parameter gradients through an MLP head (fused, head_mlp.cu)
void mlp_bwd(Bwd &Bw, const std::string &pre, int nl, const float *x, int64_t rows, const float *dout, int nout,
             float *dx) {
  float *Z[3] = {nullptr, nullptr, nullptr};
  for (int k = 0; k + 1 < nl; ++k) Z[k] = const_cast<float *>(Bw.act(pre + "_z" + std::to_string(k)));
  head_mlp_bwd(Bw.ctx, nl, nout, x, rows, Bw.m->p(pre + ".W0"), Z, dout, Bw.G(pre + ".W0"), dx);
}

// contributions of the output linear of atom conv t: dagg = dv · W_outᵀ, dW_out, db_out
void ac_bwd_head(Bwd &Bw, int t, const float *dv, float *dagg) {
  chg_graph *g = Bw.g;
  std::string pre = "atom" + std::to_string(t);
  const float *agg = Bw.act("ac_agg_" + std::to_string(t));
  RowGemm G;
  G.A.seg[0] = aseg(dv, 64, 64);
  G.A.nseg = 1;
  G.M = (int)g->N; G.K = 64;
  G.ch[0] = chunk1(Bw.WT(pre + ".out.W"), 64, 64, nullptr, dagg, 64);
  G.tag = "ac_dagg";
  rowgemm(Bw.ctx, G);
  WGrad wg;
  wg.A.seg[0] = aseg(agg, 64, 64);
  wg.A.nseg = 1;
  wg.M = (int)g->N; wg.K = 64;
  wg.D = dv; wg.ldd = 64; wg.N = 64; wg.bias = 1;
  wg.dst[0].W = Bw.G(pre + ".out.W"); wg.dst[0].ldw = 64; wg.dst[0].b = Bw.G(pre + ".out.b");
  wg.tag = "ac_out_wg";
  wgrad(Bw.ctx, wg);
}

void bc_bwd_head(Bwd &Bw, int t, const float *de, float *daggb) {
  chg_graph *g = Bw.g;
  std::string pre = "bond" + std::to_string(t);
  const float *aggb = Bw.act("bc_aggb_" + std::to_string(t));
  RowGemm G;
  G.A.seg[0] = aseg(de, 64, 64, g->bond_edge, g->E);
  G.A.nseg = 1;
  G.M = (int)g->B; G.K = 64;
  G.ch[0] = chunk1(Bw.WT(pre + ".out.W"), 64, 64, nullptr, daggb, 64);
  G.tag = "bc_daggb";
  rowgemm(Bw.ctx, G);
  WGrad wg;   // dW_out = aggbᵀ · de[bond_edge] (non-bond rows of agg are zero)
  wg.A.seg[0] = aseg(aggb, 64, 64);
  wg.A.nseg = 1;
  wg.M = (int)g->B; wg.K = 64;
  wg.D = de; wg.didx = g->bond_edge; wg.ldd = 64; wg.N = 64; wg.bias = 0;
  wg.dst[0].W = Bw.G(pre + ".out.W"); wg.dst[0].ldw = 64;
  wg.tag = "bc_out_wg";
  wgrad(Bw.ctx, wg);
  colsum(Bw.ctx, g->E, de, Bw.G(pre + ".out.b"));   // db_out = Σ over ALL edges of de
}

// Backward of the factorised first layer.  With z = Σ_parts x_part·W1[part] the
// per-row adjoint dZ (the GatedMLP's layer-1 pre-activation gradient) gives
//   d(own part)  = dZ · W1[own]ᵀ                        (per-row GEMM, K = width of dZ, N = 64)
//   d(part p)    = (Σ_{rows using index i in part p} dZ) · W1[p]ᵀ  (segmented sums, then per-atom /
//                   per-bond GEMMs; the gather adjoints follow the CSR / rev / swap orders: no atomics)
//   dW1[part p]  = Σ_i x_p,iᵀ · (Σ_{rows of i} dZ)             (weight gradients over atoms / bonds)
void ac_bwd_body(Bwd &Bw, int t, const float *v, const float *e, const float *ea, const float *dagg, float *dv,
                 float *de, float *dea) {
  chg_ctx *ctx = Bw.ctx;
  chg_graph *g = Bw.g;
  const int64_t N = g->N, E = g->E;
  std::string pre = "atom" + std::to_string(t), ts = std::to_string(t);
  const float *z1 = Bw.act("ac_z1_" + ts), *y = Bw.act("ac_y_" + ts);
  float *dY = Bw.scratch("ac_dY", E, 128), *dZ = Bw.scratch("ac_dZ", E, 128);
  float *S = Bw.scratch("ac_S", N, 256);
  gate_bwd(ctx, E, y, 128, Bw.ln(pre), GATE_MUL_W, ea, nullptr, nullptr, dagg, g->center, dY, 128, dea, nullptr,
           nullptr, Bw.lng(pre));
  {  // dZ1 = (dY · blockdiag(W2ᵀ)) ⊙ SiLU'(z1)
    RowGemm G;
    G.A.seg[0] = aseg(dY, 128, 128);
    G.A.nseg = 1; G.A.rounded = ctx->tc_round();       // gate_bwd rounds dY in TF32 mode
    G.M = (int)E; G.K = 64; G.nchunk = 2; G.tc = 1;
    G.ch[0] = chunk1(Bw.WT(pre + ".core.W2"), 64, 64, nullptr, dZ, 128);
    G.ch[0].mul = z1; G.ch[0].ldm = 128; G.ch[0].round_out = ctx->tc_round();
    G.ch[1] = chunk1(Bw.WT(pre + ".gate.W2"), 64, 64, nullptr, dZ + 64, 128);
    G.ch[1].mul = z1 + 64; G.ch[1].ldm = 128; G.ch[1].a_k0 = 64; G.ch[1].round_out = ctx->tc_round();
    G.tag = "ac_dZ";
    rowgemm(ctx, G);
  }
  if (ctx->use_tc) {  // dW2, db2 of both branches in one K = N = 128 launch (diagonal blocks kept)
    WGrad wg;
    wg.A.seg[0] = aseg(z1, 128, 128);
    wg.A.nseg = 1; wg.A.act = 1;
    wg.M = (int)E; wg.K = 128; wg.tc = 1;
    wg.D = dY; wg.ldd = 128; wg.N = 128; wg.bias = 1;
    wg.dst[0].W = Bw.G(pre + ".core.W2"); wg.dst[0].ldw = 64; wg.dst[0].b = Bw.G(pre + ".core.b2");
    wg.dst[0].k0 = 0; wg.dst[0].kn = 64;
    wg.dst[1].W = Bw.G(pre + ".gate.W2"); wg.dst[1].ldw = 64; wg.dst[1].b = Bw.G(pre + ".gate.b2");
    wg.dst[1].k0 = 64; wg.dst[1].kn = 64;
    wg.tag = "ac_W2_wg";
    wgrad(ctx, wg);
  } else for (int br = 0; br < 2; ++br) {  // dW2, db2
    const char *b = br ? ".gate" : ".core";
    WGrad wg;
    wg.A.seg[0] = aseg(z1 + 64 * br, 128, 64);
    wg.A.nseg = 1; wg.A.act = 1;
    wg.M = (int)E; wg.K = 64; wg.tc = 1;
    wg.D = dY + 64 * br; wg.ldd = 128; wg.N = 64; wg.bias = 1;
    wg.dst[0].W = Bw.G(pre + b + ".W2"); wg.dst[0].ldw = 64; wg.dst[0].b = Bw.G(pre + b + ".b2");
    wg.tag = "ac_W2_wg";
    wgrad(ctx, wg);
  }
  {  // de += dZ1 · [W1_core[128:192]ᵀ ; W1_gate[128:192]ᵀ]  (the row's own part e_ij)
    RowGemm G;
    G.A.seg[0] = aseg(dZ, 128, 128);
    G.A.nseg = 1; G.A.rounded = ctx->tc_round();
    G.M = (int)E; G.K = 128; G.nchunk = 1; G.tc = 1;
    Chunk &C = G.ch[0];
    C.W[0] = Bw.WT(pre + ".core.W1") + 128; C.ldw[0] = 192;
    C.W[1] = Bw.WT(pre + ".gate.W1") + 128; C.ldw[1] = 192;
    C.wk0[0] = 0; C.wk0[1] = 64; C.wk0[2] = 128; C.nwb = 2;
    C.out = de; C.ldo = 64; C.resid = de; C.ldr = 64;
    G.tag = "ac_dX";
    rowgemm(ctx, G);
  }
  {  // S_i = Σ_{e: centre i} dZ_e (CSR rows), S_j = Σ_{e: neighbour j} dZ_e (rows of j through rev):
     // one launch, each source into its own half of S
    SegSrc s[2];
    s[0].in = dZ; s[0].ld = 128; s[0].ptr = g->row_ptr; s[0].rows = E;
    s[1] = s[0]; s[1].perm = g->rev;
    const int off[2] = {0, 128};
    segsum(ctx, N, S, 256, 0, 2, s, "segsum_ac_S", 128, off);
  }
  {  // dW1: e part over edges (with db1), v_i / v_j parts over atoms
    WGrad wg;
    wg.A.seg[0] = aseg(e, 64, 64);
    wg.A.nseg = 1;
    wg.M = (int)E; wg.K = 64; wg.tc = 1;
    wg.D = dZ; wg.ldd = 128; wg.N = 128; wg.bias = 1;
    wg.dst[0].W = Bw.G(pre + ".core.W1") + 128 * 64; wg.dst[0].ldw = 64; wg.dst[0].b = Bw.G(pre + ".core.b1");
    wg.dst[1].W = Bw.G(pre + ".gate.W1") + 128 * 64; wg.dst[1].ldw = 64; wg.dst[1].b = Bw.G(pre + ".gate.b1");
    wg.tag = "ac_W1_wg";
    wgrad(ctx, wg);
    WGrad wv;
    wv.A.seg[0] = aseg(v, 64, 64);
    wv.A.nseg = 1;
    wv.M = (int)N; wv.K = 64; wv.tc = 1;
    wv.D = S; wv.ldd = 256; wv.N = 256; wv.bias = 0;
    wv.dst[0].W = Bw.G(pre + ".core.W1"); wv.dst[0].ldw = 64;
    wv.dst[1].W = Bw.G(pre + ".gate.W1"); wv.dst[1].ldw = 64;
    wv.dst[2].W = Bw.G(pre + ".core.W1") + 64 * 64; wv.dst[2].ldw = 64;
    wv.dst[3].W = Bw.G(pre + ".gate.W1") + 64 * 64; wv.dst[3].ldw = 64;
    wv.tag = "ac_W1v_wg";
    wgrad(ctx, wv);
  }
  {  // dv += [S_i | S_j] · [W1_c[0:64]ᵀ ; W1_g[0:64]ᵀ ; W1_c[64:128]ᵀ ; W1_g[64:128]ᵀ]
    RowGemm G;
    G.A.seg[0] = aseg(S, 256, 256);
    G.A.nseg = 1;
    G.M = (int)N; G.K = 256; G.nchunk = 1; G.tc = 1;
    Chunk &C = G.ch[0];
    C.W[0] = Bw.WT(pre + ".core.W1"); C.ldw[0] = 192;
    C.W[1] = Bw.WT(pre + ".gate.W1"); C.ldw[1] = 192;
    C.W[2] = Bw.WT(pre + ".core.W1") + 64; C.ldw[2] = 192;
    C.W[3] = Bw.WT(pre + ".gate.W1") + 64; C.ldw[3] = 192;
    C.wk0[0] = 0; C.wk0[1] = 64; C.wk0[2] = 128; C.wk0[3] = 192; C.wk0[4] = 256; C.nwb = 4;
    C.out = dv; C.ldo = 64; C.resid = dv; C.ldr = 64;
    G.tag = "ac_dvS";
    rowgemm(ctx, G);
  }
}

// phase 1: everything that touches neither dv nor de (may run concurrently with ac_bwd_body);
// phase 2: the dv / de updates (after the atom conv's updates, fixed order)
void bc_bwd_body(Bwd &Bw, int t, bool angle_branch, const float *v, const float *e, const float *a, const float *eb,
                 const float *daggb, float *dv, float *de, float *da, float *deb, int phase) {
  chg_ctx *ctx = Bw.ctx;
  chg_graph *g = Bw.g;
  const int64_t N = g->N, E = g->E, B = g->B, A = g->A;
  if (A == 0) return;
  std::string bp = "bond" + std::to_string(t), ap = "angle" + std::to_string(t), ts = std::to_string(t);
  const float *W[4], *bias[4];
  const int nw = bc_first_weights(Bw.m, t, angle_branch, W, bias);
  const int Kx = 64 * nw;                           // width of dZ used: bond hidden (+ angle pre-LN)
  float *S1 = Bw.scratch("bc_S12", B, 512), *S2 = S1 + 256, *Sv = Bw.scratch("bc_Sv", N, 256);
  float *tb = Bw.scratch("bc_tb", B, 64);
  auto WTp = [&](int c) { return Bw.WT(c < 2 ? bp + (c ? ".gate.W1" : ".core.W1") : ap + (c == 3 ? ".gate.W" : ".core.W")); };
  auto Gp = [&](int c) { return Bw.G(c < 2 ? bp + (c ? ".gate.W1" : ".core.W1") : ap + (c == 3 ? ".gate.W" : ".core.W")); };
  // d(part) GEMM: out (+)= Src · [W_c[r0:r0+64]ᵀ]_c   (Src [rows, Kx], ld 256)
  auto part_adjoint = [&](const float *Src, int lds, int64_t rows, int r0, float *out, bool accumulate, const char *tag) {
    if (rows <= 0) return;
    RowGemm G;
    G.A.seg[0] = aseg(Src, lds, Kx);
    G.A.nseg = 1;                                    // fp32 sums (not TF32-rounded)
    G.M = (int)rows; G.K = Kx; G.nchunk = 1; G.tc = 1;
    Chunk &C = G.ch[0];
    for (int c = 0; c < nw; ++c) { C.W[c] = WTp(c) + r0; C.ldw[c] = 256; C.wk0[c] = 64 * c; }
    C.wk0[nw] = Kx; C.nwb = nw;
    C.out = out; C.ldo = 64;
    if (accumulate) { C.resid = out; C.ldr = 64; }
    G.tag = tag;
    rowgemm(ctx, G);
  };
  if (phase == 2) {
    part_adjoint(Sv, 256, N, 0, dv, true, "bc_dvS");                 // v_i part
    if (B > 0) {  // e_ij (first bond) and e_ik (second bond) parts: tb = [S1 | S2] · [W[64:128]ᵀ ; W[128:192]ᵀ]
      RowGemm G;
      G.A.seg[0] = aseg(S1, 512, Kx);
      G.A.seg[1] = aseg(S2, 512, Kx);
      G.A.nseg = 2;
      G.M = (int)B; G.K = 2 * Kx; G.nchunk = 1; G.tc = 1;
      Chunk &C = G.ch[0];
      for (int c = 0; c < nw; ++c) {
        C.W[c] = WTp(c) + 64; C.ldw[c] = 256; C.wk0[c] = 64 * c;
        C.W[nw + c] = WTp(c) + 128; C.ldw[nw + c] = 256; C.wk0[nw + c] = Kx + 64 * c;
      }
      C.wk0[2 * nw] = 2 * Kx; C.nwb = 2 * nw;
      C.out = tb; C.ldo = 64;
      G.tag = "bc_deS";
      rowgemm(ctx, G);
    }
    rows_add(ctx, B, g->bond_edge, tb, de);                          // bond rows -> their edges
    return;
  }
  const float *z1 = Bw.act("bc_z1_" + ts), *yb = Bw.act("bc_yb_" + ts);
  float *dYb = Bw.scratch("bc_dYb", A, 128), *dZ = Bw.scratch("bc_dZ", A, 256);
  float *q1 = Bw.scratch("bc_q1", A, 64), *q2 = Bw.scratch("bc_q2", A, 64);
  gate_bwd(ctx, A, yb, 128, Bw.ln(bp), GATE_MUL_W1W2, eb, g->angle_b1, g->angle_b2, daggb, g->angle_b1, dYb, 128,
           nullptr, q1, q2, Bw.lng(bp));
  if (angle_branch)
    gate_bwd(ctx, A, Bw.act("bc_ya_" + ts), 128, Bw.ln(ap), GATE_RESID, nullptr, nullptr, nullptr, da, nullptr,
             dZ + 128, 256, nullptr, nullptr, nullptr, Bw.lng(ap));
  {
    RowGemm G;
    G.A.seg[0] = aseg(dYb, 128, 128);
    G.A.nseg = 1; G.A.rounded = ctx->tc_round();
    G.M = (int)A; G.K = 64; G.nchunk = 2; G.tc = 1;
    G.ch[0] = chunk1(Bw.WT(bp + ".core.W2"), 64, 64, nullptr, dZ, 256);
    G.ch[0].mul = z1; G.ch[0].ldm = 128; G.ch[0].round_out = ctx->tc_round();
    G.ch[1] = chunk1(Bw.WT(bp + ".gate.W2"), 64, 64, nullptr, dZ + 64, 256);
    G.ch[1].mul = z1 + 64; G.ch[1].ldm = 128; G.ch[1].a_k0 = 64; G.ch[1].round_out = ctx->tc_round();
    G.tag = "bc_dZ";
    rowgemm(ctx, G);
  }
  if (ctx->use_tc) {  // dW2, db2 of both branches in one K = N = 128 launch (diagonal blocks kept)
    WGrad wg;
    wg.A.seg[0] = aseg(z1, 128, 128);
    wg.A.nseg = 1; wg.A.act = 1;
    wg.M = (int)A; wg.K = 128; wg.tc = 1;
    wg.D = dYb; wg.ldd = 128; wg.N = 128; wg.bias = 1;
    wg.dst[0].W = Bw.G(bp + ".core.W2"); wg.dst[0].ldw = 64; wg.dst[0].b = Bw.G(bp + ".core.b2");
    wg.dst[0].k0 = 0; wg.dst[0].kn = 64;
    wg.dst[1].W = Bw.G(bp + ".gate.W2"); wg.dst[1].ldw = 64; wg.dst[1].b = Bw.G(bp + ".gate.b2");
    wg.dst[1].k0 = 64; wg.dst[1].kn = 64;
    wg.tag = "bc_W2_wg";
    wgrad(ctx, wg);
  } else for (int br = 0; br < 2; ++br) {
    const char *b = br ? ".gate" : ".core";
    WGrad wg;
    wg.A.seg[0] = aseg(z1 + 64 * br, 128, 64);
    wg.A.nseg = 1; wg.A.act = 1;
    wg.M = (int)A; wg.K = 64; wg.tc = 1;
    wg.D = dYb + 64 * br; wg.ldd = 128; wg.N = 64; wg.bias = 1;
    wg.dst[0].W = Bw.G(bp + b + ".W2"); wg.dst[0].ldw = 64; wg.dst[0].b = Bw.G(bp + b + ".b2");
    wg.tag = "bc_W2_wg";
    wgrad(ctx, wg);
  }
  // da += [dZ1_bond | dY_angle] · [W_c[192:256]ᵀ]_c   (the row's own part a_ijk)
  {
    RowGemm G;
    G.A.seg[0] = aseg(dZ, 256, Kx);
    G.A.nseg = 1; G.A.rounded = ctx->tc_round();
    G.M = (int)A; G.K = Kx; G.nchunk = 1; G.tc = 1;
    Chunk &C = G.ch[0];
    for (int c = 0; c < nw; ++c) { C.W[c] = WTp(c) + 192; C.ldw[c] = 256; C.wk0[c] = 64 * c; }
    C.wk0[nw] = Kx; C.nwb = nw;
    C.out = da; C.ldo = 64; C.resid = da; C.ldr = 64;
    G.tag = "bc_dX";
    rowgemm(ctx, G);
  }
  {  // S1[b] = Σ_{angles with first bond b} dZ, S2[b] = Σ_{angles with second bond b} dZ (swap
     // order), Sv[i] = Σ_{bonds b at centre i} S1[b]
    SegSrc s[2];
    s[0].in = dZ; s[0].ld = 256; s[0].ptr = g->angle_ptr; s[0].rows = A;
    s[1] = s[0]; s[1].perm = g->swap;
    const int off[2] = {0, 256};                       // S1 | S2 rows of one [B, 512] table, one launch
    segsum(ctx, B, S1, 512, 0, 2, s, "segsum_bc_S", Kx, off);
    SegSrc u;
    u.in = S1; u.ld = 512; u.ptr = g->bond_ptr; u.rows = B;
    segsum(ctx, N, Sv, 256, 0, 1, &u, "segsum_bc_S", Kx);
  }
  {  // dW (bond W1 and angle W): a part over angles (with the biases), v / e_ij / e_ik parts over
     // atoms and bonds
    auto wpart = [&](const ASeg &x, int64_t rows, const float *D, int ldd, int r0, int with_bias, const char *tag) {
      if (rows <= 0) return;
      WGrad wg;
      wg.A.seg[0] = x;
      wg.A.nseg = 1;
      wg.M = (int)rows; wg.K = 64; wg.tc = 1;
      wg.D = D; wg.ldd = ldd; wg.N = Kx; wg.bias = with_bias;
      for (int c = 0; c < nw; ++c) {
        wg.dst[c].W = Gp(c) + (size_t)r0 * 64; wg.dst[c].ldw = 64;
        if (with_bias) wg.dst[c].b = Bw.G(c < 2 ? bp + (c ? ".gate.b1" : ".core.b1") : ap + (c == 3 ? ".gate.b" : ".core.b"));
      }
      wg.tag = tag;
      wgrad(ctx, wg);
    };
    wpart(aseg(a, 64, 64), A, dZ, 256, 192, 1, "bc_W1_wg");
    wpart(aseg(v, 64, 64), N, Sv, 256, 0, 0, "bc_W1p_wg");
    wpart(aseg(e, 64, 64, g->bond_edge, E), B, S1, 512, 64, 0, "bc_W1p_wg");
    wpart(aseg(e, 64, 64, g->bond_edge, E), B, S2, 512, 128, 0, "bc_W1p_wg");
  }
  SegSrc s[2];
  s[0] = SegSrc(); s[0].in = q1; s[0].ptr = g->angle_ptr; s[0].rows = A;
  s[1] = SegSrc(); s[1].in = q2; s[1].ptr = g->angle_ptr; s[1].perm = g->swap; s[1].rows = A;
  segsum(ctx, B, deb, 64, 1, 2, s, "segsum_bc_deb");
}

const float *labels_dev(chg_ctx *ctx, const void *p, size_t bytes, const char *name, int on_device) {
  if (on_device || !p) return (const float *)p;   // NULL = task skipped
  void *d = ctx->get(name, bytes);
  if (bytes) CUDA_OK(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return (const float *)d;
}

}  // namespace

// NEXT-3 ("perform all-reduce once after the gradient calculation of a part of parameters
// is completed"): the flat gradient ranges of the parameter groups whose gradients are final are
// summed over the ranks on the comm stream while the backward of the earlier layers continues.
// Groups are contiguous ranges of the canonical layout (prefix match: "atom2.", "bond2.", ...).
static std::pair<int64_t, int64_t> group_range(const chg_model *m, const std::vector<std::string> &prefixes) {
  int64_t lo = -1, hi = -1;
  for (size_t t = 0; t < m->names.size(); ++t) {
    bool in = false;
    for (auto &p : prefixes) in |= m->names[t].compare(0, p.size(), p) == 0;
    if (!in) continue;
    const int64_t end = t + 1 < m->names.size() ? m->offsets[t + 1] : m->P;
    if (lo < 0) lo = m->offsets[t];
    else if (m->offsets[t] != hi) CHG_THROW(CHG_ERR_STATE, "gradient bucket %s is not contiguous", prefixes[0].c_str());
    hi = end;
  }
  return {lo, hi};
}

static void grad_bucket(chg_ctx *ctx, chg_model *m, const std::vector<std::vector<std::string>> &groups) {
  if (!ctx->grad_overlap || !ctx->nccl_comm || ctx->nranks <= 1 || ctx->no_param_grads) return;
  if (!ctx->comm) {
    CUDA_OK(cudaStreamCreateWithFlags(&ctx->comm, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_comm_in, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ctx->ev_comm_done, cudaEventDisableTiming));
  }
  CUDA_OK(cudaEventRecord(ctx->ev_comm_in, ctx->stream));        // the group's reductions are queued
  CUDA_OK(cudaStreamWaitEvent(ctx->comm, ctx->ev_comm_in, 0));
  ncclGroupStart();
  for (auto &g : groups) {
    auto r = group_range(m, g);
    if (r.first < 0 || r.second <= r.first) continue;
    ncclResult_t e = ncclAllReduce(m->grads + r.first, m->grads + r.first, (size_t)(r.second - r.first), ncclFloat32,
                                   ncclSum, (ncclComm_t)ctx->nccl_comm, ctx->comm);
    if (e != ncclSuccess) { ncclGroupEnd(); CHG_THROW(CHG_ERR_NCCL, "ncclAllReduce (bucket): %s", ncclGetErrorString(e)); }
    ++ctx->ar_buckets;
  }
  ncclResult_t e = ncclGroupEnd();
  if (e != ncclSuccess) CHG_THROW(CHG_ERR_NCCL, "ncclGroupEnd: %s", ncclGetErrorString(e));
  CUDA_OK(cudaEventRecord(ctx->ev_comm_done, ctx->comm));
  ctx->ar_pending = true;
}

// Everything after the loss seeds: head adjoints, interaction blocks (last to first), and —
// for training — the embedding / projection / frequency gradients.  deriv = 1: the
// conservative-force pass (seed ∂E/∂e_atom = 1 only, no parameter gradients): the force,
// stress and magmom heads are skipped and dE/d(e⁰, eᵃ, eᵇ, a⁰) are left in the de, dea, deb,
// da scratch rows for the geometry kernels (deriv.cu).
static void backward_core(chg_ctx *ctx, chg_model *m, chg_graph *g, const LossSeeds &sd, bool deriv) {
  const int64_t N = g->N, E = g->E, B = g->B, A = g->A;
  const int T = m->cfg.n_bond_conv;
  Bwd Bw{ctx, m, g, nullptr};
  if (!m->wt) CUDA_OK(cudaMalloc(&m->wt, 4 * (size_t)std::max<int64_t>(m->P, 1)));
  Bw.wt = m->wt;
  ctx->set_precision(m->cfg.mlp_precision);
  if (!ctx->use_tc) transpose_params(ctx, m, Bw.wt);   // tensor-core modes: the forward's copy is current
  ctx->cur_model = m;
  ctx->cur_wt = Bw.wt;
  float *dv = Bw.scratch("dv", N, 64), *de = Bw.scratch("de", E, 64), *da = Bw.scratch("da", A, 64);
  float *dea = Bw.scratch("dea", E, 64), *deb = Bw.scratch("deb", B, 64);
  fill_zero(ctx, dv, 4 * 64 * N);
  fill_zero(ctx, de, 4 * 64 * E);
  fill_zero(ctx, da, 4 * 64 * A);
  fill_zero(ctx, dea, 4 * 64 * E);
  fill_zero(ctx, deb, 4 * 64 * B);
  const float *vf = Bw.act("v" + std::to_string(T + 1)), *ef = Bw.act("e" + std::to_string(T));
  // heads backward: the force head (-> de) beside the atom-side heads (-> dv)
  if (!deriv) on_side(ctx, [&] { mlp_bwd(Bw, "head_F", 3, ef, E, sd.d_ne, 1, de); });
  mlp_bwd(Bw, "head_E", 4, vf, N, sd.d_eatom, 1, dv);
  if (!deriv) {
    WGrad wg;
    wg.A.seg[0] = aseg(vf, 64, 64);
    wg.A.nseg = 1;
    wg.M = (int)N; wg.K = 64;
    wg.D = sd.d_mag; wg.ldd = 1; wg.N = 1; wg.bias = 1;
    wg.dst[0].W = Bw.G("head_M.W"); wg.dst[0].ldw = 1; wg.dst[0].b = Bw.G("head_M.b");
    wg.tag = "headM_wg";
    wgrad(ctx, wg);
    RowGemm G;
    G.A.seg[0] = aseg(sd.d_mag, 1, 1);
    G.A.nseg = 1;
    G.M = (int)N; G.K = 1;
    G.ch[0] = chunk1(Bw.WT("head_M.W"), 64, 1, nullptr, dv, 64);
    G.ch[0].resid = dv; G.ch[0].ldr = 64;
    G.tag = "headM_b";
    rowgemm(ctx, G);
  }
  if (!deriv) mlp_bwd(Bw, "head_S", 3, vf, N, sd.d_M9, 9, dv);
  // A8 interaction blocks, last to first
  const float *ea = Bw.act("ea"), *eb = Bw.act("eb");
  float *dagg = Bw.scratch("dagg", N, 64), *daggb = Bw.scratch("daggb", B, 64);
  auto V = [&](int t) { return Bw.act("v" + std::to_string(t)); };
  auto Ef = [&](int t) { return Bw.act("e" + std::to_string(t)); };
  auto Af = [&](int t) { return Bw.act("a" + std::to_string(t)); };
  ac_bwd_head(Bw, T, dv, dagg);
  join_side(ctx);                                   // de complete before the atom conv adds to it
  ac_bwd_body(Bw, T, V(T), Ef(T), ea, dagg, dv, de, dea);
  // the split-partial reductions run per layer when the layer's gradients feed a bucketed
  // allreduce (NEXT-3); otherwise all of them in one launch at the end of the backward
  const bool per_layer = ctx->grad_overlap && ctx->nccl_comm && ctx->nranks > 1;
  if (per_layer) red_flush(ctx);
  ctx->ar_buckets = 0;
  grad_bucket(ctx, m, {{"head_"}, {"atom" + std::to_string(T) + "."}});
  for (int t = T - 1; t >= 0; --t) {
    bool ab = t + 1 < T;
    // both output linears read the incoming gradients before any update
    ac_bwd_head(Bw, t, dv, dagg);
    bc_bwd_head(Bw, t, de, daggb);
    if (!ctx->concurrent()) {
      ac_bwd_body(Bw, t, V(t), Ef(t), ea, dagg, dv, de, dea);
      bc_bwd_body(Bw, t, ab, V(t), Ef(t), Af(t), eb, daggb, dv, de, da, deb, 1);
    } else {   // the bond/angle adjoints up to their dv/de sums run beside the atom conv's
      cudaStream_t main_stream = ctx->stream;
      CUDA_OK(cudaEventRecord(ctx->ev_fork, main_stream));
      CUDA_OK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
      ctx->forked = true;
      ctx->stream = ctx->side;
      try {
        bc_bwd_body(Bw, t, ab, V(t), Ef(t), Af(t), eb, daggb, dv, de, da, deb, 1);
      } catch (...) {
        ctx->stream = main_stream;
        throw;
      }
      ctx->stream = main_stream;
      CUDA_OK(cudaEventRecord(ctx->ev_join, ctx->side));
      ac_bwd_body(Bw, t, V(t), Ef(t), ea, dagg, dv, de, dea);
      CUDA_OK(cudaStreamWaitEvent(main_stream, ctx->ev_join, 0));
      ctx->forked = false;
    }
    bc_bwd_body(Bw, t, ab, V(t), Ef(t), Af(t), eb, daggb, dv, de, da, deb, 2);
    if (per_layer) red_flush(ctx);
    const std::string ts = std::to_string(t);
    grad_bucket(ctx, m, {{"atom" + ts + "."}, {"bond" + ts + "."}, {"angle" + ts + "."}});
  }
  if (deriv) {                                      // no parameter gradients on this pass
    red_flush(ctx);
    return;
  }
  // embedding (rows of W_v gathered by species -> grouped sum, no atomics)
  embed_grad(ctx, N, m->cfg.n_species, g->species, dv, Bw.G("embed.W"));
  // projections (Eq. 2) and trainable frequencies, from the saved bases (proj.cu)
  proj_bwd(ctx, E, Bw.act("ea_t"), Bw.act("ea_g"), de, dea, m->p("proj.W0"), m->p("proj.Wa"), Bw.G("proj.W0"),
           Bw.G("proj.Wa"), Bw.G("rbf_a.freq"));
  proj_bwd(ctx, B, Bw.act("eb_t"), Bw.act("eb_g"), deb, nullptr, m->p("proj.Wb"), nullptr, Bw.G("proj.Wb"), nullptr,
           Bw.G("rbf_b.freq"));
  proj_bwd(ctx, A, Bw.act("a_t"), nullptr, da, nullptr, m->p("proj.Wtheta"), nullptr, Bw.G("proj.Wtheta"), nullptr,
           nullptr);
  red_flush(ctx);
  grad_bucket(ctx, m, {{"embed.", "rbf_a.", "rbf_b.", "proj."}});
  ctx->dbg["dv0"] = {dv, N, 64, 64};
  ctx->dbg["de0"] = {de, E, 64, 64};
  ctx->dbg["da0"] = {da, A, 64, 64};
  ctx->dbg["dea"] = {dea, E, 64, 64};
  ctx->dbg["deb"] = {deb, B, 64, 64};
}

void backward_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, const chg_labels *lab_in, const chg_loss_cfg *cfg,
                   double *loss_out) {
  const int64_t N = g->N, E = g->E, B = g->B, A = g->A;
  const int S = g->S, T = m->cfg.n_bond_conv;
  // a NULL label array skips that task; all four missing is a contract error
  if (!lab_in->energy_per_atom && !lab_in->forces && !lab_in->stress && !lab_in->magmom)
    CHG_THROW(CHG_ERR_ARG, "no labels: energy_per_atom, forces, stress and magmom are all NULL");
  Bwd Bw{ctx, m, g, nullptr};
  // split-partial reductions of a layer are batched into one launch (reduce.cu)
  struct RedScope {
    chg_ctx *c;
    explicit RedScope(chg_ctx *x) : c(x) { c->red_on = true; c->red_jobs.clear(); }
    ~RedScope() { c->red_on = false; c->red_jobs.clear(); }
  } red_scope(ctx);
  chg_labels lab = *lab_in;
  lab.energy_per_atom = labels_dev(ctx, lab_in->energy_per_atom, 4 * S, "lab_epa", lab_in->on_device);
  lab.forces = labels_dev(ctx, lab_in->forces, 12 * N, "lab_f", lab_in->on_device);
  lab.stress = labels_dev(ctx, lab_in->stress, 36 * (size_t)S, "lab_s", lab_in->on_device);
  lab.magmom = labels_dev(ctx, lab_in->magmom, 4 * N, "lab_m", lab_in->on_device);
  lab.magmom_mask = (const uint8_t *)labels_dev(ctx, lab_in->magmom_mask, N, "lab_mask", lab_in->on_device);
  lab.on_device = 1;
  // A7 loss + seeds
  LossSeeds sd;
  sd.d_eatom = Bw.scratch("seed_eatom", N, 1);
  sd.d_M9 = Bw.scratch("seed_M9", N, 9);
  sd.d_mag = Bw.scratch("seed_mag", N, 1);
  sd.d_ne = Bw.scratch("seed_ne", E, 1);
  loss_and_seeds(ctx, g, Bw.act("energy_per_atom"), Bw.act("forces"), Bw.act("stress"), Bw.act("magmom"), lab, *cfg,
                 sd);
  backward_core(ctx, m, g, sd, false);
  if (loss_out) {
    double *h = (double *)ctx->pinned_get(64);
    CUDA_OK(cudaMemcpyAsync(h, ctx->d_loss, 5 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 5; ++k) loss_out[k] = h[k];
  }
}

// ===========================================================================
// conservative forces and stress: F = −∂E/∂r, σ = (160.2/V)·∂E/∂ε
// ===========================================================================
void derivative_impl(chg_ctx *ctx, chg_model *m, chg_graph *g, chg_pred *out) {
  const int64_t N = g->N, E = g->E, B = g->B, A = g->A;
  forward_impl(ctx, m, g, 1, nullptr);
  struct Scope {
    chg_ctx *c;
    explicit Scope(chg_ctx *x) : c(x) { c->red_on = true; c->red_jobs.clear(); c->no_param_grads = true; }
    ~Scope() { c->red_on = false; c->red_jobs.clear(); c->no_param_grads = false; }
  } scope(ctx);
  Bwd Bw{ctx, m, g, nullptr};
  LossSeeds sd;                                      // ∂E/∂e_atom = 1 (E = Σ_s E_s); the other heads off
  sd.d_eatom = Bw.scratch("seed_eatom", N, 1);
  sd.d_M9 = Bw.scratch("seed_M9", N, 9);
  sd.d_mag = Bw.scratch("seed_mag", N, 1);
  sd.d_ne = Bw.scratch("seed_ne", E, 1);
  fill_value(ctx, sd.d_eatom, N, 1.0f);
  backward_core(ctx, m, g, sd, true);
  float *forces = Bw.scratch("dforces", N, 3), *stress = Bw.scratch("dstress", g->S, 9);
  deriv_geometry(ctx, g, m->p("rbf_a.freq"), m->p("rbf_b.freq"), m->cfg.envelope_p, m->p("proj.W0"), m->p("proj.Wa"),
                 m->p("proj.Wb"), m->p("proj.Wtheta"), Bw.scratch("de", E, 64), Bw.scratch("dea", E, 64),
                 Bw.scratch("deb", B, 64), Bw.scratch("da", A, 64), forces, stress);
  ctx->fwd_train = false;                            // the activations were consumed by this pass
  if (out) {
    copy_out(ctx, out->energy, Bw.act("energy"), g->S, out->on_device);
    copy_out(ctx, out->energy_per_atom, Bw.act("energy_per_atom"), g->S, out->on_device);
    copy_out(ctx, out->forces, forces, 3 * N, out->on_device);
    copy_out(ctx, out->stress, stress, 9 * (int64_t)g->S, out->on_device);
    copy_out(ctx, out->magmom, Bw.act("magmom"), N, out->on_device);
    if (!out->on_device) CUDA_OK(cudaStreamSynchronize(ctx->stream));
  }
}

// ===========================================================================
// A9 allreduce + Adam
// ===========================================================================

static std::string param_name_at(const chg_model *m, int flat) {
  std::string name = "?";
  for (size_t t = 0; t < m->names.size(); ++t)
    if (m->offsets[t] <= flat) name = m->names[t];
  return name;
}

// deferred finite checks (defer_check / captured steps): resolve every pending flag whose
// event has completed (all of them when block); the first non-finite one is reported
void check_pending(chg_ctx *ctx, bool block) {
  size_t k = 0;
  for (; k < ctx->pending.size(); ++k) {
    chg_ctx::Pending &p = ctx->pending[k];
    if (block) CUDA_OK(cudaEventSynchronize(p.ev));
    else if (cudaEventQuery(p.ev) != cudaSuccess) break;
    const int bad = ctx->h_flags[p.slot];
    ctx->flag_ev_pool.push_back(p.ev);
    if (bad != 0x7f7f7f7f) {
      const std::string name = p.m ? param_name_at(p.m, bad) : "?";
      for (size_t r = k + 1; r < ctx->pending.size(); ++r) ctx->flag_ev_pool.push_back(ctx->pending[r].ev);
      ctx->pending.clear();
      CHG_THROW(CHG_ERR_NONFINITE, "non-finite gradient in %s (flat index %d) at a deferred step: that update "
                "and the following ones were skipped on the device", name.c_str(), bad);
    }
  }
  ctx->pending.erase(ctx->pending.begin(), ctx->pending.begin() + k);
}

// a pinned flag slot and a completion event for a deferred check
void push_pending(chg_ctx *ctx, int slot, const chg_model *m) {
  cudaEvent_t ev;
  if (!ctx->flag_ev_pool.empty()) { ev = ctx->flag_ev_pool.back(); ctx->flag_ev_pool.pop_back(); }
  else CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_OK(cudaEventRecord(ev, ctx->stream));
  ctx->pending.push_back({ev, slot, m});
  if (ctx->pending.size() > chg_ctx::NFLAG / 2) check_pending(ctx, true);   // bounded: oldest are long done
}

int next_flag_slot(chg_ctx *ctx) {
  const int s = ctx->flag_next;
  ctx->flag_next = (ctx->flag_next + 1) % chg_ctx::NFLAG;
  return s;
}

void step_impl(chg_ctx *ctx, chg_model *m, const chg_adam_cfg *cfg, int slot) {
  if (cfg->step < 1) CHG_THROW(CHG_ERR_ARG, "adam step must be >= 1");
  if (!ctx->capturing) check_pending(ctx, false);
  if (ctx->ar_pending) {                            // bucketed during the backward (NEXT-3)
    CUDA_OK(cudaStreamWaitEvent(ctx->stream, ctx->ev_comm_done, 0));
    ctx->ar_pending = false;
  } else if (cfg->allreduce && ctx->nccl_comm && ctx->nranks > 1) {
    ProfScope ps(ctx, "allreduce", 0.0, 4.0 * m->P);
    ncclResult_t r = ncclAllReduce(m->grads, m->grads, (size_t)m->P, ncclFloat32, ncclSum,
                                   (ncclComm_t)ctx->nccl_comm, ctx->stream);
    if (r != ncclSuccess) CHG_THROW(CHG_ERR_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
  } else if (cfg->allreduce && ctx->nranks > 1) {
    CHG_THROW(CHG_ERR_STATE, "allreduce requested but no NCCL communicator");
  }
  double bc1 = 1.0 - std::pow((double)cfg->beta1, (double)cfg->step);
  double bc2 = 1.0 - std::pow((double)cfg->beta2, (double)cfg->step);
  if (slot < 0) slot = next_flag_slot(ctx);
  finite_adam(ctx, m->P, m->params, m->grads, m->m, m->v, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, bc1, bc2,
              ctx->h_flags + slot);
  if (ctx->capturing) return;                       // the replay records the check (chg_exec_step)
  if (cfg->defer_check) {                           // no host synchronisation: resolved by a later call
    push_pending(ctx, slot, m);
    return;
  }
  CUDA_OK(cudaStreamSynchronize(ctx->stream));
  const int bad = ctx->h_flags[slot];
  if (bad != 0x7f7f7f7f)   // nothing was updated (k_adam is guarded by the same flag)
    CHG_THROW(CHG_ERR_NONFINITE, "non-finite gradient in %s (flat index %d)", param_name_at(m, bad).c_str(), bad);
}
