// ops.cuh — non-GEMM kernels of the hot path (declarations; see ops.cu).
#pragma once
#include "common.cuh"

// GatedMLP output stage: φ = σ(LN_g(y_g)) ⊙ SiLU(LN_c(y_c)); y [rows,128] = [core | gate]
struct GateLN { const float *gc, *bc, *gg, *bg; };
enum GateMode { GATE_MUL_W = 0, GATE_MUL_W1W2 = 1, GATE_RESID = 2 };
void gate_fwd(chg_ctx *ctx, int64_t rows, const float *y, int ldy, GateLN ln, int mode, const float *w,
              const int32_t *i1, const int32_t *i2, const float *resid, float *out);
// backward: dout gathered via didx (nullptr = row); writes dy [rows, 128] (ldd), LN grads
// accumulated into (dgc, dbc, dgg, dbg).  mode GATE_MUL_W: dw_out[row] += dout*φ (dea).
// mode GATE_MUL_W1W2: q1[row] = dout*φ*w[i2], q2[row] = dout*φ*w[i1].
struct GateLNGrad { float *gc, *bc, *gg, *bg; };
void gate_bwd(chg_ctx *ctx, int64_t rows, const float *y, int ldy, GateLN ln, int mode, const float *w,
              const int32_t *i1, const int32_t *i2, const float *dout, const int32_t *didx, float *dy,
              int lddy, float *dw_acc, float *q1, float *q2, GateLNGrad g);

// segmented row sums: out[t] (+)= Σ_src Σ_{r ∈ [ptr[s], ptr[s+1])} in[perm ? perm[r] : r]
// with s = segmap ? segmap[t] : t + ptr_off (segmap < 0 -> nothing).  64 columns.
struct SegSrc { const float *in = nullptr; const int32_t *ptr = nullptr; const int32_t *perm = nullptr;
                const int32_t *segmap = nullptr; int ptr_off = 0;
                int ld = 64;        // row stride of `in` (floats, multiple of 4)
                int64_t rows = 0;   // total input rows summed (algorithmic-bytes bookkeeping only)
};
// ncols (multiple of 64): column groups of 64 summed by grid.y (input column 64·y of every source).
// outoff != nullptr: the sources are NOT added — source k is summed into out + outoff[k] (grid.z)
void segsum(chg_ctx *ctx, int64_t targets, float *out, int ldo, int accumulate, int nsrc, const SegSrc *src,
            const char *tag = "segsum", int ncols = 64, const int *outoff = nullptr);

// segmented sum fused with the 64x64 linear that consumes it: agg = Σ rows (stored),
// out = (agg·W + bias) + resid (bias / resid optional); W row-major [64][64]
// agg_by_seg = 1: one source with a segmap; agg is stored at row segmap[t] (skipped when < 0)
void segsum_linear(chg_ctx *ctx, int64_t targets, int nsrc, const SegSrc *src, float *agg, const float *W,
                   const float *bias, const float *resid, float *out, const char *tag, int agg_by_seg = 0);

// embedding gradient: dW[z - 1] += Σ_{i: Z_i = z} dv[i] (species 1..n_species); per-block
// species bins reduced by the batched reduction (reduce.cu); deterministic
void embed_grad(chg_ctx *ctx, int64_t N, int n_species, const int32_t *species, const float *dv, float *dW);

// fused readout MLPs (head_mlp.cu): nl linear layers (hidden 64 + SiLU, last 64 -> nout),
// P / G = the head's parameter / gradient block in the flat layout (W0 b0 W1 b1 ...),
// Z[k] = hidden pre-activations [rows, 64] (written forward, read backward),
// dX [rows, 64] accumulates the input gradient.  Supported: (4, 1), (3, 1), (3, 9).
void head_mlp_fwd(chg_ctx *ctx, int nl, int nout, const float *X, int64_t rows, const float *P, float *const *Z,
                  float *out, int ldo);
void head_mlp_bwd(chg_ctx *ctx, int nl, int nout, const float *X, int64_t rows, const float *P, float *const *Z,
                  const float *dout, float *G, float *dX);

// fused basis + projection (proj.cu): radial sRBF (one or two 31x64 projections; basis and
// ∂basis/∂f saved [rows][32]) and Fourier angle basis; backward from the saved bases:
// dW (+)= basisᵀ·dE into G0/G1 and ∂L/∂f (+)= Σ_c W ⊙ (∂basis/∂f)ᵀ·dE (dbdf == nullptr: no freqs)
void proj_radial_fwd(chg_ctx *ctx, int64_t rows, const double4 *vec, const int32_t *eor, const float *freq,
                     double rc, int p, const float *W0, const float *W1, float *out0, float *out1, float *basis,
                     float *dbdf);
void proj_angle_fwd(chg_ctx *ctx, int64_t rows, const double4 *vec, const int32_t *e1, const int32_t *e2,
                    const float *W, float *out, float *basis);
void proj_bwd(chg_ctx *ctx, int64_t rows, const float *basis, const float *dbdf, const float *dE0, const float *dE1,
              const float *W0, const float *W1, float *G0, float *G1, float *dfreq);

// e' = e + (tmp[bond_id] or 0) + bias on all E edges (bond-conv output linear, Eq. 5 / Q16);
// float4 rows (64 floats), tmp holds the product for the B bond rows
void edge_update(chg_ctx *ctx, int64_t E, const float *e, const float *bias, const int32_t *bond_id, const float *tmp,
                 float *out);
// dst[idx[r]] += src[r], 64-float rows, idx injective (bond rows -> their atom-graph edges)
void rows_add(chg_ctx *ctx, int64_t rows, const int32_t *idx, const float *src, float *dst);
// grad[0..63] += column sums of D [rows, 64] (deterministic)
void colsum(chg_ctx *ctx, int64_t rows, const float *D, float *grad);

// conservative forces / stress (deriv.cu): from dE/d(e⁰, eᵃ, eᵇ, a⁰) of an energy-seeded backward
void deriv_geometry(chg_ctx *ctx, const chg_graph *g, const float *freq_a, const float *freq_b, int p,
                    const float *W0, const float *Wa, const float *Wb, const float *Wth, const float *de,
                    const float *dea, const float *deb, const float *da, float *forces, float *stress);
void fill_value(chg_ctx *ctx, float *x, int64_t n, float v);
// md.cu: velocity-Verlet half step (chg_md_verlet)
void md_verlet(chg_ctx *ctx, int64_t n, double *pos, double *vel, const float *F, const double *inv_mass, double dt,
               int drift);

// heads (Eq. 7, Eq. 9)
void heads_forces(chg_ctx *ctx, const chg_graph *g, const float *n_e, float *forces);
void heads_struct(chg_ctx *ctx, const chg_graph *g, const float *e_atom, const float *M9, float *energy,
                  float *epa, float *stress);
// loss + seeds; returns nothing, writes ctx->d_loss[0..4]
struct LossSeeds { float *d_eatom, *d_M9, *d_mag, *d_ne; };
void loss_and_seeds(chg_ctx *ctx, const chg_graph *g, const float *epa, const float *forces,
                    const float *stress, const float *mag, const chg_labels &lab, const chg_loss_cfg &cfg,
                    LossSeeds seeds);

// utilities
void transpose_params(chg_ctx *ctx, const chg_model *m, float *wt);
void fill_zero(chg_ctx *ctx, void *p, size_t bytes);
void embed_fwd(chg_ctx *ctx, int64_t N, const int32_t *species, const float *W, float *v);
// Adam (PyTorch semantics) + finite check
const void *adam_kernel();                        // k_adam (captured-step parameter updates)
void finite_adam(chg_ctx *ctx, int64_t n, float *p, float *g, float *m, float *v, float lr, float b1, float b2,
                 float eps, double bc1, double bc2, int *host_flag);
