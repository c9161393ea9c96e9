// gemm.cuh — fp32 CUDA-core GEMM engine of the strict-parity path.
//
// Row GEMM: out[m, n] = epi( Σ_k A(m, k) · W(k, n) + b[n] ) with A gathered on the
// fly from up to 4 row tables (the concatenations [v_i, v_j, e_ij] of Eq. 4 and
// [v_i, e_ij, e_ik, a_ijk] of Eq. 5/6 are never materialised), W split in up to
// 4 row blocks (weight concatenation of Fig. 3a without copying), and up to 4
// output column chunks of 64 with their own W / bias / destination (core and
// gate branches of Fig. 3b in one launch).
//
// Weight-gradient GEMM: G[k, n] += Σ_m A(m, k) · D(m, n) (+ column sums of D as
// the bias gradient), split over m across CTAs, partials reduced in a fixed
// order (deterministic, no atomics).
#pragma once
#include "common.cuh"

struct ASeg {
  const float *base = nullptr;   // row table
  const int32_t *idx = nullptr;  // row index per m (nullptr = m); idx < 0 -> zero row
  int ld = 0;                    // row stride (floats)
  int width = 0;                 // columns contributed by this segment
  int64_t rows = 0;              // rows of the gathered table (algorithmic bytes: read once); 0 = M
};

struct AOp {
  ASeg seg[4];
  int nseg = 0;
  int act = 0;                   // 0: identity, 1: silu applied on load
  int rounded = 0;               // 1: values are already TF32-rounded (tcgen05 path: no conversion pass)
};

struct Chunk {
  const float *W[8] = {};        // row blocks of W (up to 8)
  int ldw[8] = {};
  int wk0[9] = {};               // row-block starts, wk0[nwb] = K
  int nwb = 1;
  const float *bias = nullptr;
  int a_k0 = 0;                  // first A column read by this chunk
  int ncols = 64;                // valid output columns (<= 64)
  float *out = nullptr; int ldo = 0;
  const float *resid = nullptr; int ldr = 0;   // added after activation
  float *pre = nullptr; int ldp = 0;           // pre-activation store
  const float *mul = nullptr; int ldm = 0;     // v *= dsilu(mul) (backward of silu)
  float *sout = nullptr; int ldso = 0;         // second output tf32(SiLU(v)) (the next GEMM's operand)
  int round_out = 0;                           // 1: out is stored TF32-rounded (consumed by tcgen05 only)
  // gathered row additions before the activation: v += gadd[k][gidx[k][m] * ldga[k] + n]
  // (the per-atom / per-bond products of the factorised first GatedMLP layer)
  const float *gadd[3] = {nullptr, nullptr, nullptr};
  const int32_t *gidx[3] = {nullptr, nullptr, nullptr};
  int ldga[3] = {0, 0, 0};
  int ngadd = 0;
  // K-major view of the same weight blocks (element (n, k) at Wk[b][n*ldwk[b] + k - wk0[b]]),
  // filled by the orchestration for the tensor-core path (tc_gemm.cu)
  const float *Wk[8] = {};
  int ldwk[8] = {};
};

struct RowGemm {
  AOp A;
  int M = 0;
  int K = 0;                     // reduction length (per chunk)
  int act = 0;                   // 0 none, 1 silu
  int nchunk = 1;
  int tc = 0;                    // 1: a GatedMLP contraction -> tensor cores in TF32 mode (NS)
  const char *tag = nullptr;     // profiling label (chg_profile)
  Chunk ch[4];
};

struct WGradDst {
  float *W = nullptr; int ldw = 0;   // gradient of W columns [n0, n0+64), rows 0..K-1
  float *b = nullptr;                // gradient of bias (column sums), optional
  int k0 = 0, kn = -1;               // only rows [k0, k0+kn) go to W (kn < 0: all K rows)
};

struct WGrad {
  AOp A;                         // A(m, k), k < K
  int M = 0, K = 0;
  const float *D = nullptr;      // D(m, n) = D[(didx ? didx[m] : m) * ldd + n]
  const int32_t *didx = nullptr;
  int ldd = 0;
  int N = 0;                     // columns of D (<= 256)
  int bias = 0;                  // 1: also column sums of D -> dst.b
  int tc = 0;                    // 1: a GatedMLP weight gradient -> tensor cores in TF32 mode
  const char *tag = nullptr;     // profiling label (chg_profile)
  WGradDst dst[4];               // per 64-column chunk of N
};

void tc_repack_all(chg_ctx *ctx, chg_model *m);   // forward start (TF32 mode): refresh cached weight images
void tc_cache_free(chg_model *m);
void rowgemm(chg_ctx *ctx, const RowGemm &g);      // tcgen05 when ctx->use_tc and eligible, else SIMT
bool rowgemm_tc(chg_ctx *ctx, const RowGemm &g);   // false if the shape does not fit the tensor-core path
void wgrad(chg_ctx *ctx, const WGrad &g);
bool wgrad_tc(chg_ctx *ctx, const WGrad &g, float **partial, int *Kp, int *splits, bool *bias_done);

// helpers to fill descriptors
inline ASeg aseg(const float *base, int ld, int width, const int32_t *idx = nullptr, int64_t table_rows = 0) {
  ASeg s; s.base = base; s.ld = ld; s.width = width; s.idx = idx; s.rows = table_rows; return s;
}
// Algorithmic (compulsory) bytes of reading A columns [lo, hi) for M rows: a direct
// segment is streamed once (4·w·M); a gathered one costs its indices (4·M) plus its
// table read once (4·w·min(rows, M)) — repeated gathers of a row are L2 hits.
double gemm_a_bytes(const AOp &A, int64_t M, int lo, int hi);
inline Chunk chunk1(const float *W, int ldw, int K, const float *bias, float *out, int ldo, int ncols = 64) {
  Chunk c; c.W[0] = W; c.ldw[0] = ldw; c.wk0[0] = 0; c.wk0[1] = K; c.nwb = 1; c.bias = bias;
  c.out = out; c.ldo = ldo; c.ncols = ncols; return c;
}
