// head_mlp.cu — fused readout MLPs (A6 heads and their A8 adjoints).
//
// The heads are plain MLPs: hidden layers Linear(64→64)+SiLU, last Linear(64→n_out)
// (P:141 energy head, Eq. 7 force head on e, Eq. 9 stress head on v).  They are not
// GatedMLP contractions, so they stay on the fp32 CUDA cores (NS), but each head is
// one kernel per direction instead of one GEMM launch per layer:
//
//   forward  (k_head_fwd):  a CTA keeps every weight of the head in shared memory and
//            walks R-row tiles (persistent grid; R = 64, or 16 when the rows — a small batch's
//            atoms — would leave most SMs idle): tile -> Z_k = H_{k-1} W_k + b_k
//            (stored for the backward), H_k = SiLU(Z_k) in smem -> out = H W_L + b_L.
//   backward (k_head_bwd):  per tile, dZ runs down the layers in smem; dX += dZ_0 W_0ᵀ is
//            added into the caller's gradient rows; dW_k, db_k are accumulated in
//            registers / fixed smem slots across the CTA's tiles and written once as a
//            per-CTA partial in the flat layout of the head's parameter block, reduced
//            in a fixed order by the batched reduction (reduce.cu; deterministic, no atomics).
//
// Register tiling: 256 threads, thread (a = t / 16, b = t % 16) owns R/16 rows x 4 columns of
// a layer output (4 x 4 input x output entries of a weight gradient).
// Shared tiles are [64][65] (odd pitch: column walks are conflict-free).
#include "common.cuh"
#include "ops.cuh"

namespace {

constexpr int HT = 64;        // rows per tile (16 when the rows would give fewer than 2 tiles per SM)
constexpr int HP = 65;        // smem pitch of the forward activation tile (odd: row walks across lanes are conflict-free)
constexpr int TPB = 68;       // smem pitch of the backward tiles (16-B rows: float4 row reads in the dW loop)
constexpr int HMAXL = 4;      // max linear layers per head

struct HeadArgs {
  const float *X;             // [rows, 64] input (v or e)
  int64_t rows;
  const float *P;             // head parameter block: W0 b0 W1 b1 ... (flat layout)
  float *Z[HMAXL - 1];        // pre-activations of the hidden layers [rows, 64]
  float *out; int ldo;        // forward output [rows, nout]
  const float *dout;          // backward seed [rows, nout]
  float *dX;                  // backward: dX[rows, 64] += ...
  float *part;                // backward: per-CTA partial [grid][block_size]
};

__host__ __device__ constexpr int head_block_size(int NL, int NOUT) { return (NL - 1) * (64 * 64 + 64) + 64 * NOUT + NOUT; }
// per-CTA partial stride (16-B aligned rows for the float4 stores)
__host__ __device__ constexpr int head_part_stride(int NL, int NOUT) { return (head_block_size(NL, NOUT) + 3) & ~3; }

__device__ __forceinline__ float silu_(float x) { return x / (1.0f + __expf(-x)); }
__device__ __forceinline__ float dsilu_(float x) {
  const float s = 1.0f / (1.0f + __expf(-x));
  return s * (1.0f + x * (1.0f - s));
}

// smem layout (floats): W hidden [NL-1][64][64] (forward: W[k][n]; backward: transposed W[n][k], so
// both kernels read 4 consecutive outputs as one float4) | b hidden [NL-1][64] | W last [64][NOUT]
// | b last [NOUT]
//                       | tiles ...
template <int NL, int NOUT>
struct HeadSmem {
  static constexpr int W = 0;
  static constexpr int B = W + (NL - 1) * 64 * 64;
  static constexpr int WL = B + (NL - 1) * 64;
  static constexpr int BL = WL + 64 * NOUT;
  static constexpr int T0 = (BL + NOUT + 3) & ~3;
};

template <int NL, int NOUT, bool TRANS>
__device__ void load_weights(const float *__restrict__ P, float *sm) {
  using S = HeadSmem<NL, NOUT>;
  for (int l = 0; l < NL - 1; ++l) {
    const float *Wg = P + l * (64 * 64 + 64);
#pragma unroll 8   // independent loads in flight (one latency, not one per iteration)
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x)
      sm[S::W + l * 64 * 64 + (TRANS ? (i % 64) * 64 + i / 64 : i)] = Wg[i];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) sm[S::B + l * 64 + i] = Wg[64 * 64 + i];
  }
  const float *Wl = P + (NL - 1) * (64 * 64 + 64);
  for (int i = threadIdx.x; i < 64 * NOUT; i += blockDim.x) sm[S::WL + i] = Wl[i];
  for (int i = threadIdx.x; i < NOUT; i += blockDim.x) sm[S::BL + i] = Wl[64 * NOUT + i];
}

// load a [64][64] row tile of a [rows, 64] matrix into smem [64][P] (zero rows past the end)
template <int P, int R>
__device__ __forceinline__ void load_tile(const float *__restrict__ src, int64_t r0, int64_t rows, float *dst) {
#pragma unroll 8   // independent loads in flight (one latency, not one per iteration)
  for (int i = threadIdx.x; i < R * 16; i += blockDim.x) {
    const int r = i >> 4, c4 = (i & 15) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r0 + r < rows) v = __ldg((const float4 *)(src + (r0 + r) * 64 + c4));
    float *d = dst + r * P + c4;
    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
  }
}

template <int NL, int NOUT, int R>
__global__ void __launch_bounds__(256) k_head_fwd(const __grid_constant__ HeadArgs a) {
  pdl_begin();
  extern __shared__ float sm[];
  using S = HeadSmem<NL, NOUT>;
  float *sH = sm + S::T0;            // [64][HP] layer input / activation
  load_weights<NL, NOUT, false>(a.P, sm);
  constexpr int RPT = R / 16;        // rows per thread
  const int t = threadIdx.x, ra = (t >> 4) * RPT, cb = (t & 15) * 4;
  const int64_t ntiles = (a.rows + R - 1) / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * R;
    __syncthreads();
    load_tile<HP, R>(a.X, r0, a.rows, sH);
    __syncthreads();
#pragma unroll 1
    for (int l = 0; l < NL - 1; ++l) {
      const float *W = sm + S::W + l * 64 * 64;
      float acc[RPT][4];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 8
      for (int k = 0; k < 64; ++k) {
        float h[RPT], w[4];
#pragma unroll
        for (int i = 0; i < RPT; ++i) h[i] = sH[(ra + i) * HP + k];
        const float4 w4 = *(const float4 *)&W[k * 64 + cb];
        w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(h[i], w[j], acc[i][j]);
      }
      __syncthreads();                 // every thread has read sH
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        float z[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          z[j] = acc[i][j] + sm[S::B + l * 64 + cb + j];
          sH[(ra + i) * HP + cb + j] = silu_(z[j]);
        }
        if (r0 + ra + i < a.rows) *(float4 *)(a.Z[l] + (r0 + ra + i) * 64 + cb) = make_float4(z[0], z[1], z[2], z[3]);
      }
      __syncthreads();
    }
    // last layer: out[r][o] = Σ_k H[r][k] W_L[k][o] + b_L[o]
    for (int p = t; p < R * NOUT; p += blockDim.x) {
      const int r = p / NOUT, o = p % NOUT;
      if (r0 + r >= a.rows) continue;
      float s = 0.f;
#pragma unroll 8
      for (int k = 0; k < 64; ++k) s = fmaf(sH[r * HP + k], sm[S::WL + k * NOUT + o], s);
      a.out[(r0 + r) * a.ldo + o] = s + sm[S::BL + o];
    }
  }
}

template <int NL, int NOUT, int R>
__global__ void __launch_bounds__(256) k_head_bwd(const __grid_constant__ HeadArgs a) {
  pdl_begin();
  extern __shared__ float sm[];
  using S = HeadSmem<NL, NOUT>;
  float *sA = sm + S::T0;            // layer input H_{k-1} (or X)
  float *sZ = sA + R * TPB;          // pre-activation z_{k-1}
  float *sG = sZ + R * TPB;          // dZ_k
  float *sD = sG + R * TPB;          // dout tile [R][NOUT]
  load_weights<NL, NOUT, true>(a.P, sm);
  constexpr int RPT = R / 16;        // tile rows per thread (dH); ta indexes inputs k in dW
  const int t = threadIdx.x, ta = (t >> 4) * 4, tr = (t >> 4) * RPT, tb = (t & 15) * 4;
  constexpr int NH = NL - 1;
  // per-thread accumulators: dW_k[ta..ta+3][tb..tb+3] (k = input row, n = output col), db_k[tb..] (ta == 0)
  float gW[NH][4][4], gb[NH][4];
#pragma unroll
  for (int l = 0; l < NH; ++l)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      gb[l][i] = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) gW[l][i][j] = 0.f;
    }
  constexpr int NLP = (64 * NOUT + 255) / 256;   // last-layer weight grads per thread
  float gWL[NLP], gbL = 0.f;
#pragma unroll
  for (int q = 0; q < NLP; ++q) gWL[q] = 0.f;

  const int64_t ntiles = (a.rows + R - 1) / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * R;
    __syncthreads();
    for (int p = t; p < R * NOUT; p += blockDim.x) {
      const int r = p / NOUT, o = p % NOUT;
      sD[p] = (r0 + r < a.rows) ? a.dout[(r0 + r) * NOUT + o] : 0.f;
    }
    load_tile<TPB, R>(a.Z[NH - 1], r0, a.rows, sZ);
    __syncthreads();
    for (int i = t; i < R * 64; i += blockDim.x) {
      const int r = i >> 6, c = i & 63;
      sA[r * TPB + c] = silu_(sZ[r * TPB + c]);
    }
    __syncthreads();
    // last layer: dW_L[k][o] += Σ_r H[r][k] dout[r][o], db_L[o] += Σ_r dout[r][o]
#pragma unroll
    for (int q = 0; q < NLP; ++q) {
      const int p = t + 256 * q;
      if (p < 64 * NOUT) {
        const int k = p / NOUT, o = p % NOUT;
        float s = 0.f;
        for (int r = 0; r < R; ++r) s = fmaf(sA[r * TPB + k], sD[r * NOUT + o], s);
        gWL[q] += s;
      }
    }
    if (t < NOUT) {
      float s = 0.f;
      for (int r = 0; r < R; ++r) s += sD[r * NOUT + t];
      gbL += s;
    }
    // dZ_{NH-1}[r][k] = (Σ_o dout[r][o] W_L[k][o]) · SiLU'(z[r][k])
    for (int i = t; i < R * 64; i += blockDim.x) {
      const int r = i >> 6, k = i & 63;
      float s = 0.f;
#pragma unroll
      for (int o = 0; o < NOUT; ++o) s = fmaf(sD[r * NOUT + o], sm[S::WL + k * NOUT + o], s);
      sG[r * TPB + k] = s * dsilu_(sZ[r * TPB + k]);
    }
    __syncthreads();
#pragma unroll
    for (int l = NH - 1; l >= 0; --l) {   // unrolled: gW[l] stays in registers
      // layer input: H_{l-1} = SiLU(z_{l-1}) (z kept in sZ for the next dZ), or X for l = 0
      if (l > 0) {
        load_tile<TPB, R>(a.Z[l - 1], r0, a.rows, sZ);
        __syncthreads();
        for (int i = t; i < R * 64; i += blockDim.x) {
          const int r = i >> 6, c = i & 63;
          sA[r * TPB + c] = silu_(sZ[r * TPB + c]);
        }
      } else {
        load_tile<TPB, R>(a.X, r0, a.rows, sA);
      }
      __syncthreads();
      // dW_l[k][n] += Σ_r A[r][k] G[r][n]; db_l[n] += Σ_r G[r][n]
      {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
        float cs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int r = 0; r < R; ++r) {
          const float4 x4 = *(const float4 *)&sA[r * TPB + ta], g4 = *(const float4 *)&sG[r * TPB + tb];
          const float x[4] = {x4.x, x4.y, x4.z, x4.w}, gg[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(x[i], gg[j], acc[i][j]);
#pragma unroll
          for (int j = 0; j < 4; ++j) cs[j] += gg[j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) gW[l][i][j] += acc[i][j];
        if (ta == 0)
#pragma unroll
          for (int j = 0; j < 4; ++j) gb[l][j] += cs[j];
      }
      // dH[r][k] = Σ_n G[r][n] W_l[k][n]: thread owns rows tr.., inputs k = tb..
      float dh[RPT][4];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dh[i][j] = 0.f;
      {
        const float *WT = sm + S::W + l * 64 * 64;     // WT[n][k] = W[k][n]
#pragma unroll 8
        for (int n = 0; n < 64; ++n) {
          float gg[RPT];
#pragma unroll
          for (int i = 0; i < RPT; ++i) gg[i] = sG[(tr + i) * TPB + n];
          const float4 w4 = *(const float4 *)&WT[n * 64 + tb];
          const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int i = 0; i < RPT; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dh[i][j] = fmaf(gg[i], w[j], dh[i][j]);
        }
      }
      __syncthreads();                 // all reads of sG / sZ done
      if (l > 0) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) sG[(tr + i) * TPB + tb + j] = dh[i][j] * dsilu_(sZ[(tr + i) * TPB + tb + j]);
      } else {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int64_t r = r0 + tr + i;
          if (r < a.rows) {
            float4 *d = (float4 *)(a.dX + r * 64 + tb);
            float4 v = *d;
            v.x += dh[i][0]; v.y += dh[i][1]; v.z += dh[i][2]; v.w += dh[i][3];
            *d = v;
          }
        }
      }
      __syncthreads();
    }
  }
  // per-CTA partial in the flat layout of the head block
  float *pp = a.part + (size_t)blockIdx.x * head_part_stride(NL, NOUT);
#pragma unroll
  for (int l = 0; l < NH; ++l) {
    float *Wp = pp + l * (64 * 64 + 64);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *(float4 *)(Wp + (ta + i) * 64 + tb) = make_float4(gW[l][i][0], gW[l][i][1], gW[l][i][2], gW[l][i][3]);
    if (ta == 0) *(float4 *)(Wp + 64 * 64 + tb) = make_float4(gb[l][0], gb[l][1], gb[l][2], gb[l][3]);
  }
  float *Lp = pp + NH * (64 * 64 + 64);
#pragma unroll
  for (int q = 0; q < NLP; ++q) {
    const int p = t + 256 * q;
    if (p < 64 * NOUT) Lp[p] = gWL[q];
  }
  if (t < NOUT) Lp[64 * NOUT + t] = gbL;
}

template <int NL, int NOUT, int R>
size_t head_smem_fwd() { return 4 * ((size_t)HeadSmem<NL, NOUT>::T0 + R * HP); }
template <int NL, int NOUT, int R>
size_t head_smem_bwd() { return 4 * ((size_t)HeadSmem<NL, NOUT>::T0 + 3 * R * TPB + R * NOUT); }

int sm_count() { return device_sm_count(); }

template <int NL, int NOUT, int R>
void run_fwd_r(chg_ctx *ctx, const HeadArgs &a, const char *tag) {
  const size_t smem = head_smem_fwd<NL, NOUT, R>();
  smem_optin((const void *)k_head_fwd<NL, NOUT, R>, (int)smem);
  const int64_t ntiles = (a.rows + R - 1) / R;
  const int grid = (int)std::min<int64_t>(ntiles, 2 * sm_count());
  ProfScope ps(ctx, tag, 2.0 * a.rows * (64.0 * 64 * (NL - 1) + 64.0 * NOUT),
               a.rows * 4.0 * (64 + 64 * (NL - 1) + NOUT) + 4.0 * head_block_size(NL, NOUT) * grid);
  launch_k(ctx, k_head_fwd<NL, NOUT, R>, grid, 256, smem, ctx->stream, a);
  check_launch(ctx);
}

// 64-row tiles; 16-row tiles when the rows (e.g. a small batch's atoms) would leave most SMs idle
template <int NL, int NOUT>
void run_fwd(chg_ctx *ctx, const HeadArgs &a, const char *tag) {
  if ((a.rows + HT - 1) / HT < 2 * sm_count()) run_fwd_r<NL, NOUT, 16>(ctx, a, tag);
  else run_fwd_r<NL, NOUT, HT>(ctx, a, tag);
}

template <int NL, int NOUT, int R>
void run_bwd_r(chg_ctx *ctx, HeadArgs a, float *G, const char *tag) {
  const size_t smem = head_smem_bwd<NL, NOUT, R>();
  smem_optin((const void *)k_head_bwd<NL, NOUT, R>, (int)smem);
  const int64_t ntiles = (a.rows + R - 1) / R;
  const int grid = (int)std::min<int64_t>(ntiles, 2 * sm_count());
  const int nb = head_block_size(NL, NOUT);
  const int stride = head_part_stride(NL, NOUT);
  a.part = red_partial(ctx, (size_t)grid * stride);
  {
    ProfScope ps(ctx, tag, 2.0 * a.rows * (2.0 * 64 * 64 * (NL - 1) + 2.0 * 64 * NOUT),
                 a.rows * 4.0 * (64 * 3 + 64 * (NL - 1) + NOUT) + 4.0 * nb * (double)grid * 2);
    launch_k(ctx, k_head_bwd<NL, NOUT, R>, grid, 256, smem, ctx->stream, a);
    check_launch(ctx);
  }
  RedJob j;                                        // per-CTA partials -> the head's gradient block
  j.kind = 1; j.n = nb; j.splits = grid; j.stride = stride; j.part = a.part; j.W[0] = G;
  red_push(ctx, j);
}

template <int NL, int NOUT>
void run_bwd(chg_ctx *ctx, HeadArgs a, float *G, const char *tag) {
  if ((a.rows + HT - 1) / HT < 2 * sm_count()) run_bwd_r<NL, NOUT, 16>(ctx, a, G, tag);
  else run_bwd_r<NL, NOUT, HT>(ctx, a, G, tag);
}

}  // namespace

void head_mlp_fwd(chg_ctx *ctx, int nl, int nout, const float *X, int64_t rows, const float *P, float *const *Z,
                  float *out, int ldo) {
  if (rows <= 0) return;
  HeadArgs a{};
  a.X = X; a.rows = rows; a.P = P; a.out = out; a.ldo = ldo;
  for (int l = 0; l + 1 < nl; ++l) a.Z[l] = Z[l];
  if (nl == 4 && nout == 1) run_fwd<4, 1>(ctx, a, "head_mlp_f");
  else if (nl == 3 && nout == 1) run_fwd<3, 1>(ctx, a, "head_mlp_f");
  else if (nl == 3 && nout == 9) run_fwd<3, 9>(ctx, a, "head_mlp_f");
  else CHG_THROW(CHG_ERR_ARG, "head_mlp_fwd: unsupported head shape (%d layers, %d outputs)", nl, nout);
}

void head_mlp_bwd(chg_ctx *ctx, int nl, int nout, const float *X, int64_t rows, const float *P, float *const *Z,
                  const float *dout, float *G, float *dX) {
  if (rows <= 0) return;
  HeadArgs a{};
  a.X = X; a.rows = rows; a.P = P; a.dout = dout; a.dX = dX;
  for (int l = 0; l + 1 < nl; ++l) a.Z[l] = Z[l];
  if (nl == 4 && nout == 1) run_bwd<4, 1>(ctx, a, G, "head_mlp_b");
  else if (nl == 3 && nout == 1) run_bwd<3, 1>(ctx, a, G, "head_mlp_b");
  else if (nl == 3 && nout == 9) run_bwd<3, 9>(ctx, a, G, "head_mlp_b");
  else CHG_THROW(CHG_ERR_ARG, "head_mlp_bwd: unsupported head shape (%d layers, %d outputs)", nl, nout);
}
