// proj.cu — fused basis expansion + basis projection (A2 + A3) and their adjoints (A8).
//
// Forward (Eq. 2; the "Fused-sRBF" / "Fused-Fourier" of P:276-326 realised as one
// kernel per basis): a CTA computes the basis of a 64-row tile in fp64 (rounded once to fp32,
// same expressions as the reading Q2–Q6 in DESIGN.md), keeps it in shared memory and
// multiplies it by the projection weights held in shared memory: e⁰ | eᵃ = ẽᵃ [W₀ | Wₐ],
// eᵇ = ẽᵇ W_b, a⁰ = ã W_θ.  The basis rows (and, for the radial bases in train mode,
// ∂ẽ/∂f_n) are also written once: they are the backward's inputs, so the backward needs no
// transcendental recomputation.
//
// Backward: per tile, dW += ẽᵀ·dE and H += (∂ẽ/∂f)ᵀ·dE are accumulated per CTA (4 x 4 or
// 2 x 4 register blocks; H in fp64 across tiles), written once as per-CTA partials and reduced
// in CTA order; the frequency gradient is ∂L/∂f_n = Σ_c W[n][c] · H[n][c]
// (since ∂L/∂ẽ[r][n] = Σ_c dE[r][c] W[n][c]), so ∂L/∂ẽ is never materialised.
#include <cmath>

#include "ops.cuh"

namespace {

constexpr int PT = 64;            // rows per tile
constexpr int PBP = 33;           // smem pitch of basis tiles [64][33]

// u(ξ) for ξ < 1 and 0 beyond (u(1) = u'(1) = u''(1) = 0, so the clamp is smooth): pairs of a
// skin graph beyond the model cutoff then carry exactly zero bases
__device__ __forceinline__ double envelope_p(double xi, int p) {
  if (xi >= 1.0) return 0.0;
  double xp = 1.0;
  for (int k = 0; k < p; ++k) xp *= xi;
  double a = 0.5 * (p + 1) * (p + 2), b = (double)p * (p + 2), c = 0.5 * p * (p + 1);
  return 1.0 - xp * (a - xi * (b - c * xi));
}

struct ProjFwd {
  int64_t rows;
  const double4 *vec;             // fp64 geometry (graph builder)
  const int32_t *eor;             // radial: geometry row of basis row r (nullptr = r)
  const int32_t *e1, *e2;         // angle: the two bond edges
  const float *freq;              // radial: trainable frequencies [31]
  double rc;
  int p;
  const float *W[2];              // projection weights [31][64] (flat parameter layout)
  float *out[2];                  // [rows][64]
  float *basis;                   // [rows][32] saved basis (col 31 = 0)
  float *dbdf;                    // radial, train: [rows][32] ∂basis/∂f_n, or nullptr
};

// KIND 0: radial (sRBF with envelope), 1: angle (Fourier)
template <int NC, int KIND>
__global__ void __launch_bounds__(256) k_proj_fwd(const __grid_constant__ ProjFwd a) {
  pdl_begin();
  __shared__ float sW[32][NC * 64];
  __shared__ float sB[PT][PBP];
  const int t = threadIdx.x;
#pragma unroll 4
  for (int i = t; i < 32 * NC * 64; i += 256) {
    const int k = i / (NC * 64), c = i % (NC * 64);
    sW[k][c] = k < CHG_K ? a.W[c >> 6][k * 64 + (c & 63)] : 0.f;
  }
  const int64_t ntiles = (a.rows + PT - 1) / PT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * PT;
    __syncthreads();
    // ---- basis of the tile (fp64, rounded once)
    if (KIND == 0) {
      const int rr = t >> 2, n0 = (t & 3) * 8;
      const int64_t row = r0 + rr;
      float bv[8], gv[8];
      if (row < a.rows) {
        const int e = a.eor ? a.eor[row] : (int)row;
        const double r = a.vec[e].w, xi = r / a.rc;
        const double u = envelope_p(xi, a.p);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int n = n0 + q;
          bv[q] = gv[q] = 0.f;
          if (n < CHG_K) {
            double s, c;
            sincos((double)a.freq[n] * xi, &s, &c);
            bv[q] = (float)(u * sqrt(2.0 / a.rc) * s / r);
            gv[q] = (float)(u * sqrt(2.0 / a.rc) * c / a.rc);
          }
        }
        float4 *bo = (float4 *)(a.basis + row * CHG_KP + n0);
        bo[0] = make_float4(bv[0], bv[1], bv[2], bv[3]);
        bo[1] = make_float4(bv[4], bv[5], bv[6], bv[7]);
        if (a.dbdf) {
          float4 *go = (float4 *)(a.dbdf + row * CHG_KP + n0);
          go[0] = make_float4(gv[0], gv[1], gv[2], gv[3]);
          go[1] = make_float4(gv[4], gv[5], gv[6], gv[7]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) bv[q] = 0.f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) sB[rr][n0 + q] = bv[q];
    } else {
      if (t < PT) {
        const int64_t row = r0 + t;
        float v[32];
        if (row < a.rows) {
          const double4 d1 = a.vec[a.e1[row]], d2 = a.vec[a.e2[row]];
          double c = (d1.x * d2.x + d1.y * d2.y + d1.z * d2.z) / (d1.w * d2.w);
          c = fmin(1.0, fmax(-1.0, c));
          const double s = sqrt(fmax(0.0, 1.0 - c * c));   // sin θ >= 0 for θ in [0, π]
          const double isp = 0.56418958354775628695, is2p = 0.39894228040143267794;  // 1/√π, 1/√(2π)
          v[0] = (float)is2p;
          double ck = c, sk = s;
#pragma unroll
          for (int k = 1; k <= 15; ++k) {
            v[2 * k - 1] = (float)(ck * isp);
            v[2 * k] = (float)(sk * isp);
            const double cn = ck * c - sk * s, sn = sk * c + ck * s;   // angle addition: (k+1)θ
            ck = cn; sk = sn;
          }
          v[31] = 0.f;
          float4 *o = (float4 *)(a.basis + row * CHG_KP);
#pragma unroll
          for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) sB[t][q] = v[q];
      }
    }
    __syncthreads();
    // ---- projection: out[r][c] = Σ_k B[r][k] W[k][c]
    constexpr int RPT = NC == 2 ? 8 : 4;            // rows per thread
    const int rb = NC == 2 ? (t >> 5) * 8 : (t >> 4) * 4;
    const int cb = NC == 2 ? (t & 31) * 4 : (t & 15) * 4;
    float acc[RPT][4];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < CHG_K; ++k) {
      const float4 w = *(const float4 *)&sW[k][cb];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const float b = sB[rb + i][k];
        acc[i][0] = fmaf(b, w.x, acc[i][0]);
        acc[i][1] = fmaf(b, w.y, acc[i][1]);
        acc[i][2] = fmaf(b, w.z, acc[i][2]);
        acc[i][3] = fmaf(b, w.w, acc[i][3]);
      }
    }
    float *o = a.out[cb >> 6];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t row = r0 + rb + i;
      if (row < a.rows) *(float4 *)(o + row * 64 + (cb & 63)) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
  }
}

struct ProjBwd {
  int64_t rows;
  const float *basis;             // [rows][32]
  const float *dbdf;              // [rows][32] or nullptr (no trainable frequencies)
  const float *dE[2];             // [rows][64] incoming gradients of the projections
  float *partW;                   // [grid][32][NC*64]
  double *partH;                  // [grid][32][NC*64] (radial only)
};

constexpr int PTB = 32;           // rows per backward tile (static smem < 48 KB)

template <int NC, bool RADIAL>
__global__ void __launch_bounds__(256) k_proj_bwd(const __grid_constant__ ProjBwd a) {
  pdl_begin();
  constexpr int C = NC * 64;
  __shared__ float sB[PTB][PBP];
  __shared__ float sG[RADIAL ? PTB : 1][PBP];
  __shared__ float sD[PTB][C + 1];
  const int t = threadIdx.x;
  // thread owns basis functions nb.. (NPT of them) x columns c = cl + CS·j (conflict-free rows)
  constexpr int NPT = NC == 2 ? 4 : 2;
  constexpr int CS = NC == 2 ? 32 : 16;
  const int nb = NC == 2 ? (t >> 5) * 4 : (t >> 4) * 2;
  const int cl = NC == 2 ? (t & 31) : (t & 15);
  float gW[NPT][4];
  double gH[NPT][4];
#pragma unroll
  for (int i = 0; i < NPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { gW[i][j] = 0.f; gH[i][j] = 0.0; }
  const int64_t ntiles = (a.rows + PTB - 1) / PTB;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * PTB;
    __syncthreads();
#pragma unroll 4
    for (int i = t; i < PTB * 8; i += 256) {         // basis (and derivative) tiles: float4 per thread
      const int r = i >> 3, q = (i & 7) * 4;
      float4 b = make_float4(0.f, 0.f, 0.f, 0.f), g = b;
      if (r0 + r < a.rows) {
        b = __ldg((const float4 *)(a.basis + (r0 + r) * CHG_KP + q));
        if (RADIAL) g = __ldg((const float4 *)(a.dbdf + (r0 + r) * CHG_KP + q));
      }
      sB[r][q] = b.x; sB[r][q + 1] = b.y; sB[r][q + 2] = b.z; sB[r][q + 3] = b.w;
      if (RADIAL) { sG[r][q] = g.x; sG[r][q + 1] = g.y; sG[r][q + 2] = g.z; sG[r][q + 3] = g.w; }
    }
#pragma unroll 4
    for (int i = t; i < PTB * C / 4; i += 256) {
      const int r = i / (C / 4), c = (i % (C / 4)) * 4;
      float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r0 + r < a.rows) d = __ldg((const float4 *)(a.dE[c >> 6] + (r0 + r) * 64 + (c & 63)));
      sD[r][c] = d.x; sD[r][c + 1] = d.y; sD[r][c + 2] = d.z; sD[r][c + 3] = d.w;
    }
    __syncthreads();
    float w[NPT][4], h[NPT][4];
#pragma unroll
    for (int i = 0; i < NPT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) { w[i][j] = 0.f; h[i][j] = 0.f; }
#pragma unroll 4
    for (int r = 0; r < PTB; ++r) {
      float d[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = sD[r][cl + CS * j];
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        const float b = sB[r][nb + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[i][j] = fmaf(b, d[j], w[i][j]);
        if (RADIAL) {
          const float g = sG[r][nb + i];
#pragma unroll
          for (int j = 0; j < 4; ++j) h[i][j] = fmaf(g, d[j], h[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NPT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        gW[i][j] += w[i][j];
        if (RADIAL) gH[i][j] += (double)h[i][j];
      }
  }
  float *pw = a.partW + (size_t)blockIdx.x * 32 * C;
  double *ph = RADIAL ? a.partH + (size_t)blockIdx.x * 32 * C : nullptr;
#pragma unroll
  for (int i = 0; i < NPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pw[(nb + i) * C + cl + CS * j] = gW[i][j];
      if (RADIAL) ph[(nb + i) * C + cl + CS * j] = gH[i][j];
    }
}

// ∂L/∂f_n += Σ_c W[n][c] · Σ_cta partH[cta][n][c]: block n (1024 threads), thread (split, c);
// splits of the CTA range, combined in order, then a fixed-order tree over c
__global__ void __launch_bounds__(1024) k_proj_reduce_f(const double *__restrict__ partH, int nctas, int C,
                                                        const float *W0, const float *W1, float *dfreq) {
  pdl_begin();
  __shared__ double sh[1024];
  const int n = blockIdx.x, t = threadIdx.x, c = t % C, sp = t / C, nsp = 1024 / C;
  double h = 0.0;
  for (int k = sp; k < nctas; k += nsp) h += partH[(size_t)k * 32 * C + n * C + c];
  sh[t] = h;
  __syncthreads();
  if (sp == 0) {
    double hs = 0.0;
    for (int q = 0; q < nsp; ++q) hs += sh[q * C + c];
    const float *W = c < 64 ? W0 : W1;
    sh[c] = hs * (double)W[n * 64 + (c & 63)];
  }
  __syncthreads();
  for (int o = C / 2; o > 0; o >>= 1) {
    if (t < o) sh[t] += sh[t + o];
    __syncthreads();
  }
  if (t == 0) dfreq[n] += (float)sh[0];
}

int sm_count_p() { return device_sm_count(); }

}  // namespace

void proj_radial_fwd(chg_ctx *ctx, int64_t rows, const double4 *vec, const int32_t *eor, const float *freq,
                     double rc, int p, const float *W0, const float *W1, float *out0, float *out1, float *basis,
                     float *dbdf) {
  if (rows <= 0) return;
  ProjFwd a{};
  a.rows = rows; a.vec = vec; a.eor = eor; a.freq = freq; a.rc = rc; a.p = p;
  a.W[0] = W0; a.W[1] = W1; a.out[0] = out0; a.out[1] = out1; a.basis = basis; a.dbdf = dbdf;
  const int nc = W1 ? 2 : 1;
  const int grid = (int)std::min<int64_t>((rows + PT - 1) / PT, 4 * sm_count_p());
  ProfScope ps(ctx, "proj_basis", 2.0 * rows * CHG_K * 64 * nc,
               rows * (32.0 + (eor ? 4 : 0) + 128.0 * (dbdf ? 2 : 1) + 256.0 * nc));
  if (nc == 2) launch_k(ctx, k_proj_fwd<2, 0>, grid, 256, 0, ctx->stream, a);
  else launch_k(ctx, k_proj_fwd<1, 0>, grid, 256, 0, ctx->stream, a);
  check_launch(ctx);
}

void proj_angle_fwd(chg_ctx *ctx, int64_t rows, const double4 *vec, const int32_t *e1, const int32_t *e2,
                    const float *W, float *out, float *basis) {
  if (rows <= 0) return;
  ProjFwd a{};
  a.rows = rows; a.vec = vec; a.e1 = e1; a.e2 = e2; a.W[0] = W; a.out[0] = out; a.basis = basis;
  const int grid = (int)std::min<int64_t>((rows + PT - 1) / PT, 4 * sm_count_p());
  ProfScope ps(ctx, "proj_basis", 2.0 * rows * CHG_K * 64, rows * (8.0 + 64.0 + 128.0 + 256.0));
  launch_k(ctx, k_proj_fwd<1, 1>, grid, 256, 0, ctx->stream, a);
  check_launch(ctx);
}

void proj_bwd(chg_ctx *ctx, int64_t rows, const float *basis, const float *dbdf, const float *dE0, const float *dE1,
              const float *W0, const float *W1, float *G0, float *G1, float *dfreq) {
  if (rows <= 0) return;
  const int nc = dE1 ? 2 : 1, C = 64 * nc;
  const bool radial = dbdf != nullptr;
  const int grid = (int)std::min<int64_t>((rows + PTB - 1) / PTB, 2 * sm_count_p());
  ProjBwd a{};
  a.rows = rows; a.basis = basis; a.dbdf = dbdf; a.dE[0] = dE0; a.dE[1] = dE1;
  a.partW = red_partial(ctx, (size_t)grid * 32 * C);
  a.partH = radial ? (double *)ctx->get("proj_partH", (size_t)grid * 32 * C * 8) : nullptr;
  {
    ProfScope ps(ctx, "proj_bwd", 2.0 * rows * CHG_K * C * (radial ? 2 : 1),
                 rows * (128.0 * (radial ? 2 : 1) + 256.0 * nc) + grid * 32.0 * C * (radial ? 12 : 4));
    if (nc == 2 && radial) launch_k(ctx, k_proj_bwd<2, true>, grid, 256, 0, ctx->stream, a);
    else if (nc == 1 && radial) launch_k(ctx, k_proj_bwd<1, true>, grid, 256, 0, ctx->stream, a);
    else if (nc == 1) launch_k(ctx, k_proj_bwd<1, false>, grid, 256, 0, ctx->stream, a);
    else CHG_THROW(CHG_ERR_ARG, "proj_bwd: unsupported shape");
    check_launch(ctx);
  }
  RedJob j;                                        // dW: batched reduction (reduce.cu)
  j.kind = 3; j.n = CHG_K * C; j.N = C; j.splits = grid; j.stride = 32 * C; j.part = a.partW;
  j.W[0] = G0; j.W[1] = G1;
  red_push(ctx, j);
  if (radial) {
    ProfScope ps(ctx, "proj_reduce", 0.0, grid * 32.0 * C * 8);
    launch_k(ctx, k_proj_reduce_f, CHG_K, 1024, 0, ctx->stream, a.partH, grid, C, W0, W1, dfreq);
    check_launch(ctx);
  }
}
