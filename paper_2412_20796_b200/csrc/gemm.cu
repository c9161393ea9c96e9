// gemm.cu — fp32 CUDA-core GEMMs of the strict-parity path (see gemm.cuh).
#include "gemm.cuh"

namespace {

constexpr int TM = 128, TN = 64;   // default rows per CTA, columns per chunk (K step: template TK)

// A(m, col) for 4 consecutive columns (segment widths are multiples of 4)
__device__ __forceinline__ float4 loadA4(const AOp &A, int m, int col) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  int start = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < A.nseg) {
      int w = A.seg[s].width;
      if (col >= start && col < start + w) {
        int row = A.seg[s].idx ? __ldg(A.seg[s].idx + m) : m;
        if (row >= 0) v = __ldg((const float4 *)(A.seg[s].base + (size_t)row * A.seg[s].ld + (col - start)));
      }
      start += w;
    }
  }
  if (A.act == 1) { v.x = siluf_(v.x); v.y = siluf_(v.y); v.z = siluf_(v.z); v.w = siluf_(v.w); }
  return v;
}

__device__ __forceinline__ float loadA1(const AOp &A, int m, int col) {
  float v = 0.f;
  int start = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < A.nseg) {
      int w = A.seg[s].width;
      if (col >= start && col < start + w) {
        int row = A.seg[s].idx ? __ldg(A.seg[s].idx + m) : m;
        if (row >= 0) v = __ldg(A.seg[s].base + (size_t)row * A.seg[s].ld + (col - start));
      }
      start += w;
    }
  }
  if (A.act == 1) v = siluf_(v);
  return v;
}


// W(k, n..n+3) as one 16-B load when aligned (else per element; zeros past ncols)
__device__ __forceinline__ float4 loadW4(const Chunk &c, int k, int n) {
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if (b < c.nwb && k >= c.wk0[b] && k < c.wk0[b + 1]) {
      const float *p = c.W[b] + (size_t)(k - c.wk0[b]) * c.ldw[b] + n;
      if (n + 3 < c.ncols && ((uintptr_t)p & 15) == 0) return __ldg((const float4 *)p);
      float4 v;
      v.x = n < c.ncols ? __ldg(p) : 0.f;
      v.y = n + 1 < c.ncols ? __ldg(p + 1) : 0.f;
      v.z = n + 2 < c.ncols ? __ldg(p + 2) : 0.f;
      v.w = n + 3 < c.ncols ? __ldg(p + 3) : 0.f;
      return v;
    }
  return make_float4(0.f, 0.f, 0.f, 0.f);
}

// TM rows per CTA (128 for large M; 32 when few CTAs would be launched),
// 256 threads = 16 (x 4 columns) x 16 (x TM/16 rows)
template <bool VEC, int TM, int TK = 32>
__global__ void __launch_bounds__(256) k_rowgemm(const __grid_constant__ RowGemm g) {
  pdl_begin();
  constexpr int RPT = TM / 16;
  __shared__ __align__(16) float As[TK][TM + 4];
  __shared__ __align__(16) float Ws[TK][TN];
  const Chunk &c = g.ch[blockIdx.y];
  const int m0 = blockIdx.x * TM;
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  float acc[RPT][4];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < g.K; k0 += TK) {
    if (VEC) {
#pragma unroll
      for (int i = 0; i < (TM * TK / 4 + 255) / 256; ++i) {
        const int e = t + 256 * i;
        if (TM * TK / 4 % 256 != 0 && e >= TM * TK / 4) break;
        int r = e / (TK / 4), c4 = e % (TK / 4);
        int m = m0 + r, kk = k0 + 4 * c4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < g.M && kk < g.K) v = loadA4(g.A, m, c.a_k0 + kk);
        As[4 * c4 + 0][r] = v.x; As[4 * c4 + 1][r] = v.y; As[4 * c4 + 2][r] = v.z; As[4 * c4 + 3][r] = v.w;
      }
    } else {
#pragma unroll 4
      for (int i = 0; i < (TM * TK) / 256; ++i) {
        int e = t + 256 * i, r = e / TK, kk = e % TK;
        int m = m0 + r, k = k0 + kk;
        As[kk][r] = (m < g.M && k < g.K) ? loadA1(g.A, m, c.a_k0 + k) : 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < (TK * TN) / 1024; ++i) {       // independent 16-B weight loads (one latency)
      const int e = t + 256 * i, kr = e / (TN / 4), n = (e % (TN / 4)) * 4;
      const int k = k0 + kr;
      *(float4 *)&Ws[kr][n] = (k < g.K) ? loadW4(c, k, n) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < TK; ++kk) {
      float a[RPT];
      if (RPT == 8) {
        float4 a0 = *(const float4 *)&As[kk][ty * 8];
        float4 a1 = *(const float4 *)&As[kk][ty * 8 + 4];
        a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
        a[RPT > 4 ? 4 : 0] = a1.x; a[RPT > 5 ? 5 : 0] = a1.y; a[RPT > 6 ? 6 : 0] = a1.z; a[RPT > 7 ? 7 : 0] = a1.w;
      } else {
#pragma unroll
        for (int i = 0; i < RPT; ++i) a[i] = As[kk][ty * RPT + i];
      }
      float4 b = *(const float4 *)&Ws[kk][tx * 4];
      float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    int m = m0 + ty * RPT + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = tx * 4 + j;
      if (n >= c.ncols) continue;
      float v = acc[i][j];
      if (c.bias) v += __ldg(c.bias + n);
      for (int k = 0; k < c.ngadd; ++k) {
        const int r = c.gidx[k] ? __ldg(c.gidx[k] + m) : m;
        v += __ldg(c.gadd[k] + (size_t)r * c.ldga[k] + n);
      }
      if (c.pre) c.pre[(size_t)m * c.ldp + n] = v;
      if (g.act == 1) v = siluf_(v);
      if (c.mul) v *= dsiluf_(c.mul[(size_t)m * c.ldm + n]);
      if (c.resid) v += c.resid[(size_t)m * c.ldr + n];
      if (c.sout) c.sout[(size_t)m * c.ldso + n] = tf32_round(silu_fast(v));
      c.out[(size_t)m * c.ldo + n] = c.round_out ? tf32_round(v) : v;
    }
  }
}

constexpr int WK = 64, WN = 64, WM = 32;

template <bool VEC>
__global__ void __launch_bounds__(256) k_wgrad(const WGrad g, float *__restrict__ partial, int Kp, int rows_per_split) {
  pdl_begin();
  __shared__ __align__(16) float As[WM][WK + 4];
  __shared__ __align__(16) float Ds[WM][WN + 4];
  const int kt = blockIdx.x, nt = blockIdx.y, sp = blockIdx.z;
  const int mb = sp * rows_per_split, me = min(g.M, mb + rows_per_split);
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const bool dvec = VEC && (g.ldd % 4 == 0) && (g.N % 4 == 0);
  for (int m0 = mb; m0 < me; m0 += WM) {
    // A tile [WM][WK]
    if (VEC) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        int e = t + 256 * i, r = e >> 4, c4 = e & 15;
        int m = m0 + r, col = kt * WK + 4 * c4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < me) {
          if (col < g.K) v = loadA4(g.A, m, col);
          float *pv = &v.x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (col + q >= g.K) pv[q] = 0.f;
            if (g.bias && col + q == g.K) pv[q] = 1.f;
          }
        }
        *(float4 *)&As[r][4 * c4] = v;
      }
    } else {
#pragma unroll 4
      for (int i = 0; i < (WM * WK) / 256; ++i) {
        int e = t + 256 * i, r = e / WK, cc = e % WK;
        int m = m0 + r, col = kt * WK + cc;
        float v = 0.f;
        if (m < me) {
          if (col < g.K) v = loadA1(g.A, m, col);
          else if (g.bias && col == g.K) v = 1.f;
        }
        As[r][cc] = v;
      }
    }
    // D tile [WM][WN]
    if (dvec) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        int e = t + 256 * i, r = e >> 4, c4 = e & 15;
        int m = m0 + r, n = nt * WN + 4 * c4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < me && n < g.N) {
          int row = g.didx ? __ldg(g.didx + m) : m;
          v = __ldg((const float4 *)(g.D + (size_t)row * g.ldd + n));
        }
        *(float4 *)&Ds[r][4 * c4] = v;
      }
    } else {
#pragma unroll 4
      for (int i = 0; i < (WM * WN) / 256; ++i) {
        int e = t + 256 * i, r = e / WN, cc = e % WN;
        int m = m0 + r, n = nt * WN + cc;
        float v = 0.f;
        if (m < me && n < g.N) {
          int row = g.didx ? __ldg(g.didx + m) : m;
          v = __ldg(g.D + (size_t)row * g.ldd + n);
        }
        Ds[r][cc] = v;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < WM; ++r) {
      float4 a = *(const float4 *)&As[r][ty * 4];
      float4 d = *(const float4 *)&Ds[r][tx * 4];
      float av[4] = {a.x, a.y, a.z, a.w}, dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], dv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float *P = partial + (size_t)sp * Kp * g.N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int k = kt * WK + ty * 4 + i;
    if (k >= Kp) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = nt * WN + tx * 4 + j;
      if (n < g.N) P[(size_t)k * g.N + n] = acc[i][j];
    }
  }
}

bool aop_vec(const AOp &A) {
  for (int s = 0; s < A.nseg; ++s) {
    const ASeg &S = A.seg[s];
    if (S.width % 4 || S.ld % 4 || ((uintptr_t)S.base & 15)) return false;
  }
  return true;
}

}  // namespace

// K-major view of an N-major weight block through the transposed parameter copy
// (params and wt share flat offsets; tensor t = [R, C] in params, [C, R] in wt).
static bool kmajor_of(const chg_model *m, const float *wt, const float *p, int ldw, const float **pk, int *ldk) {
  for (int side = 0; side < 2; ++side) {
    const float *base = side == 0 ? m->params : wt;
    if (p < base || p >= base + m->P) continue;
    int64_t rel = p - base;
    auto it = std::upper_bound(m->offsets.begin(), m->offsets.end(), rel);
    int t = (int)(it - m->offsets.begin()) - 1;
    int R = m->shapes[2 * t], C = m->shapes[2 * t + 1];
    if (C == 0) return false;
    int64_t o = m->offsets[t], r = rel - o;
    if (side == 0) {                      // W [R, C] used N-major with ld C
      if (ldw != C) return false;
      int64_t k0 = r / C, n0 = r % C;
      *pk = wt + o + n0 * R + k0; *ldk = R;
    } else {                              // Wᵀ [C, R] used N-major with ld R
      if (ldw != R) return false;
      int64_t k0 = r / R, n0 = r % R;
      *pk = m->params + o + n0 * C + k0; *ldk = C;
    }
    return true;
  }
  return false;
}

double gemm_a_bytes(const AOp &A, int64_t M, int lo, int hi) {
  double b = 0;
  int start = 0;
  for (int s = 0; s < A.nseg; ++s) {
    const ASeg &S = A.seg[s];
    const int w = std::max(0, std::min(hi, start + S.width) - std::max(lo, start));
    start += S.width;
    if (w <= 0) continue;
    if (S.idx) b += 4.0 * M + 4.0 * w * (double)(S.rows > 0 ? std::min<int64_t>(S.rows, M) : M);
    else b += 4.0 * w * (double)M;
  }
  return b;
}

void rowgemm(chg_ctx *ctx, const RowGemm &g) {
  if (g.M <= 0) return;
  // small problems (per-atom / per-bond products of the factorised layer 1): the persistent
  // tensor-core kernel's fixed cost (TMEM, barriers, resident weight image) outweighs the math
  static const int tc_min_rows = getenv("CHG_TC_MIN_ROWS") ? atoi(getenv("CHG_TC_MIN_ROWS")) : 0;
  if (g.tc && ctx->use_tc && ctx->cur_model && ctx->cur_wt && g.M >= tc_min_rows) {
    RowGemm h = g;
    bool ok = true;
    for (int c = 0; c < h.nchunk && ok; ++c)
      for (int b = 0; b < h.ch[c].nwb && ok; ++b)
        ok = kmajor_of(ctx->cur_model, ctx->cur_wt, h.ch[c].W[b], h.ch[c].ldw[b], &h.ch[c].Wk[b], &h.ch[c].ldwk[b]);
    if (ok && rowgemm_tc(ctx, h)) return;
  }
  bool vec = aop_vec(g.A);
  int tot = 0;
  for (int s = 0; s < g.A.nseg; ++s) tot += g.A.seg[s].width;
  for (int c = 0; c < g.nchunk; ++c)
    if (g.ch[c].a_k0 + ((g.K + 3) & ~3) > tot) vec = false;
  // algorithmic work: 2·M·K·Σncols flops; bytes = A columns read once (union of
  // chunk windows) + gather indices + outputs (+pre/mul/resid) + weights
  double cols = 0, outb = 0, wb = 0;
  int lo = 1 << 30, hi = 0;
  for (int c = 0; c < g.nchunk; ++c) {
    const Chunk &C = g.ch[c];
    cols += C.ncols;
    outb += C.ncols * (1.0 + (C.pre != nullptr) + (C.mul != nullptr) + (C.resid != nullptr) + (C.sout != nullptr));
    wb += (double)g.K * C.ncols;
    lo = std::min(lo, C.a_k0);
    hi = std::max(hi, C.a_k0 + g.K);
  }
  ProfScope ps(ctx, g.tag ? g.tag : "rowgemm", 2.0 * g.M * (double)g.K * cols,
               gemm_a_bytes(g.A, g.M, lo, hi) + (double)g.M * 4.0 * outb + 4.0 * wb);
  const bool small = (int64_t)ceil_div(g.M, TM) * g.nchunk < 2 * 148;
  if (small && g.K > 32) {
    // few rows: short tiles and the whole K = 64 in one smem stage (one load latency, not two)
    const bool tiny = (int64_t)ceil_div(g.M, 32) * g.nchunk < 148;
    if (tiny) {
      dim3 grid(ceil_div(g.M, 16), g.nchunk);
      if (vec) launch_k(ctx, k_rowgemm<true, 16, 64>, grid, 256, 0, ctx->stream, g);
      else launch_k(ctx, k_rowgemm<false, 16, 64>, grid, 256, 0, ctx->stream, g);
    } else {
      dim3 grid(ceil_div(g.M, 32), g.nchunk);
      if (vec) launch_k(ctx, k_rowgemm<true, 32, 64>, grid, 256, 0, ctx->stream, g);
      else launch_k(ctx, k_rowgemm<false, 32, 64>, grid, 256, 0, ctx->stream, g);
    }
  } else if (small) {
    dim3 grid(ceil_div(g.M, 32), g.nchunk);
    if (vec) launch_k(ctx, k_rowgemm<true, 32>, grid, 256, 0, ctx->stream, g);
    else launch_k(ctx, k_rowgemm<false, 32>, grid, 256, 0, ctx->stream, g);
  } else {
    dim3 grid(ceil_div(g.M, TM), g.nchunk);
    if (vec) launch_k(ctx, k_rowgemm<true, TM>, grid, 256, 0, ctx->stream, g);
    else launch_k(ctx, k_rowgemm<false, TM>, grid, 256, 0, ctx->stream, g);
  }
  check_launch(ctx);
}

// split partials [splits][Kp][N] -> W / bias of each 64-column chunk (reduce.cu, batched)
static void launch_wgrad_reduce(chg_ctx *ctx, const WGrad &g, const float *partial, int Kp, int splits) {
  RedJob j;
  j.kind = 0;
  j.n = Kp * g.N;
  j.splits = splits;
  j.stride = (int64_t)Kp * g.N;
  j.part = partial;
  j.K = g.K;
  j.N = g.N;
  for (int c = 0; c < 4; ++c) {
    j.W[c] = g.dst[c].W; j.ldw[c] = g.dst[c].ldw; j.b[c] = g.dst[c].b; j.k0[c] = g.dst[c].k0; j.kn[c] = g.dst[c].kn;
  }
  red_push(ctx, j);
}

void wgrad(chg_ctx *ctx, const WGrad &g) {
  if (ctx->no_param_grads) return;
  int Kp = g.K + (g.bias ? 1 : 0);
  if (Kp <= 0 || g.N <= 0) return;
  static const int tc_min_rows = getenv("CHG_TC_MIN_ROWS") ? atoi(getenv("CHG_TC_MIN_ROWS")) : 0;
  if (g.tc && ctx->use_tc && g.M > 0 && g.M >= tc_min_rows) {
    float *partial = nullptr;
    int kp = 0, splits = 0;
    bool bias_done = false;
    if (wgrad_tc(ctx, g, &partial, &kp, &splits, &bias_done)) {
      launch_wgrad_reduce(ctx, g, partial, kp, splits);
      if (!bias_done) {            // K is a multiple of 128: column sums of D on the CUDA cores
        WGrad b = g;
        b.A.nseg = 0;
        b.K = 0;
        b.tc = 0;
        wgrad(ctx, b);
      }
      return;
    }
    bool plain_dst = true;
    for (int c = 0; c < 4; ++c) plain_dst &= g.dst[c].k0 == 0 && g.dst[c].kn < 0;
    if (ctx->tc_split && g.K > 128 && plain_dst) {
      // 3xTF32 stages ([hi | lo] operands) are twice as large: the rows k of the gradient (the
      // A columns) are split into pieces of 128, each a launch over the same D; a piece takes the
      // column ranges of the A segments it overlaps (a segment's columns are base + offset)
      for (int k0 = 0; k0 < g.K; k0 += 128) {
        const int k1 = std::min(g.K, k0 + 128);
        WGrad h = g;
        h.A.nseg = 0;
        for (int sg = 0, c0 = 0; sg < g.A.nseg; c0 += g.A.seg[sg].width, ++sg) {
          const int lo = std::max(k0, c0), hi = std::min(k1, c0 + g.A.seg[sg].width);
          if (lo >= hi) continue;
          ASeg piece = g.A.seg[sg];
          piece.base += lo - c0;
          piece.width = hi - lo;
          h.A.seg[h.A.nseg++] = piece;
        }
        h.K = k1 - k0;
        h.bias = (k0 == 0) ? g.bias : 0;
        for (int c = 0; c < 4; ++c) {
          h.dst[c].W = g.dst[c].W ? g.dst[c].W + (size_t)k0 * g.dst[c].ldw : nullptr;
          if (k0 != 0) h.dst[c].b = nullptr;
        }
        wgrad(ctx, h);
      }
      return;
    }
  }
  int ktiles = ceil_div(Kp, WK), ntiles = ceil_div(g.N, WN);
  int splits = 1;
  if (g.M > 0) {
    splits = std::max(1, std::min(ceil_div(g.M, WM), 296 / (ktiles * ntiles)));
  }
  int rps = g.M > 0 ? ceil_div(ceil_div(g.M, splits), WM) * WM : WM;
  splits = g.M > 0 ? ceil_div(g.M, rps) : 1;
  float *partial = red_partial(ctx, (size_t)splits * Kp * g.N);
  {
    ProfScope ps(ctx, g.tag ? g.tag : "wgrad", 2.0 * g.M * (double)Kp * g.N,
                 gemm_a_bytes(g.A, g.M, 0, g.K) + (double)g.M * (4.0 * g.N + (g.didx ? 4.0 : 0.0)) + 4.0 * Kp * g.N);
    bool vec = aop_vec(g.A);
    dim3 grid(ktiles, ntiles, splits);
    if (vec)
      launch_k(ctx, k_wgrad<true>, grid, 256, 0, ctx->stream, g, partial, Kp, rps);
    else
      launch_k(ctx, k_wgrad<false>, grid, 256, 0, ctx->stream, g, partial, Kp, rps);
    check_launch(ctx);
  }
  launch_wgrad_reduce(ctx, g, partial, Kp, splits);
}

// ---------------------------------------------------------------------------
// kernel unit-test hook (chg_debug_gemm, include/chg.h)
// ---------------------------------------------------------------------------
extern "C" chg_status chg_debug_gemm(chg_ctx *ctx, int kind, int engine, int M, int K, int N, const float *A,
                                     const float *W, float *out) {
  if (!ctx || !A || !W || !out || M <= 0 || K <= 0 || N <= 0 || (kind != 0 && kind != 1)) return CHG_ERR_ARG;
  try {
    cudaStream_t st = ctx->stream;
    const size_t na = (size_t)M * K, nw = kind == 0 ? (size_t)K * N : (size_t)M * N;
    const size_t no = kind == 0 ? (size_t)M * N : (size_t)K * N;
    float *dA = ctx->getf("dbg_gemm_A", na), *dW = ctx->getf("dbg_gemm_W", nw), *dO = ctx->getf("dbg_gemm_O", no);
    float *dWk = ctx->getf("dbg_gemm_Wk", kind == 0 ? nw : 1);
    CUDA_OK(cudaMemcpyAsync(dA, A, 4 * na, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(dW, W, 4 * nw, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemsetAsync(dO, 0, 4 * no, st));
    const bool old = ctx->use_tc, old_split = ctx->tc_split, old_bf16 = ctx->tc_bf16;
    const chg_model *old_model = ctx->cur_model;
    ctx->set_precision(engine);
    ctx->cur_model = nullptr;                  // no weight-image caching for the hook's scratch operands
    if (kind == 0) {
      std::vector<float> wk((size_t)K * N);
      for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) wk[(size_t)n * K + k] = W[(size_t)k * N + n];
      CUDA_OK(cudaMemcpyAsync(dWk, wk.data(), 4 * nw, cudaMemcpyHostToDevice, st));
      RowGemm G;
      G.A.seg[0] = aseg(dA, K, K);
      G.A.nseg = 1;
      G.M = M; G.K = K;
      G.nchunk = (N + 63) / 64;
      G.tc = 1;
      if (G.nchunk > 4) CHG_THROW(CHG_ERR_ARG, "N > 256");
      for (int c = 0; c < G.nchunk; ++c) {
        G.ch[c] = chunk1(dW + 64 * c, N, K, nullptr, dO + 64 * c, N, std::min(64, N - 64 * c));
        G.ch[c].Wk[0] = dWk + (size_t)64 * c * K;
        G.ch[c].ldwk[0] = K;
      }
      bool done = engine != 0 ? rowgemm_tc(ctx, G) : false;
      if (engine != 0 && !done) CHG_THROW(CHG_ERR_ARG, "shape not supported by the tensor-core engine");
      if (!done) { G.tc = 0; rowgemm(ctx, G); }
    } else {
      WGrad g;
      g.A.seg[0] = aseg(dA, K, K);
      g.A.nseg = 1;
      g.M = M; g.K = K;
      g.D = dW; g.ldd = N; g.N = N; g.bias = 0; g.tc = engine != 0;
      if (N > 256) CHG_THROW(CHG_ERR_ARG, "N > 256");
      for (int c = 0; c * 64 < N; ++c) { g.dst[c].W = dO + 64 * c; g.dst[c].ldw = N; }
      wgrad(ctx, g);
    }
    ctx->use_tc = old;
    ctx->tc_split = old_split;
    ctx->tc_bf16 = old_bf16;
    ctx->cur_model = old_model;
    CUDA_OK(cudaMemcpyAsync(out, dO, 4 * no, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  } catch (const ChgError &e) {
    ctx->err = e.msg;
    return e.code;
  }
  return CHG_OK;
}
