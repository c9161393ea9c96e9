// ops.cu — non-GEMM kernels of the FastCHGNet training step (see ops.cuh).
#include <climits>
#include <cmath>

#include "ops.cuh"

namespace {

// ---------------------------------------------------------------------------
// GatedMLP output stage
// ---------------------------------------------------------------------------
struct RowStats { float mu, rstd; };
__device__ __forceinline__ RowStats ln_stats(float a, float b) {
  float mu = warp_sum(a + b) * (1.0f / 64.0f);
  float da = a - mu, db = b - mu;
  float var = warp_sum(da * da + db * db) * (1.0f / 64.0f);
  return {mu, rsqrtf(var + 1e-5f)};
}

// 16 lanes per row, 2 rows per warp: lane j = lane & 15 of row slot rs = lane >> 4 owns columns
// 4j..4j+3 of each 64-wide branch (one float4: a row is one coalesced 256-B access).  LayerNorm
// statistics are 4-step shuffle reductions inside the half-warp, and a warp carries 2
// independent rows through every dependent chain (the row loop is latency-bound, not HBM-bound).
typedef float4 G8;                                   // a lane's 4 columns of one 64-wide row
__device__ __forceinline__ G8 ld8(const float *row, int j) { return __ldg((const float4 *)(row + 4 * j)); }
__device__ __forceinline__ G8 ld8p(const float *row, int j) { return *(const float4 *)(row + 4 * j); }
__device__ __forceinline__ void st8(float *row, int j, const float (&v)[4]) {
  *(float4 *)(row + 4 * j) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void un8(const G8 &g, float (&v)[4]) { v[0] = g.x; v[1] = g.y; v[2] = g.z; v[3] = g.w; }
// LayerNorm affine vectors sit at canonical flat offsets (only 8-B aligned): two float2 loads
__device__ __forceinline__ G8 ldp8(const float *p, int j) {
  const float2 a = __ldg((const float2 *)(p + 4 * j)), b = __ldg((const float2 *)(p + 4 * j + 2));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float sum8(float v) {     // over the 16 lanes of a row group
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  return v;
}
__device__ __forceinline__ RowStats ln_stats8(const float (&v)[4]) {
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += v[q];
  const float mu = sum8(s) * (1.0f / 64.0f);
  float s2 = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) s2 += (v[q] - mu) * (v[q] - mu);
  return {mu, rsqrtf(sum8(s2) * (1.0f / 64.0f) + 1e-5f)};
}

__global__ void __launch_bounds__(256) k_gate_fwd(int64_t rows, const float *__restrict__ y, int ldy, GateLN ln,
                                                  int mode, const float *__restrict__ w,
                                                  const int32_t *__restrict__ i1, const int32_t *__restrict__ i2,
                                                  const float *__restrict__ resid, float *__restrict__ out) {
  pdl_begin();
  const int lane = threadIdx.x & 31, j = lane & 15, rs = lane >> 4;
  const int64_t step = (int64_t)gridDim.x * (blockDim.x >> 5) * 2;
  float gc[4], bc[4], gg[4], bg[4];
  un8(ldp8(ln.gc, j), gc); un8(ldp8(ln.bc, j), bc); un8(ldp8(ln.gg, j), gg); un8(ldp8(ln.bg, j), bg);
  struct Ops { G8 yc, yg, w1, w2; };
  auto load = [&](int64_t r, Ops &o) {
    o.yc = ld8(y + r * ldy, j);
    o.yg = ld8(y + r * ldy + 64, j);
    if (mode == GATE_MUL_W) {
      o.w1 = ld8(w + r * 64, j);
    } else if (mode == GATE_MUL_W1W2) {
      o.w1 = ld8(w + (int64_t)__ldg(i1 + r) * 64, j);
      o.w2 = ld8(w + (int64_t)__ldg(i2 + r) * 64, j);
    } else {
      o.w1 = ld8(resid + r * 64, j);
    }
  };
  int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2;
  Ops nx;
  if (base + rs < rows) load(base + rs, nx);
  for (; base < rows; base += step) {
    const int64_t r = base + rs;
    const bool ok = r < rows;
    const Ops cu = nx;
    if (base + step + rs < rows) load(base + step + rs, nx);      // next rows in flight
    float yc[4], yg[4], w1[4], w2[4];
    un8(cu.yc, yc); un8(cu.yg, yg); un8(cu.w1, w1);
    if (mode == GATE_MUL_W1W2) un8(cu.w2, w2);
    const RowStats sc = ln_stats8(yc), sg = ln_stats8(yg);
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float nc = gc[q] * (yc[q] - sc.mu) * sc.rstd + bc[q];
      const float ng = gg[q] * (yg[q] - sg.mu) * sg.rstd + bg[q];
      const float p = sigmoidf_(ng) * siluf_(nc);
      o[q] = mode == GATE_MUL_W ? p * w1[q] : mode == GATE_MUL_W1W2 ? p * w1[q] * w2[q] : w1[q] + p;
    }
    if (ok) st8(out + r * 64, j, o);
  }
}

__global__ void __launch_bounds__(256) k_gate_bwd(int64_t rows, int64_t rpb, const float *__restrict__ y, int ldy,
                                                  GateLN ln, int mode, const float *__restrict__ w,
                                                  const int32_t *__restrict__ i1, const int32_t *__restrict__ i2,
                                                  const float *__restrict__ dout, const int32_t *__restrict__ didx,
                                                  float *__restrict__ dy, int lddy, float *__restrict__ dw_acc,
                                                  float *__restrict__ q1, float *__restrict__ q2,
                                                  float *__restrict__ partial, int rnd) {
  pdl_begin();
  __shared__ float sh[8][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, j = lane & 15, rs = lane >> 4;
  const int64_t r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  float gc[4], bc[4], gg[4], bg[4];
  un8(ldp8(ln.gc, j), gc); un8(ldp8(ln.bc, j), bc); un8(ldp8(ln.gg, j), gg); un8(ldp8(ln.bg, j), bg);
  float a_gc[4], a_bc[4], a_gg[4], a_bg[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) a_gc[q] = a_bc[q] = a_gg[q] = a_bg[q] = 0.f;
  struct Ops { G8 yc, yg, d, w1, w2; };
  auto load = [&](int64_t r, Ops &o) {
    o.yc = ld8(y + r * ldy, j);
    o.yg = ld8(y + r * ldy + 64, j);
    o.d = ld8p(dout + (didx ? (int64_t)__ldg(didx + r) : r) * 64, j);
    if (mode == GATE_MUL_W) {
      o.w1 = ld8(w + r * 64, j);
    } else if (mode == GATE_MUL_W1W2) {
      o.w1 = ld8(w + (int64_t)__ldg(i1 + r) * 64, j);
      o.w2 = ld8(w + (int64_t)__ldg(i2 + r) * 64, j);
    }
  };
  // block = rpb contiguous rows; warp w takes row pairs r0 + 2 (w + 8 i) + rs
  int64_t base = r0 + 2 * wid;
  Ops nx;
  if (base + rs < r1) load(base + rs, nx);
  for (; base < r1; base += 16) {
    const int64_t r = base + rs;
    const bool ok = r < r1;
    const Ops cu = nx;
    if (base + 16 + rs < r1) load(base + 16 + rs, nx);
    float yc[4], yg[4], d[4], w1[4], w2[4];
    un8(cu.yc, yc); un8(cu.yg, yg); un8(cu.d, d);
    if (mode != GATE_RESID) un8(cu.w1, w1);
    if (mode == GATE_MUL_W1W2) un8(cu.w2, w2);
    if (!ok) {
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q] = 0.f;               // padding rows contribute nothing
    }
    const RowStats sc = ln_stats8(yc), sg = ln_stats8(yg);
    float xc[4], xg[4], dnc[4], dng[4], phi[4], dphi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      xc[q] = (yc[q] - sc.mu) * sc.rstd;
      xg[q] = (yg[q] - sg.mu) * sg.rstd;
      const float nc = gc[q] * xc[q] + bc[q], ng = gg[q] * xg[q] + bg[q];
      const float s_g = sigmoidf_(ng), s_c = siluf_(nc);
      phi[q] = s_g * s_c;
      dphi[q] = mode == GATE_MUL_W ? d[q] * w1[q] : mode == GATE_MUL_W1W2 ? d[q] * w1[q] * w2[q] : d[q];
      dnc[q] = dphi[q] * s_g * dsiluf_(nc);
      dng[q] = dphi[q] * s_c * s_g * (1.0f - s_g);
      a_gc[q] += dnc[q] * xc[q]; a_bc[q] += dnc[q];
      a_gg[q] += dng[q] * xg[q]; a_bg[q] += dng[q];
    }
    float m1c = 0.f, m2c = 0.f, m1g = 0.f, m2g = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      m1c += gc[q] * dnc[q]; m2c += gc[q] * dnc[q] * xc[q];
      m1g += gg[q] * dng[q]; m2g += gg[q] * dng[q] * xg[q];
    }
    m1c = sum8(m1c) * (1.0f / 64.0f); m2c = sum8(m2c) * (1.0f / 64.0f);
    m1g = sum8(m1g) * (1.0f / 64.0f); m2g = sum8(m2g) * (1.0f / 64.0f);
    if (!ok) continue;
    float oc[4], og[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      oc[q] = sc.rstd * (gc[q] * dnc[q] - m1c - xc[q] * m2c);
      og[q] = sg.rstd * (gg[q] * dng[q] - m1g - xg[q] * m2g);
      if (rnd) { oc[q] = tf32_round(oc[q]); og[q] = tf32_round(og[q]); }   // dY feeds only TF32 GEMMs
    }
    st8(dy + r * lddy, j, oc);
    st8(dy + r * lddy + 64, j, og);
    if (mode == GATE_MUL_W) {
      float acc[4];
      un8(ld8p(dw_acc + r * 64, j), acc);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += d[q] * phi[q];
      st8(dw_acc + r * 64, j, acc);
    } else if (mode == GATE_MUL_W1W2) {
      float t1[4], t2[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { t1[q] = d[q] * phi[q] * w2[q]; t2[q] = d[q] * phi[q] * w1[q]; }
      st8(q1 + r * 64, j, t1);
      st8(q2 + r * 64, j, t2);
    }
  }
  // LN affine partials: the 2 row slots of a warp hold the same columns (xor 16), then warps
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    a_gc[q] += __shfl_xor_sync(0xffffffffu, a_gc[q], 16);
    a_bc[q] += __shfl_xor_sync(0xffffffffu, a_bc[q], 16);
    a_gg[q] += __shfl_xor_sync(0xffffffffu, a_gg[q], 16);
    a_bg[q] += __shfl_xor_sync(0xffffffffu, a_bg[q], 16);
  }
  if (rs == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col = 4 * j + q;
      sh[wid][col] = a_gc[q]; sh[wid][64 + col] = a_bc[q];
      sh[wid][128 + col] = a_gg[q]; sh[wid][192 + col] = a_bg[q];
    }
  }
  __syncthreads();
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += sh[k][threadIdx.x];
  partial[blockIdx.x * 256 + threadIdx.x] = s;
}

// half-warps per target: enough for ~16+ rows each on long segments, and enough in total to
// fill the GPU (~75K threads) when there are few targets (atoms of a small batch); the split
// depends only on (mean length, targets), so the summation order is fixed for a given batch
static int seg_split(int64_t mean, int64_t targets) {
  int H = mean >= 96 ? 8 : mean >= 48 ? 4 : mean >= 24 ? 2 : 1;
  while (H < 8 && targets * 16 * H < 75000 && mean >= 2 * H) H *= 2;
  return H;
}

// ---------------------------------------------------------------------------
// segmented sums (warp per target row, 2 columns per lane, fixed order)
// ---------------------------------------------------------------------------
struct SegArgs { SegSrc s[3]; int n; int sep; int outoff[3]; };   // sep: source k -> its own output (grid.z)

// rows [r0, r1) of S (through S.perm) added in order into acc (lane hl = float4 column quad of a
// 256-B row): row indices are fetched 16 at a time (coalesced) and broadcast by shuffle; U rows
// are in flight per lane (all loads of a group issued, predicated, before the in-order adds)
template <int U>
__device__ __forceinline__ void seg_rows(const SegSrc &S, int r0, int r1, int hl, unsigned hmask, float4 &acc,
                                         int col0 = 0) {
  const float4 *in = (const float4 *)(S.in + col0) + hl;
  const int64_t st4 = S.ld >> 2;
  for (int base = r0; base < r1; base += 16) {
    const int n = min(16, r1 - base);
    const int myrow = hl < n ? (S.perm ? __ldg(S.perm + base + hl) : base + hl) : 0;
    for (int q = 0; q < n; q += U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int qq = __shfl_sync(hmask, myrow, (q + u) & 15, 16);
        v[u] = (q + u < n) ? __ldg(in + (int64_t)qq * st4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q + u < n) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
}

// half-warp per target, one float4 (4 columns) per lane: a 256-B row is one
// 16-lane load.  Row indices are fetched 16 at a time (coalesced) and broadcast by
// shuffle; 4 or 8 rows are in flight per lane (seg_rows).  Rows are added in segment order,
// so the result is deterministic.
// H half-warps per target (H = 1, 2, 4, 8; long segments): half-warp j sums the fixed j-th
// contiguous part of every source segment, the H partials are added in j order through shared
// memory — the split points depend only on the segment length, so the result is deterministic.
template <int H, int U>
__global__ void __launch_bounds__(256) k_segsum(int64_t targets, float *__restrict__ out, int ldo, int accumulate,
                                                SegArgs a) {
  pdl_begin();
  __shared__ float4 part[16][16];                   // [half-warp in block][lane]
  const int hw = threadIdx.x >> 4;                  // half-warp in block (16)
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / (16 * H);
  const int j = hw % H;                             // part of the segments this half-warp sums
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hmask = 0xffffu << (lane & 16);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t < targets) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k >= a.n) break;
      if (a.sep && k != (int)blockIdx.z) continue;
      const SegSrc &S = a.s[k];
      const int64_t sg = S.segmap ? (int64_t)__ldg(S.segmap + t) : t + S.ptr_off;
      if (sg < 0) continue;
      int r0 = __ldg(S.ptr + sg), r1 = __ldg(S.ptr + sg + 1);
      if (H > 1) {
        const int len = r1 - r0;
        const int a0 = r0 + (int)((int64_t)len * j / H), a1 = r0 + (int)((int64_t)len * (j + 1) / H);
        r0 = a0; r1 = a1;
      }
      seg_rows<U>(S, r0, r1, hl, hmask, acc, 64 * (int)blockIdx.y);
    }
  }
  if (H > 1) {
    part[hw][hl] = acc;
    __syncthreads();
    if (j != 0 || t >= targets) return;
#pragma unroll
    for (int q = 1; q < H; ++q) {
      const float4 p = part[hw + q][hl];
      acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
    }
  } else if (t >= targets) {
    return;
  }
  float4 *o = (float4 *)(out + t * ldo + 64 * blockIdx.y + (a.sep ? a.outoff[blockIdx.z] : 0)) + hl;
  if (accumulate) { const float4 p = *o; acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w; }
  *o = acc;
}

// Segmented sum fused with the 64x64 output linear that consumes it (Eq. 4 𝓛_v, Eq. 5 𝓛_e):
// agg_t = Σ rows (as k_segsum<H>, stored for the backward), out_t = (agg_t·W + b) + resid_t.
// W sits in shared memory; the half-warp holding agg_t broadcasts its 64 values by shuffle.
template <int H, int U>
__global__ void __launch_bounds__(256) k_segsum_linear(int64_t targets, SegArgs a, float *__restrict__ agg,
                                                       const float *__restrict__ W, const float *__restrict__ bias,
                                                       const float *__restrict__ resid, float *__restrict__ out,
                                                       int agg_by_seg) {
  pdl_begin();
  __shared__ __align__(16) float sW[64][64];
  __shared__ float4 part[16][16];
  const int hw = threadIdx.x >> 4;
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / (16 * H);
  const int j = hw % H;
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const unsigned hmask = 0xffffu << (lane & 16);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t < targets) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k >= a.n) break;
      const SegSrc &S = a.s[k];
      const int64_t sg = S.segmap ? (int64_t)__ldg(S.segmap + t) : t + S.ptr_off;
      if (sg < 0) continue;
      int r0 = __ldg(S.ptr + sg), r1 = __ldg(S.ptr + sg + 1);
      if (H > 1) {
        const int len = r1 - r0;
        const int a0 = r0 + (int)((int64_t)len * j / H), a1 = r0 + (int)((int64_t)len * (j + 1) / H);
        r0 = a0; r1 = a1;
      }
      seg_rows<U>(S, r0, r1, hl, hmask, acc);
    }
  }
  // W_out is staged after the gather loop (its load latency overlaps the row loads)
#pragma unroll 8   // independent loads in flight (one latency, not one per iteration)
  for (int i = threadIdx.x; i < 64 * 64; i += 256) sW[i >> 6][i & 63] = W[i];
  if (H > 1) part[hw][hl] = acc;
  __syncthreads();
  if (H > 1) {
    if (j != 0 || t >= targets) return;
#pragma unroll
    for (int q = 1; q < H; ++q) {
      const float4 p = part[hw + q][hl];
      acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
    }
  } else if (t >= targets) {
    return;
  }
  if (agg_by_seg) {                                 // agg row = the segment (e.g. the bond of edge t)
    const int32_t sg = __ldg(a.s[0].segmap + t);
    if (sg >= 0) ((float4 *)(agg + (int64_t)sg * 64))[hl] = acc;
  } else {
    ((float4 *)(agg + t * 64))[hl] = acc;
  }
  float o[4] = {0.f, 0.f, 0.f, 0.f};
  // a target without a segment (a non-bond edge, Q16) has agg = 0: agg·W = 0 exactly, skipped
  const bool empty = agg_by_seg && __ldg(a.s[0].segmap + t) < 0;
  if (!empty) {
#pragma unroll
  for (int k = 0; k < 64; ++k) {
    const float c = (k & 3) == 0 ? acc.x : (k & 3) == 1 ? acc.y : (k & 3) == 2 ? acc.z : acc.w;
    const float ak = __shfl_sync(hmask, c, k >> 2, 16);
    const float4 w = *(const float4 *)&sW[k][4 * hl];
    o[0] = fmaf(ak, w.x, o[0]); o[1] = fmaf(ak, w.y, o[1]); o[2] = fmaf(ak, w.z, o[2]); o[3] = fmaf(ak, w.w, o[3]);
  }
  }
  if (bias) {
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] += __ldg(bias + 4 * hl + q);
  }
  if (resid) {
    const float4 r = __ldg((const float4 *)(resid + t * 64) + hl);
    o[0] += r.x; o[1] += r.y; o[2] += r.z; o[3] += r.w;
  }
  ((float4 *)(out + t * 64))[hl] = make_float4(o[0], o[1], o[2], o[3]);
}

// Embedding gradient dW_v[z] += Σ_{i: Z_i = z+1} dv_i (Eq. 2 adjoint): block b bins its 64
// consecutive atoms by species in shared memory (thread = column, atoms in index order), the
// per-block bins are reduced in block order by the batched reduction (reduce.cu) — no sort,
// no atomics, deterministic.
constexpr int EGB = 64;   // atoms per block
__global__ void __launch_bounds__(64) k_embed_grad(int64_t N, int nz, const int32_t *__restrict__ species,
                                                   const float *__restrict__ dv, float *__restrict__ part) {
  pdl_begin();
  extern __shared__ float bins[];                   // [nz][64]
  const int c = threadIdx.x;
  for (int i = c; i < nz * 64; i += 64) bins[i] = 0.f;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * EGB, i1 = min(N, i0 + EGB);
  for (int64_t i = i0; i < i1; ++i) {
    const int z = __ldg(species + i) - 1;
    bins[z * 64 + c] += __ldg(dv + i * 64 + c);
  }
  __syncthreads();
  float *p = part + (size_t)blockIdx.x * nz * 64;
  for (int i = c; i < nz * 64; i += 64) p[i] = bins[i];
}

// e' = e + 𝓛_e(agg) for every edge (Eq. 5, Q16): the 64x64 product is computed only for the
// B bond rows (tmp), non-bond edges get the bias alone; same rounding order as the fused
// epilogue ((x·W + b) + e).
__global__ void k_edge_update(int64_t E, const float4 *__restrict__ e, const float *__restrict__ bias,
                              const int32_t *__restrict__ bond_id, const float4 *__restrict__ tmp,
                              float4 *__restrict__ out) {
  pdl_begin();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // float4 index
  if (i >= E * 16) return;
  const int64_t row = i >> 4;
  const int c = (int)(i & 15);
  const int b = __ldg(bond_id + row);
  const float4 bb = make_float4(__ldg(bias + 4 * c), __ldg(bias + 4 * c + 1), __ldg(bias + 4 * c + 2),
                                __ldg(bias + 4 * c + 3));   // flat-parameter offsets need not be 16-B aligned
  const float4 ev = __ldg(e + i);
  float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
  if (b >= 0) x = __ldg(tmp + (int64_t)b * 16 + c);
  out[i] = make_float4((x.x + bb.x) + ev.x, (x.y + bb.y) + ev.y, (x.z + bb.z) + ev.z, (x.w + bb.w) + ev.w);
}

// column sums of a [rows, 64] matrix: per-block partials (fixed row ranges), reduced in block order
__global__ void __launch_bounds__(256) k_colsum_partial(int64_t rows, int64_t rpb, const float *__restrict__ D,
                                                        float *__restrict__ part) {
  pdl_begin();
  __shared__ float4 sh[16][16];
  const int t = threadIdx.x, c = t & 15, rl = t >> 4;
  const int64_t r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4   // 4 independent row loads in flight per thread
  for (int64_t r = r0 + rl; r < r1; r += 16) {
    const float4 v = __ldg((const float4 *)(D + r * 64) + c);
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  sh[rl][c] = s;
  __syncthreads();
  if (t < 16) {
    float4 a = sh[0][t];
    for (int k = 1; k < 16; ++k) { a.x += sh[k][t].x; a.y += sh[k][t].y; a.z += sh[k][t].z; a.w += sh[k][t].w; }
    ((float4 *)(part + blockIdx.x * 64))[t] = a;
  }
}

// ---------------------------------------------------------------------------
// heads
// ---------------------------------------------------------------------------
__global__ void k_heads_forces(int N, const int32_t *__restrict__ row_ptr, const float4 *__restrict__ vec,
                               const float *__restrict__ n_e, float *__restrict__ F) {
  pdl_begin();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= N) return;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  for (int e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
    float4 d = vec[e];
    float s = n_e[e] / d.w;
    fx += s * d.x; fy += s * d.y; fz += s * d.z;
  }
  fx = warp_sum(fx); fy = warp_sum(fy); fz = warp_sum(fz);
  if (lane == 0) { F[3 * i] = fx; F[3 * i + 1] = fy; F[3 * i + 2] = fz; }
}

__device__ __forceinline__ void lattice_G(const float *L, float G[9]) {
  float sh[3] = {0.f, 0.f, 0.f};
  for (int p = 0; p < 3; ++p) {
    float nx = L[3 * p], ny = L[3 * p + 1], nz = L[3 * p + 2];
    float inv = rsqrtf(nx * nx + ny * ny + nz * nz);
    sh[0] += nx * inv; sh[1] += ny * inv; sh[2] += nz * inv;
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) G[3 * a + b] = sh[a] * sh[b];
}

__global__ void k_heads_struct(const int32_t *__restrict__ atom_ptr, const float *__restrict__ lat,
                               const float *__restrict__ inv_n, const float *__restrict__ e_atom,
                               const float *__restrict__ M9, float *__restrict__ energy, float *__restrict__ epa,
                               float *__restrict__ stress) {
  pdl_begin();
  __shared__ double sh[10][128];
  int s = blockIdx.x, t = threadIdx.x;
  int a0 = atom_ptr[s], a1 = atom_ptr[s + 1];
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = a0 + t; i < a1; i += blockDim.x) {
    acc[0] += e_atom[i];
    const float *M = M9 + (int64_t)i * 9;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) acc[1 + 3 * a + b] += 0.5 * ((double)M[3 * a + b] + (double)M[3 * b + a]);
  }
  for (int k = 0; k < 10; ++k) sh[k][t] = acc[k];
  __syncthreads();
  for (int off = 64; off > 0; off >>= 1) {
    if (t < off)
      for (int k = 0; k < 10; ++k) sh[k][t] += sh[k][t + off];
    __syncthreads();
  }
  if (t == 0) {
    float G[9];
    lattice_G(lat + 9 * s, G);
    energy[s] = (float)sh[0][0];
    epa[s] = (float)(sh[0][0] * inv_n[s]);
    for (int k = 0; k < 9; ++k) stress[9 * s + k] = (float)(sh[1 + k][0] * inv_n[s] * G[k]);
  }
}

// ---------------------------------------------------------------------------
// loss + seeds (readings Q22, Q23)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double huber_d(double x, double d) {
  double ax = fabs(x);
  return ax < d ? 0.5 * x * x : d * (ax - 0.5 * d);
}
__device__ __forceinline__ float dhuber(float x, float d) { return fabsf(x) < d ? x : copysignf(d, x); }

struct LossArgs {
  int S, N;
  const float *epa, *forces, *stress, *mag;
  const float *l_epa, *l_forces, *l_stress, *l_mag;
  const uint8_t *l_mask;
  const int32_t *soa;
  const float *inv_n, *lat;
  float w_e, w_f, w_s, w_m, delta;
  double Sg, Ng, Mg;   // Mg < 0: count the mask here
};

__global__ void k_loss(LossArgs a, double *out) {
  pdl_begin();
  __shared__ double sh[5][1024];
  int t = threadIdx.x;
  double le = 0, lf = 0, ls = 0, lm = 0, cm = 0;
  // a NULL label array skips that task; a NULL mask with magmoms = all labelled
  for (int s = t; s < a.S; s += blockDim.x) {
    if (a.l_epa) le += huber_d((double)a.epa[s] - a.l_epa[s], a.delta);
    if (a.l_stress)
      for (int k = 0; k < 9; ++k) ls += huber_d((double)a.stress[9 * s + k] - a.l_stress[9 * s + k], a.delta);
  }
  for (int i = t; i < a.N; i += blockDim.x) {
    if (a.l_forces)
      for (int c = 0; c < 3; ++c) lf += huber_d((double)a.forces[3 * i + c] - a.l_forces[3 * i + c], a.delta);
    if (a.l_mag && (!a.l_mask || a.l_mask[i])) { lm += huber_d((double)a.mag[i] - a.l_mag[i], a.delta); cm += 1.0; }
  }
  sh[0][t] = le; sh[1][t] = lf; sh[2][t] = ls; sh[3][t] = lm; sh[4][t] = cm;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (t < off)
      for (int k = 0; k < 5; ++k) sh[k][t] += sh[k][t + off];
    __syncthreads();
  }
  if (t == 0) {
    double Mg = a.Mg >= 0 ? a.Mg : sh[4][0];
    double LE = a.w_e / a.Sg * sh[0][0], LF = a.w_f / (3.0 * a.Ng) * sh[1][0];
    double LS = a.w_s / (9.0 * a.Sg) * sh[2][0], LM = Mg > 0 ? a.w_m / Mg * sh[3][0] : 0.0;
    out[0] = LE + LF + LS + LM; out[1] = LE; out[2] = LF; out[3] = LS; out[4] = LM;
    out[5] = Mg;
  }
}

__global__ void k_seed_atom(LossArgs a, const double *lossbuf, float *__restrict__ d_eatom, float *__restrict__ dM9,
                            float *__restrict__ d_mag, float *__restrict__ seedF) {
  pdl_begin();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.N) return;
  int s = a.soa[i];
  float in = a.inv_n[s];
  d_eatom[i] = a.l_epa ? (float)(a.w_e / a.Sg) * dhuber(a.epa[s] - a.l_epa[s], a.delta) * in : 0.f;
  float G[9];
  lattice_G(a.lat + 9 * s, G);
  float cs = (float)(a.w_s / (9.0 * a.Sg));
  float ds[9];
  for (int k = 0; k < 9; ++k) ds[k] = a.l_stress ? cs * dhuber(a.stress[9 * s + k] - a.l_stress[9 * s + k], a.delta) : 0.f;
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q)
      dM9[(int64_t)i * 9 + 3 * p + q] = in * 0.5f * (ds[3 * p + q] * G[3 * p + q] + ds[3 * q + p] * G[3 * q + p]);
  float cf = (float)(a.w_f / (3.0 * a.Ng));
  for (int c = 0; c < 3; ++c)
    seedF[3 * i + c] = a.l_forces ? cf * dhuber(a.forces[3 * i + c] - a.l_forces[3 * i + c], a.delta) : 0.f;
  double Mg = lossbuf[5];
  d_mag[i] = (Mg > 0 && a.l_mag && (!a.l_mask || a.l_mask[i]))
                 ? (float)(a.w_m / Mg) * dhuber(a.mag[i] - a.l_mag[i], a.delta) : 0.f;
}

__global__ void k_seed_edge(int64_t E, const int32_t *__restrict__ center, const float4 *__restrict__ vec,
                            const float *__restrict__ seedF, float *__restrict__ dn) {
  pdl_begin();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  float4 d = vec[e];
  int i = center[e];
  dn[e] = (seedF[3 * i] * d.x + seedF[3 * i + 1] * d.y + seedF[3 * i + 2] * d.z) / d.w;
}

// ---------------------------------------------------------------------------
// utilities
// ---------------------------------------------------------------------------
__global__ void k_transpose(const int64_t *__restrict__ off, const int32_t *__restrict__ rc, const float *__restrict__ p,
                            float *__restrict__ wt) {
  pdl_begin();
  const int t = blockIdx.y;
  const int64_t o = off[t];
  const int R = rc[2 * t], C = rc[2 * t + 1];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * C) return;
  const int i = idx / C, j = idx % C;
  wt[o + (int64_t)j * R + i] = p[o + idx];
}

__global__ void k_embed(int64_t N, const int32_t *__restrict__ species, const float *__restrict__ W, float *__restrict__ v) {
  pdl_begin();
  int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t i = gt >> 4;
  int c4 = (int)(gt & 15);
  if (i >= N) return;
  ((float4 *)(v + i * 64))[c4] = ((const float4 *)(W + (int64_t)(species[i] - 1) * 64))[c4];
}

__global__ void k_finite(int64_t n, const float *__restrict__ g, int *bad) {
  pdl_begin();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && !isfinite(g[i])) atomicMin(bad, (int)i);
}

// Adam (PyTorch semantics, Q24), guarded by the finite check's flag: a non-finite gradient
// leaves params, m, v and the gradients untouched (the host raises after one synchronisation)
__global__ void k_adam(int64_t n, float *__restrict__ p, float *__restrict__ g, float *__restrict__ m,
                       float *__restrict__ v, float lr, float b1, float b2, float eps, float step_size,
                       float inv_sqrt_bc2, const int *__restrict__ bad) {
  pdl_begin();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || (bad && *bad != 0x7f7f7f7f)) return;
  float gi = g[i];
  float mi = b1 * m[i] + (1.f - b1) * gi;
  float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  p[i] -= step_size * mi / (sqrtf(vi) * inv_sqrt_bc2 + eps);
  g[i] = 0.f;
}

}  // namespace

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
void gate_fwd(chg_ctx *ctx, int64_t rows, const float *y, int ldy, GateLN ln, int mode, const float *w,
              const int32_t *i1, const int32_t *i2, const float *resid, float *out) {
  if (rows <= 0) return;
  ProfScope ps(ctx, "gate_fwd", 0.0, rows * (512.0 + 256.0 + (mode == GATE_MUL_W1W2 ? 520.0 : 256.0)));
  static const int bps = getenv("CHG_GATEF_BPS") ? atoi(getenv("CHG_GATEF_BPS")) : 3;   // A/B knob: blocks per SM (80 registers: 3 resident)
  const int grid = (int)std::min<int64_t>(ceil_div(rows * 16, 256), (int64_t)device_sm_count() * bps);   // 2 rows per warp, grid-stride
  launch_k(ctx, k_gate_fwd, grid, 256, 0, ctx->stream, rows, y, ldy, ln, mode, w, i1, i2, resid, out);
  check_launch(ctx);
}

void gate_bwd(chg_ctx *ctx, int64_t rows, const float *y, int ldy, GateLN ln, int mode, const float *w,
              const int32_t *i1, const int32_t *i2, const float *dout, const int32_t *didx, float *dy, int lddy,
              float *dw_acc, float *q1, float *q2, GateLNGrad g) {
  // one wave: 2 blocks per SM (128 registers -> 2 resident; A/B knob CHG_GATE_BPS)
  static const int bps = getenv("CHG_GATE_BPS") ? atoi(getenv("CHG_GATE_BPS")) : 2;
  const int64_t nbt = (int64_t)device_sm_count() * bps;
  int64_t rpb = std::max<int64_t>(64, (rows + nbt - 1) / nbt);
  int nb = rows > 0 ? ceil_div(rows, rpb) : 0;
  if (nb == 0) return;
  float *part = red_partial(ctx, (size_t)nb * 256);
  ProfScope ps(ctx, "gate_bwd", 0.0,
               rows * (512.0 + 260.0 + 512.0 + (mode == GATE_MUL_W ? 768.0 : mode == GATE_MUL_W1W2 ? 1032.0 : 0.0)));
  launch_k(ctx, k_gate_bwd, nb, 256, 0, ctx->stream, rows, rpb, y, ldy, ln, mode, w, i1, i2, dout, didx, dy, lddy, dw_acc, q1,
                                          q2, part, ctx->tc_round() ? 1 : 0);
  check_launch(ctx);
  RedJob j;                                        // LN affine gradients: batched reduction (reduce.cu)
  j.kind = 2; j.n = 256; j.splits = nb; j.stride = 256; j.part = part;
  j.W[0] = g.gc; j.W[1] = g.bc; j.W[2] = g.gg; j.W[3] = g.bg;
  red_push(ctx, j);
}

void segsum(chg_ctx *ctx, int64_t targets, float *out, int ldo, int accumulate, int nsrc, const SegSrc *src,
            const char *tag, int ncols, const int *outoff) {
  if (targets <= 0) return;
  if (ncols % 64 || ncols <= 0) CHG_THROW(CHG_ERR_STATE, "segsum: ncols %d not a multiple of 64", ncols);
  const int ng = ncols / 64;
  SegArgs a;
  a.n = nsrc;
  a.sep = outoff != nullptr;
  for (int k = 0; k < 3; ++k) a.outoff[k] = (outoff && k < nsrc) ? outoff[k] : 0;
  if (a.sep)
    for (int k = 0; k < nsrc; ++k)
      if (outoff[k] & 3) CHG_THROW(CHG_ERR_STATE, "segsum: output offsets must be multiples of 4");
  double bytes = targets * 256.0 * ng * (1 + accumulate);
  for (int k = 0; k < nsrc; ++k) {
    a.s[k] = src[k];
    bytes += src[k].rows * (256.0 * ng + (src[k].perm ? 4.0 : 0.0)) + targets * (src[k].segmap ? 12.0 : 8.0);
  }
  for (int k = 0; k < nsrc; ++k)
    if (((uintptr_t)src[k].in & 15) || ((uintptr_t)out & 15) || (ldo & 3) || (src[k].ld & 3))
      CHG_THROW(CHG_ERR_STATE, "segsum: 16-byte alignment required (in %p, out %p, ldo %d)", (const void *)src[k].in,
                (void *)out, ldo);
  // half-warps per target from the mean segment length (rows per half-warp ~ 16 or more)
  int64_t rows = 0;
  for (int k = 0; k < nsrc; ++k) rows += src[k].rows;
  const int64_t mean = rows / std::max<int64_t>(targets, 1);
  const int H = seg_split(mean, targets);
  ProfScope ps(ctx, tag, 0.0, bytes);
  const dim3 grid(ceil_div(targets * 16 * H, 256), ng, a.sep ? nsrc : 1);
  // 8 rows in flight per lane on long segments; 4 on short ones (fewer registers, more warps)
  auto go = [&](auto kern) { launch_k(ctx, kern, grid, 256, 0, ctx->stream, targets, out, ldo, accumulate, a); };
  const bool deep = mean >= 16;
  switch (H) {
    case 8: deep ? go(k_segsum<8, 8>) : go(k_segsum<8, 4>); break;
    case 4: deep ? go(k_segsum<4, 8>) : go(k_segsum<4, 4>); break;
    case 2: deep ? go(k_segsum<2, 8>) : go(k_segsum<2, 4>); break;
    default: deep ? go(k_segsum<1, 8>) : go(k_segsum<1, 4>); break;
  }
  check_launch(ctx);
}

void segsum_linear(chg_ctx *ctx, int64_t targets, int nsrc, const SegSrc *src, float *agg, const float *W,
                   const float *bias, const float *resid, float *out, const char *tag, int agg_by_seg) {
  if (agg_by_seg && (nsrc != 1 || !src[0].segmap)) CHG_THROW(CHG_ERR_STATE, "segsum_linear: agg_by_seg needs one mapped source");
  if (targets <= 0) return;
  SegArgs a;
  a.n = nsrc;
  a.sep = 0;
  double bytes = targets * (256.0 * (2 + (resid ? 1 : 0)));
  int64_t rows = 0;
  for (int k = 0; k < nsrc; ++k) {
    a.s[k] = src[k];
    rows += src[k].rows;
    bytes += src[k].rows * (256.0 + (src[k].perm ? 4.0 : 0.0)) + targets * (src[k].segmap ? 12.0 : 8.0);
    if ((uintptr_t)src[k].in & 15) CHG_THROW(CHG_ERR_STATE, "segsum_linear: 16-byte alignment required");
  }
  const int64_t mean = rows / std::max<int64_t>(targets, 1);
  const int H = seg_split(mean, targets);
  ProfScope ps(ctx, tag, 2.0 * targets * 64 * 64, bytes);
  const int grid = ceil_div(targets * 16 * H, 256);
  auto go = [&](auto kern) { launch_k(ctx, kern, grid, 256, 0, ctx->stream, targets, a, agg, W, bias, resid, out, agg_by_seg); };
  const bool deep = mean >= 16;
  switch (H) {
    case 8: deep ? go(k_segsum_linear<8, 8>) : go(k_segsum_linear<8, 4>); break;
    case 4: deep ? go(k_segsum_linear<4, 8>) : go(k_segsum_linear<4, 4>); break;
    case 2: deep ? go(k_segsum_linear<2, 8>) : go(k_segsum_linear<2, 4>); break;
    default: deep ? go(k_segsum_linear<1, 8>) : go(k_segsum_linear<1, 4>); break;
  }
  check_launch(ctx);
}

void embed_grad(chg_ctx *ctx, int64_t N, int n_species, const int32_t *species, const float *dv, float *dW) {
  if (N <= 0 || n_species <= 0) return;
  const int nb = ceil_div(N, EGB);
  float *part = red_partial(ctx, (size_t)nb * n_species * 64);
  {
    ProfScope ps(ctx, "embed_grad", 0.0, N * 260.0 + nb * n_species * 256.0);
    launch_k(ctx, k_embed_grad, nb, 64, n_species * 64 * 4, ctx->stream, N, n_species, species, dv, part);
    check_launch(ctx);
  }
  RedJob j;
  j.kind = 1; j.n = n_species * 64; j.splits = nb; j.stride = n_species * 64; j.part = part; j.W[0] = dW;
  red_push(ctx, j);
}

void edge_update(chg_ctx *ctx, int64_t E, const float *e, const float *bias, const int32_t *bond_id, const float *tmp,
                 float *out) {
  if (E <= 0) return;
  ProfScope ps(ctx, "edge_update", 0.0, E * (512.0 + 4.0) + 0.0);
  launch_k(ctx, k_edge_update, ceil_div(E * 16, 256), 256, 0, ctx->stream, E, (const float4 *)e, bias, bond_id,
                                                                 (const float4 *)tmp, (float4 *)out);
  check_launch(ctx);
}

void colsum(chg_ctx *ctx, int64_t rows, const float *D, float *grad) {
  if (rows <= 0 || ctx->no_param_grads) return;
  // 4 blocks per SM (296 blocks: 14.7 us, 592: 12.8 us per launch at C3; 1184 no better)
  const int64_t rpb = std::max<int64_t>(64, (rows + 591) / 592);
  const int nb = ceil_div(rows, rpb);
  float *part = red_partial(ctx, (size_t)nb * 64);
  {
    ProfScope ps(ctx, "colsum", 0.0, rows * 256.0 + nb * 256.0);
    launch_k(ctx, k_colsum_partial, nb, 256, 0, ctx->stream, rows, rpb, D, part);
    check_launch(ctx);
  }
  RedJob j;
  j.kind = 1; j.n = 64; j.splits = nb; j.stride = 64; j.part = part; j.W[0] = grad;
  red_push(ctx, j);
}

void heads_forces(chg_ctx *ctx, const chg_graph *g, const float *n_e, float *forces) {
  if (g->N <= 0) return;
  ProfScope ps(ctx, "heads", 0.0, g->E * 20.0 + g->N * 12.0);
  launch_k(ctx, k_heads_forces, ceil_div(g->N * 32, 256), 256, 0, ctx->stream, (int)g->N, g->row_ptr, g->vec, n_e, forces);
  check_launch(ctx);
}

void heads_struct(chg_ctx *ctx, const chg_graph *g, const float *e_atom, const float *M9, float *energy, float *epa,
                  float *stress) {
  if (g->S <= 0) return;
  ProfScope ps(ctx, "heads", 0.0, g->N * 40.0 + g->S * 48.0);
  launch_k(ctx, k_heads_struct, g->S, 128, 0, ctx->stream, g->atom_ptr, g->lattice_f, g->inv_natoms, e_atom, M9, energy, epa,
                                                stress);
  check_launch(ctx);
}

void loss_and_seeds(chg_ctx *ctx, const chg_graph *g, const float *epa, const float *forces, const float *stress,
                    const float *mag, const chg_labels &lab, const chg_loss_cfg &cfg, LossSeeds seeds) {
  LossArgs a;
  a.S = g->S; a.N = (int)g->N;
  a.epa = epa; a.forces = forces; a.stress = stress; a.mag = mag;
  a.l_epa = lab.energy_per_atom; a.l_forces = lab.forces; a.l_stress = lab.stress; a.l_mag = lab.magmom;
  a.l_mask = lab.magmom_mask;
  a.soa = g->struct_of_atom; a.inv_n = g->inv_natoms; a.lat = g->lattice_f;
  a.w_e = cfg.w_e; a.w_f = cfg.w_f; a.w_s = cfg.w_s; a.w_m = cfg.w_m; a.delta = cfg.huber_delta;
  a.Sg = cfg.n_struct_global > 0 ? (double)cfg.n_struct_global : (double)g->S;
  a.Ng = cfg.n_atoms_global > 0 ? (double)cfg.n_atoms_global : (double)g->N;
  a.Mg = cfg.n_magmom_global > 0 ? (double)cfg.n_magmom_global : -1.0;
  if (a.Sg <= 0) a.Sg = 1;
  if (a.Ng <= 0) a.Ng = 1;
  ProfScope ps(ctx, "loss", 0.0, g->N * 60.0 + g->S * 80.0 + g->E * 24.0);
  launch_k(ctx, k_loss, 1, 1024, 0, ctx->stream, a, ctx->d_loss);
  check_launch(ctx);
  if (g->N > 0) {
    float *seedF = ctx->getf("seedF", 3 * g->N);
    launch_k(ctx, k_seed_atom, ceil_div(g->N, 128), 128, 0, ctx->stream, a, ctx->d_loss, seeds.d_eatom, seeds.d_M9, seeds.d_mag,
                                                              seedF);
    check_launch(ctx);
    if (g->E > 0) {
      launch_k(ctx, k_seed_edge, ceil_div(g->E, 256), 256, 0, ctx->stream, g->E, g->center, g->vec, seedF, seeds.d_ne);
      check_launch(ctx);
    }
  }
}

void transpose_params(chg_ctx *ctx, const chg_model *m, float *wt) {
  if (m->n2d <= 0) return;
  ProfScope ps(ctx, "transpose", 0.0, 8.0 * m->P);
  launch_k(ctx, k_transpose, dim3(64, m->n2d), 256, 0, ctx->stream, m->d_toff, m->d_trc, m->params, wt);   // <= 16384 per tensor
  check_launch(ctx);
}

void fill_zero(chg_ctx *ctx, void *p, size_t bytes) {
  if (bytes) CUDA_OK(cudaMemsetAsync(p, 0, bytes, ctx->stream));
}

void embed_fwd(chg_ctx *ctx, int64_t N, const int32_t *species, const float *W, float *v) {
  if (N <= 0) return;
  ProfScope ps(ctx, "embed", 0.0, N * 260.0);
  launch_k(ctx, k_embed, ceil_div(N * 16, 256), 256, 0, ctx->stream, N, species, W, v);
  check_launch(ctx);
}

const void *adam_kernel() { return (const void *)k_adam; }

// finite check and the guarded Adam update back to back; the first non-finite flat index
// (0x7f7f7f7f = none; nothing is updated otherwise) is copied to the pinned host_flag on the
// stream — no synchronisation here (the caller checks it now or later)
void finite_adam(chg_ctx *ctx, int64_t n, float *p, float *g, float *m, float *v, float lr, float b1, float b2,
                 float eps, double bc1, double bc2, int *host_flag) {
  int *bad = ctx->d_flag;
  {
    ProfScope ps(ctx, "adam", 0.0, 4.0 * n);
    CUDA_OK(cudaMemsetAsync(bad, 0x7f, 4, ctx->stream));   // 0x7f7f7f7f means none
    launch_k(ctx, k_finite, ceil_div(n, 256), 256, 0, ctx->stream, n, g, bad);
    check_launch(ctx);
  }
  {
    const float step_size = (float)(lr / bc1);
    const float inv_sqrt_bc2 = (float)(1.0 / std::sqrt(bc2));
    ProfScope ps(ctx, "adam", 0.0, 28.0 * n);
    launch_k(ctx, k_adam, ceil_div(n, 256), 256, 0, ctx->stream, n, p, g, m, v, lr, b1, b2, eps, step_size, inv_sqrt_bc2, bad);
    check_launch(ctx);
  }
  CUDA_OK(cudaMemcpyAsync(host_flag, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
}

// dst[idx[r]] += src[r] for 64-float rows (idx injective: deterministic, no atomics)
namespace {
__global__ void k_rows_add(int64_t rows, const int32_t *__restrict__ idx, const float4 *__restrict__ src,
                           float4 *__restrict__ dst) {
  pdl_begin();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // float4 index
  if (i >= rows * 16) return;
  const int64_t r = i >> 4;
  const int c = (int)(i & 15);
  float4 *d = dst + (int64_t)__ldg(idx + r) * 16 + c;
  const float4 s = __ldg(src + i), o = *d;
  *d = make_float4(o.x + s.x, o.y + s.y, o.z + s.z, o.w + s.w);
}
}  // namespace

void rows_add(chg_ctx *ctx, int64_t rows, const int32_t *idx, const float *src, float *dst) {
  if (rows <= 0) return;
  ProfScope ps(ctx, "rows_add", 0.0, rows * (256.0 * 3 + 4.0));
  launch_k(ctx, k_rows_add, ceil_div(rows * 16, 256), 256, 0, ctx->stream, rows, idx, (const float4 *)src, (float4 *)dst);
  check_launch(ctx);
}
