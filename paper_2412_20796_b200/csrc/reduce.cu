// reduce.cu — batched, deterministic reduction of split partials into gradients.
//
// Every parameter gradient that is computed as per-CTA (or per-split) partials — the
// weight-gradient GEMMs (SIMT and tcgen05), LayerNorm affine gradients of the gated MLPs,
// the fused readout heads, the basis projections and the output-linear biases — used to
// need its own small reduction launch (~10 µs of latency each, ~50 per step).  Inside a
// backward layer they are recorded instead (red_push) and red_flush runs them all in ONE
// launch at the layer's end: block b serves a run of outputs of job j (found by binary search
// over the jobs' first blocks); the partial rows are summed in a fixed order that depends only
// on the job's shape, so results are deterministic.
#include "common.cuh"

namespace {

constexpr int MAXJ = 32;        // jobs per launch (kernel parameter: 32 x ~170 B, large-parameter launch)
struct RedBatch {
  RedJob j[MAXJ];
  int n;
};

__device__ __forceinline__ float *red_dst(const RedJob &J, int idx) {
  switch (J.kind) {
    case 0: {                               // weight gradient: (k, n) -> W chunk / bias
      const int k = idx / J.N, n = idx % J.N, c = n >> 6, nn = n & 63;
      if (k < J.K) {
        if (J.W[c] && k >= J.k0[c] && (J.kn[c] < 0 || k < J.k0[c] + J.kn[c]))
          return J.W[c] + (size_t)(k - J.k0[c]) * J.ldw[c] + nn;
        return nullptr;
      }
      return J.b[c] ? J.b[c] + nn : nullptr;
    }
    case 1: return J.W[0] + idx;            // flat
    case 2: return J.W[idx >> 6] + (idx & 63);   // LayerNorm gc | bc | gg | bg
    default: {                              // projection [31][C]: column c < 64 -> W[0], else W[1]
      const int n = idx / J.N, c = idx % J.N;
      return J.W[c >> 6] + n * 64 + (c & 63);
    }
  }
}

// block = qpb consecutive float4 quads of one job; its 256 threads are (quad q, group r),
// G = 256 / qpb groups: group r sums partial rows r, r + G, ... (fixed), then the G group
// sums of a quad are added in group order.  qpb depends only on the job's (n, splits), so
// the summation order — and the result — is the same on every run.  Tall jobs (few outputs,
// hundreds of splits: LayerNorm / bias / head partials) get many groups instead of one
// long serial chain per lane.
__global__ void __launch_bounds__(256) k_reduce_all(const __grid_constant__ RedBatch B) {
  pdl_begin();
  __shared__ float4 sh[256];
  __shared__ int sj;
  if (threadIdx.x == 0) {
    int lo = 0, hi = B.n - 1;
    while (lo < hi) {                       // last job with block0 <= blockIdx.x
      const int mid = (lo + hi + 1) >> 1;
      if (B.j[mid].block0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    sj = lo;
  }
  __syncthreads();
  const RedJob &J = B.j[sj];
  const int qpb = J.qpb, G = 256 / qpb;
  const int ql = threadIdx.x % qpb, grp = threadIdx.x / qpb;
  const int q = ((int)blockIdx.x - J.block0) * qpb + ql;   // quad index
  const int idx = 4 * q;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (idx < J.n) {
    if (J.stride % 4 == 0) {                // 16-B rows: one float4 per partial row
      const float4 *p = (const float4 *)J.part + q;
      const int64_t st4 = J.stride / 4;
#pragma unroll 8
      for (int sp = grp; sp < J.splits; sp += G) {
        const float4 u = __ldcg(p + (size_t)sp * st4);
        s.x += u.x; s.y += u.y; s.z += u.z; s.w += u.w;
      }
    } else {                                // odd row length (N = 1 or 9 heads): scalar loads
      const int m = min(4, J.n - idx);
      for (int sp = grp; sp < J.splits; sp += G) {
        const float *p = J.part + (size_t)sp * J.stride + idx;
        s.x += __ldcg(p);
        if (m > 1) s.y += __ldcg(p + 1);
        if (m > 2) s.z += __ldcg(p + 2);
        if (m > 3) s.w += __ldcg(p + 3);
      }
    }
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  if (grp != 0 || idx >= J.n) return;
  float4 t = sh[ql];
  for (int k = 1; k < G; ++k) {
    const float4 u = sh[k * qpb + ql];
    t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
  }
  const float v[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (idx + e >= J.n) break;
    float *d = red_dst(J, idx + e);
    if (d) *d += v[e];
  }
}

}  // namespace

float *red_partial(chg_ctx *ctx, size_t floats) {
  if (!ctx->red_on) return ctx->getf(ctx->ws_name("red_part_now"), floats);
  return ctx->getf("red_part_" + std::to_string(ctx->red_jobs.size()), floats);
}

void red_push(chg_ctx *ctx, RedJob j) {
  if (j.n <= 0 || ctx->no_param_grads) return;
  if ((uintptr_t)j.part & 15) CHG_THROW(CHG_ERR_STATE, "red_push: partial buffer must be 16-byte aligned");
  if (ctx->red_on) {
    ctx->red_jobs.push_back(j);
    return;
  }
  const bool was = ctx->red_on;
  ctx->red_on = true;
  ctx->red_jobs.push_back(j);
  red_flush(ctx);
  ctx->red_on = was;
}

void red_flush(chg_ctx *ctx) {
  for (size_t j0 = 0; j0 < ctx->red_jobs.size(); j0 += MAXJ) {
    RedBatch B;
    B.n = (int)std::min<size_t>(MAXJ, ctx->red_jobs.size() - j0);
    int blocks = 0;
    double bytes = 0;
    for (int k = 0; k < B.n; ++k) {
      B.j[k] = ctx->red_jobs[j0 + k];
      B.j[k].block0 = blocks;
      // ~8-16 partial rows per thread: G = 256 / qpb split groups (8..32, a power of two; measured)
      static const int gmax = getenv("CHG_RED_GMAX") ? atoi(getenv("CHG_RED_GMAX")) : 32;   // A/B knob
      static const int rpt = getenv("CHG_RED_RPT") ? atoi(getenv("CHG_RED_RPT")) : 16;      // A/B knob
      int G = 8;
      while (G < gmax && G * rpt < B.j[k].splits) G *= 2;
      B.j[k].qpb = 256 / G;
      blocks += ceil_div(ceil_div(B.j[k].n, 4), B.j[k].qpb);
      bytes += 4.0 * B.j[k].n * (B.j[k].splits + 2.0);
    }
    ProfScope ps(ctx, "reduce_all", 0.0, bytes);
    launch_k(ctx, k_reduce_all, blocks, 256, 0, ctx->stream, B);
    check_launch(ctx);
  }
  ctx->red_jobs.clear();
}
