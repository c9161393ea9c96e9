// reduce.cu — batched, deterministic reduction of split partials into gradients.
//
// Every parameter gradient that is computed as per-CTA (or per-split) partials — the
// weight-gradient GEMMs (SIMT and tcgen05), LayerNorm affine gradients of the gated MLPs,
// the fused readout heads, the basis projections and the output-linear biases — used to
// need its own small reduction launch (~10 µs of latency each, ~50 per step).  Inside a
// backward layer they are recorded instead (red_push) and red_flush runs them all in ONE
// launch at the layer's end: block b serves 32 outputs of job j (found by binary search over
// the jobs' first blocks), warp w sums partial rows w, w+8, ..., warp 0 adds the 8
// subtotals in order — the same fixed order as a per-job reduction, so results are
// bit-identical and deterministic.
#include "common.cuh"

namespace {

constexpr int MAXJ = 32;        // jobs per launch (kernel parameter: 32 x ~170 B, large-parameter launch)
struct RedBatch {
  RedJob j[MAXJ];
  int n;
};

__global__ void __launch_bounds__(256) k_reduce_all(const __grid_constant__ RedBatch B) {
  __shared__ float sh[8][32];
  __shared__ int sj;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
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
  const int idx = ((int)blockIdx.x - J.block0) * 32 + lane;
  float s = 0.f;
  if (idx < J.n) {
#pragma unroll 8
    for (int sp = w; sp < J.splits; sp += 8) s += __ldcg(J.part + (size_t)sp * J.stride + idx);
  }
  sh[w][lane] = s;
  __syncthreads();
  if (w != 0 || idx >= J.n) return;
  float t = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) t += sh[k][lane];
  float *dst = nullptr;
  switch (J.kind) {
    case 0: {                               // weight gradient: (k, n) -> W chunk / bias
      const int k = idx / J.N, n = idx % J.N, c = n >> 6, nn = n & 63;
      if (k < J.K) {
        if (J.W[c] && k >= J.k0[c] && (J.kn[c] < 0 || k < J.k0[c] + J.kn[c])) dst = J.W[c] + (size_t)(k - J.k0[c]) * J.ldw[c] + nn;
      } else {
        dst = J.b[c] ? J.b[c] + nn : nullptr;
      }
      break;
    }
    case 1: dst = J.W[0] + idx; break;      // flat
    case 2: dst = J.W[idx >> 6] + (idx & 63); break;   // LayerNorm gc | bc | gg | bg
    case 3: {                               // projection [31][C]: column c < 64 -> W[0], else W[1]
      const int n = idx / J.N, c = idx % J.N;
      dst = J.W[c >> 6] + n * 64 + (c & 63);
      break;
    }
  }
  if (dst) *dst += t;
}

}  // namespace

float *red_partial(chg_ctx *ctx, size_t floats) {
  if (!ctx->red_on) return ctx->getf(ctx->ws_name("red_part_now"), floats);
  return ctx->getf("red_part_" + std::to_string(ctx->red_jobs.size()), floats);
}

void red_push(chg_ctx *ctx, RedJob j) {
  if (j.n <= 0) return;
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
      blocks += ceil_div(B.j[k].n, 32);
      bytes += 4.0 * B.j[k].n * (B.j[k].splits + 2.0);
    }
    ProfScope ps(ctx, "reduce_all", 0.0, bytes);
    k_reduce_all<<<blocks, 256, 0, ctx->stream>>>(B);
    check_launch(ctx);
  }
  ctx->red_jobs.clear();
}
