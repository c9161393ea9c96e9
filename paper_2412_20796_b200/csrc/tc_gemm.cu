// tc_gemm.cu — tcgen05 (5th-gen tensor core) version of the gathered row GEMM.
//
// Same contract as k_rowgemm (gemm.cuh): out[m, n] = epi(Σ_k A(m, k) W(k, n) + b)
// with A gathered row by row from up to 4 tables.  One CTA = 128 rows (UMMA
// M = 128, cta_group::1), all output chunks; the accumulator lives in TMEM
// (128 lanes × up to 256 fp32 columns) and is read back by the 4 epilogue
// warps with tcgen05.ld (one TMEM lane = one output row = one thread).
//
// Operands: kind::tf32 (fp32 bits rounded to TF32 with cvt.rna), K-major,
// SWIZZLE_NONE canonical layout: element (row, k) of a tile with R rows at
// byte  (k/4)·(R·16) + row·16 + (k%4)·4   (core matrix = 8 rows × 16 B;
// SBO = 128 B between 8-row groups, LBO = R·16 B between 16-B K chunks).
// A is staged by all 128 threads (thread = row; the gather is the row index),
// B (weights, K-major copy) likewise; 2-stage smem ring over K chunks of 32,
// MMA completion tracked with tcgen05.commit -> mbarrier.
#include "gemm.cuh"

namespace {

constexpr int TCM = 128;   // rows per CTA
constexpr int KC = 32;     // K chunk per stage

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // descriptor version (sm_100)
  return d;                        // base offset 0, SWIZZLE_NONE (layout type 0)
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"(
                   (uint64_t)__cvta_generic_to_shared(bar))
               : "memory");
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// A(m, col..col+3) (segments are 32-column aligned on this path)
__device__ __forceinline__ float4 tc_loadA4(const AOp &A, int m, int col) {
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

// K-major weight row n (of chunk c), 4 consecutive k starting at k (k multiple of 4)
__device__ __forceinline__ float4 tc_loadB4(const Chunk &c, int n, int k) {
  if (n >= c.ncols) return make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (b < c.nwb && k >= c.wk0[b] && k < c.wk0[b + 1]) {
      // flat parameter offsets are not 16-B aligned: scalar (L1/L2-resident) loads
      const float *p = c.Wk[b] + (size_t)n * c.ldwk[b] + (k - c.wk0[b]);
      return make_float4(__ldg(p), __ldg(p + 1), __ldg(p + 2), __ldg(p + 3));
    }
  return make_float4(0.f, 0.f, 0.f, 0.f);
}

struct TcPlan {
  int lo;            // first A column of the union window
  int width;         // union window width (multiple of 32)
  int cpad[4];       // padded N of each chunk (multiple of 16)
  int coff[4];       // TMEM column offset of each chunk
  int ntot;          // total padded N
  uint32_t tmem_cols;
};

__global__ void __launch_bounds__(128, 1) k_rowgemm_tc(const RowGemm g, const TcPlan P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int m0 = blockIdx.x * TCM;
  const int NT = P.ntot;
  // smem carve: 2 stages of A [KC/4][128][4] and B [KC/4][NT][4] floats, barriers, tmem slot
  const uint32_t a_bytes = KC * TCM * 4, b_bytes = KC * NT * 4;
  uint8_t *sA[2] = {smem, smem + a_bytes + b_bytes};
  uint8_t *sB[2] = {smem + a_bytes, smem + 2 * a_bytes + b_bytes};
  uint64_t *bar = (uint64_t *)(smem + 2 * (a_bytes + b_bytes));
  uint32_t *tslot = (uint32_t *)(bar + 2);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  // instruction descriptor: D f32, A/B tf32, K-major, M = 128, N = chunk width
  auto idesc_for = [&](int n) -> uint32_t {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TCM >> 4) << 24);
  };

  const int nkc = P.width / KC;
  const int m = m0 + tid;
  const bool row_ok = m < g.M;
  bool started[4] = {false, false, false, false};
  for (int kc = 0; kc < nkc; ++kc) {
    const int s = kc & 1;
    if (kc >= 2) mbar_wait(&bar[s], ((kc - 2) >> 1) & 1);
    const int col0 = P.lo + kc * KC;   // A column of this chunk
    // --- stage A: thread = row, 8 float4 along k
    {
      uint8_t *dst = sA[s];
#pragma unroll
      for (int q = 0; q < KC / 4; ++q) {
        float4 v = row_ok ? tc_loadA4(g.A, m, col0 + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
        uint4 u = make_uint4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
        *(uint4 *)(dst + (q * TCM + tid) * 16) = u;
      }
    }
    // --- stage B: rows n of every chunk whose window covers this A chunk
    for (int c = 0; c < g.nchunk; ++c) {
      const Chunk &C = g.ch[c];
      int kk = col0 - C.a_k0;                 // k within the chunk's reduction
      if (kk < 0 || kk >= g.K) continue;
      for (int n = tid; n < P.cpad[c]; n += 128) {
        uint8_t *dst = sB[s];
#pragma unroll
        for (int q = 0; q < KC / 4; ++q) {
          float4 v = tc_loadB4(C, n, kk + 4 * q);
          uint4 u = make_uint4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
          *(uint4 *)(dst + (q * NT + P.coff[c] + n) * 16) = u;
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_base = smem_u32(sA[s]), b_base = smem_u32(sB[s]);
      for (int c = 0; c < g.nchunk; ++c) {
        const Chunk &C = g.ch[c];
        int kk = col0 - C.a_k0;
        if (kk < 0 || kk >= g.K) continue;
#pragma unroll
        for (int j = 0; j < KC / 8; ++j) {
          // K step of 8 tf32 = 2 core-matrix columns of 16 B
          uint64_t ad = make_desc(a_base + j * 2 * (TCM * 16), TCM * 16, 128);
          uint64_t bd = make_desc(b_base + j * 2 * (NT * 16) + P.coff[c] * 16, NT * 16, 128);
          mma_tf32(tmem + P.coff[c], ad, bd, idesc_for(P.cpad[c]), (started[c] || j > 0) ? 1u : 0u);
        }
        started[c] = true;
      }
      mma_commit(&bar[s]);
    }
  }
  // wait for the last commit (covers every MMA issued before it)
  {
    int last = nkc - 1;
    mbar_wait(&bar[last & 1], (last >> 1) & 1);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // --- epilogue: warp w reads TMEM lanes 32w..32w+31; thread = row
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < g.nchunk; ++c) {
    const Chunk &C = g.ch[c];
    for (int j0 = 0; j0 < P.cpad[c]; j0 += 32) {
      uint32_t r[32];
      if (j0 + 32 <= P.cpad[c]) {
        tmem_ld32(tmem + lane_base + P.coff[c] + j0, r);
      } else {
        // 16-column tail: load 32 (the allocation is wide enough), use 16
        tmem_ld32(tmem + lane_base + P.coff[c] + j0, r);
      }
      if (!row_ok) continue;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        int n = j0 + q;
        if (n >= C.ncols) continue;
        float v = __uint_as_float(r[q]);
        if (C.bias) v += __ldg(C.bias + n);
        if (C.pre) C.pre[(size_t)m * C.ldp + n] = v;
        if (g.act == 1) v = siluf_(v);
        if (C.mul) v *= dsiluf_(C.mul[(size_t)m * C.ldm + n]);
        if (C.resid) v += C.resid[(size_t)m * C.ldr + n];
        C.out[(size_t)m * C.ldo + n] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
}

}  // namespace

// Returns false if the GEMM does not fit this path (caller uses the SIMT kernel).
bool rowgemm_tc(chg_ctx *ctx, const RowGemm &g) {
  if (g.M <= 0 || g.K % KC != 0 || g.nchunk < 1) return false;
  TcPlan P{};
  int lo = 1 << 30, hi = 0, off = 0;
  for (int c = 0; c < g.nchunk; ++c) {
    const Chunk &C = g.ch[c];
    if (C.a_k0 % KC) return false;
    for (int b = 0; b < C.nwb; ++b)
      if (!C.Wk[b] || (C.wk0[b] % 4)) return false;
    lo = std::min(lo, C.a_k0);
    hi = std::max(hi, C.a_k0 + g.K);
    P.cpad[c] = std::max(16, (C.ncols + 15) / 16 * 16);
    P.coff[c] = off;
    off += (C.ncols + 31) / 32 * 32;   // keep 32-column TMEM alignment per chunk
  }
  int tot = 0;
  for (int s = 0; s < g.A.nseg; ++s) {
    const ASeg &S = g.A.seg[s];
    if (S.width % KC || S.ld % 4 || ((uintptr_t)S.base & 15)) return false;
    tot += S.width;
  }
  if (hi > tot) return false;
  P.lo = lo;
  P.width = hi - lo;
  P.ntot = off;
  if (P.ntot > 256) return false;
  P.tmem_cols = P.ntot <= 32 ? 32 : P.ntot <= 64 ? 64 : P.ntot <= 128 ? 128 : 256;
  size_t smem = 2 * (size_t)(KC * TCM * 4 + KC * P.ntot * 4) + 64;
  static bool attr = false;
  if (!attr) {
    CUDA_OK(cudaFuncSetAttribute(k_rowgemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  double cols = 0;
  for (int c = 0; c < g.nchunk; ++c) cols += g.ch[c].ncols;
  ProfScope ps(ctx, "rowgemm_tc", 2.0 * g.M * (double)g.K * cols,
               (double)g.M * (4.0 * P.width + 4.0 * cols * 2) + 4.0 * g.K * cols);
  k_rowgemm_tc<<<ceil_div(g.M, TCM), 128, smem, ctx->stream>>>(g, P);
  check_launch(ctx);
  return true;
}
