// tc_gemm.cu — tcgen05 (5th-gen tensor core) GEMM engines of the GatedMLP contractions.
//
// k_rowgemm_tc: out[m, n] = epi(Σ_k A(m, k) W(k, n) + b) with A gathered row by row from up to
// 4 tables (the concatenations of Eq. 4 / Eq. 5-6 are never materialised).  Persistent, one CTA
// per SM, 128-row tiles (UMMA M = 128, cta_group::1), fp32 accumulators double-buffered in TMEM.
// Warp roles (18 warps):
//   warps 0-3   A loaders: gathered rows by 16-B cp.async straight into SWIZZLE_128B K-major
//               stage slots (row r's 32 tf32 at bytes [128r, 128r+128), 16-B unit u stored at
//               u ^ (r & 7)); direct (non-gathered) segments by one TMA 2-D box per stage
//   warps 4-7   converters: thread = row, SiLU (second GatedMLP layer) + TF32 rounding in place,
//               fence.proxy.async, one mbarrier arrival per warp (skipped when the operand was
//               written TF32-rounded by its producer: the MMA then waits on the TMA barrier)
//   warp 8      weight image: cp.async.bulk of the packed K-major TF32 image (resident when it
//               fits, else a 3-slot ring)
//   warp 9      one thread issues tcgen05.mma.kind::tf32 and tcgen05.commit
//   warps 10-17 epilogue: tcgen05.ld (lane = row) -> bias / dSiLU(mul) / residual in registers ->
//               swizzled staging box -> TMA bulk tensor store (or TMA reduce-add store)
// k_wgrad_tc: weight gradients Σ_m A(m, k) D(m, n), rows m as the MMA K dimension, per-CTA
// partials reduced in a fixed order (reduce.cu).  See DESIGN.md §5.
// Debug / timing knobs (CHG_TC_SKIP, per-CTA trace) exist only in -DCHG_TC_DEBUG builds.
#include <cuda.h>
#include <cuda_bf16.h>

#include "gemm.cuh"

#ifdef CHG_TC_DEBUG
#define TC_SKIP(bit) ((skip & (bit)) != 0)
#else
#define TC_SKIP(bit) (false)
#endif

namespace {

constexpr int TCM = 128;   // rows per CTA (UMMA M)
constexpr int KC = 32;     // K chunk per pipeline stage


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

// tensor-map descriptors are fetched into the TMA unit's cache before the PDL wait, so their
// first use (the first A box, the first store) does not pay the fetch
__device__ __forceinline__ void prefetch_tmap(const void *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
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

// BF16 operands, fp32 accumulator (kind::f16; UMMA K = 16)
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

// two fp32 -> one packed bf16x2 (round to nearest even; lo in the low half)
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t *>(&h);
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"(
                   (uint64_t)__cvta_generic_to_shared(bar))
               : "memory");
}

// SiLU with the approximate reciprocal (MUFU.RCP): its error (~2 ulp fp32) is far
// below the TF32 rounding that follows, and it avoids the IEEE division sequence.
// round to nearest TF32, ties away from zero (= cvt.rna.tf32.f32) as two integer ops: add half
// a TF32 ulp to the bit pattern and clear the 13 dropped mantissa bits (a carry moves into the
// exponent exactly as rounding up does; Inf / NaN stay Inf / NaN)
__device__ __forceinline__ uint32_t to_tf32(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }

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

// TMA descriptors of the direct (non-gathered) A segments: one 32-column x 128-row box per
// stage lands, 128B-swizzled, exactly where the UMMA descriptor expects it
struct TcMaps {
  CUtensorMap m[4];
  int use[4];                      // 1: segment s is loaded by TMA
  CUtensorMap e[4];                // epilogue operand (mul or resid) of chunk c: 32 x 32 boxes
  int use_e[4];
  int nbuf;                        // operand boxes in flight per epilogue warp (0: plain loads)
  CUtensorMap o[4];                // output of chunk c (TMA-store epilogue): 32 x 32 boxes, SWIZZLE_128B
  CUtensorMap o2[4];               // second output (sout) of chunk c
  int tstore;                      // 1: lane = row epilogue, results leave through TMA stores
  int radd[4];                     // chunk c accumulates into its output (resid == out): TMA reduce-add store
  int nst;                         // staging boxes per epilogue warp (tstore)
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// out[box] += smem box (element-wise fp32 add at L2; one writer per element -> deterministic)
__device__ __forceinline__ void tma_store_add_2d(const CUtensorMap *map, uint32_t src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ float dsilu_fast(float x) {
  const float s = __fdividef(1.0f, 1.0f + __expf(-x));
  return s * (1.0f + x * (1.0f - s));
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

struct TcPlan {
  int lo;            // first A column of the union window
  int width;         // union window width (multiple of KC)
  int cpad[4];       // padded N of each chunk (multiple of 16)
  int coff[4];       // TMEM / image column offset of each chunk (multiple of 32)
  int ntot;          // total image rows N
  uint32_t tmem_cols;
  int bst;           // B smem slots: NSB (ring, one K chunk each) or nkc (whole image resident)
  int ngrp;          // MMA groups: adjacent chunks over the same A window issue ONE MMA of N = gn
  int gfirst[4], gn[4];
  int nsa;           // A stages
  int bres;          // 1: the whole weight image is loaded once per CTA (no per-stage B traffic)
  int noconv;        // 1: A arrives TF32-rounded by TMA: no conversion pass, the MMA waits on the load
  int lconv;         // 1: every A segment arrives by TMA and needs conversion: the weight warp issues
                     //    the A boxes and warps 0-7 all convert (thread = row, half a row each)
  int split;         // 1: 3xTF32 (mlp_precision 1): operands split x = hi + lo (both TF32), three MMAs
                     //    A_lo·B_hi + A_hi·B_lo + A_hi·B_hi per K step; stages hold [hi | lo]
  int bf16;          // 1: BF16 operands (mlp_precision 3): stages hold [fp32 as loaded | bf16 copy
                     //    (SWIZZLE_64B K-major, 64 B per row)], weight image in BF16, 2 MMAs (K = 16) per stage
  int nsb;           // B ring slots (<= NSB) when the image is not resident
  // compact weight image: K chunk kc holds only the chunks whose A window covers it (block-
  // diagonal GEMMs — the second GatedMLP layer, its adjoint — store half the columns), bnt
  // columns per K chunk, chunk c at column bcoff[kc][c] (-1: not active in kc)
  int bnt;
  int16_t bcoff[16][4];
  // column split of one-wave dense GEMMs (every chunk reads the same A window): CTA (tile =
  // blockIdx.x, part = blockIdx.y) computes chunks [cs_c0, cs_c1) only — image columns
  // [cs_n0, cs_n0 + cs_nt) — so small-M launches spread over more SMs with a smaller weight slice
  int csplit;
  int cs_c0[4], cs_c1[4], cs_n0[4], cs_nt[4];
  // split-K of one-wave single-chunk GEMMs with a plain epilogue: CTA (tile, y = blockIdx.y) sums
  // K chunks [y·kper, (y+1)·kper) and stores its raw partial tile at rows y·kmpad + m of the
  // partial buffer; k_splitk_sum adds the partials in order (+ bias + resid) — deterministic
  int ksplit, kper, kmpad;
};

// B image: img[kc][q][n][4] = tf32(W_chunk(n - bcoff[kc][c], k = lo + kc·KC - a_k0 + 4q + r))
__device__ __forceinline__ void pack_elem(const RowGemm &g, const TcPlan &P, uint32_t *__restrict__ img, int kc,
                                          int n, int k) {
  float v = 0.f;
  for (int c = 0; c < g.nchunk; ++c) {
    const Chunk &C = g.ch[c];
    if (P.bcoff[kc][c] < 0) continue;
    int j = n - P.bcoff[kc][c];
    if (j < 0 || j >= C.ncols) continue;
    int kk = P.lo + kc * KC - C.a_k0 + k;
    if (kk < 0 || kk >= g.K) continue;
    for (int b = 0; b < C.nwb; ++b)
      if (kk >= C.wk0[b] && kk < C.wk0[b + 1]) v = C.Wk[b][(size_t)j * C.ldwk[b] + (kk - C.wk0[b])];
  }
  if (P.bf16) {                                  // BF16 image: [kc][k/8][n][8] in the first half of kc's slot
    reinterpret_cast<__nv_bfloat16 *>(img)[(size_t)kc * P.bnt * KC * 2 + ((k >> 3) * P.bnt + n) * 8 + (k & 7)] =
        __float2bfloat16_rn(v);
    return;
  }
  const size_t at = (size_t)kc * P.bnt * KC + ((k >> 2) * P.bnt + n) * 4 + (k & 3);
  const uint32_t hi = to_tf32(v);
  img[at] = hi;
  if (P.split)                                   // lo image: the TF32 rounding of the remainder
    img[(size_t)(P.width / KC) * P.bnt * KC + at] = to_tf32(v - __uint_as_float(hi));
}

// every cached image of a model in one launch (blockIdx.y = site), after the weights changed
struct PackJob {
  RowGemm g;
  TcPlan P;
  uint32_t *img;
  int nkc;
};
__global__ void k_pack_all(const PackJob *__restrict__ jobs) {
  pdl_begin();
  const PackJob &J = jobs[blockIdx.y];
  const int per = J.P.bnt * KC, total = J.nkc * per;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int kc = idx / per, r = idx % per;
    pack_elem(J.g, J.P, J.img, kc, r / KC, r % KC);
  }
}

__global__ void k_pack_b(const RowGemm g, const TcPlan P, uint32_t *__restrict__ img) {
  pdl_begin();
  int kc = blockIdx.y;
  int idx = blockIdx.x * blockDim.x + threadIdx.x;   // over bnt * KC
  if (idx >= P.bnt * KC) return;
  int n = idx / KC, k = idx % KC;
  pack_elem(g, P, img, kc, n, k);
}


// ---------------------------------------------------------------------------
// warp-specialised persistent row GEMM (warp roles: file header)
// ---------------------------------------------------------------------------
constexpr int NSA_MAX = 10;         // A stages (16 KB each): P.nsa <= NSA_MAX, as many as shared memory allows
constexpr int NSB = 3;              // B stages (<= 32 KB each)
constexpr int WS_THREADS = 18 * 32;  // 4 loader, 4 converter, 1 B, 1 MMA, 8 epilogue warps
constexpr int NEPI = 8;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// epilogue of one 32x32 block (lane = column n, rows row0..row0+nrows): v = acc + b,
// optional pre-store, SiLU, ·SiLU'(mul), + resid.  Loads of a 16-row half are issued first.
template <bool PRE, bool MUL, bool RESID, bool ACT>
__device__ __forceinline__ void epi_rows(const Chunk &C, const float *stile, int lane, int row0, int nrows, int n,
                                         float bn) {
  // every dependent load of the block (32 rows) is issued before the first use: one memory
  // latency per 32x32 block
  float mv[32], rv[32];
  if (MUL || RESID) {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const size_t mr = (size_t)(row0 + rr);
      const bool ok = rr < nrows;
      if (MUL) mv[rr] = ok ? C.mul[mr * C.ldm + n] : 0.f;
      if (RESID) rv[rr] = ok ? C.resid[mr * C.ldr + n] : 0.f;
    }
  }
  if (nrows >= 32) {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const size_t mr = (size_t)(row0 + rr);
      float v = stile[rr * 33 + lane] + bn;
      if (PRE) C.pre[mr * C.ldp + n] = v;
      if (ACT) v = siluf_(v);
      if (MUL) v *= dsiluf_(mv[rr]);
      if (RESID) v += rv[rr];
      C.out[mr * C.ldo + n] = v;
    }
  } else {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      if (rr >= nrows) break;
      const size_t mr = (size_t)(row0 + rr);
      float v = stile[rr * 33 + lane] + bn;
      if (PRE) C.pre[mr * C.ldp + n] = v;
      if (ACT) v = siluf_(v);
      if (MUL) v *= dsiluf_(mv[rr]);
      if (RESID) v += rv[rr];
      C.out[mr * C.ldo + n] = v;
    }
  }
}

// epilogue rows with the mul / resid operand already in shared memory ([32 rows][32 cols], TMA)
template <bool MUL>
__device__ __forceinline__ void epi_rows_op(const Chunk &C, const float *stile, const float *ob, int lane, int row0,
                                            int nrows, int n, float bn) {
#pragma unroll 8
  for (int rr = 0; rr < 32; ++rr) {
    if (rr >= nrows) break;
    float v = stile[rr * 33 + lane] + bn;
    const float o = ob[rr * 32 + lane];
    if (MUL) v *= dsiluf_(o);
    else v += o;
    C.out[(size_t)(row0 + rr) * C.ldo + n] = v;
  }
}

__device__ __noinline__ void epi_rows_any(const Chunk &C, int act, const float *stile, int lane, int row0, int nrows,
                                          int n, float bn) {
  for (int rr = 0; rr < nrows; ++rr) {
    const size_t mr = (size_t)(row0 + rr);
    float v = stile[rr * 33 + lane] + bn;
    for (int k = 0; k < C.ngadd; ++k) {
      const int r = C.gidx[k] ? __ldg(C.gidx[k] + mr) : (int)mr;
      v += __ldg(C.gadd[k] + (size_t)r * C.ldga[k] + n);
    }
    if (C.pre) C.pre[mr * C.ldp + n] = v;
    if (act == 1) v = siluf_(v);
    if (C.mul) v *= dsiluf_(C.mul[mr * C.ldm + n]);
    if (C.resid) v += C.resid[mr * C.ldr + n];
    C.out[mr * C.ldo + n] = v;
  }
}

__global__ void __launch_bounds__(WS_THREADS, 1) k_rowgemm_tc(const __grid_constant__ RowGemm g, const TcPlan P,
                                                               const uint32_t *__restrict__ bimg, int ntiles,
                                                               int skip, const __grid_constant__ TcMaps TM) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SWIZZLE_128B operand atoms need 1024-B aligned stage bases
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int part = P.csplit > 1 ? (int)blockIdx.y : 0;
  const int NTg = P.bnt;                                // weight-image columns per K chunk (global image)
  const int NT = P.csplit > 1 ? P.cs_nt[part] : NTg;    // ... of this CTA's slice (shared memory)
  const int cb0 = P.csplit > 1 ? P.cs_c0[part] : 0, cb1 = P.csplit > 1 ? P.cs_c1[part] : g.nchunk;
  const uint32_t a_bytes = KC * TCM * 4, b_bytes = P.bf16 ? KC * NT * 2 : KC * NT * 4;
  // [hi | lo] in split mode, [fp32 | bf16] in BF16 mode
  const uint32_t a_stage = P.bf16 ? a_bytes + a_bytes / 2 : a_bytes << P.split, b_stage = b_bytes << P.split;
  const int NSA = P.nsa, NSBr = P.nsb;
  const uint32_t *bimg_lo = bimg + (size_t)(P.width / KC) * NTg * KC;
  uint8_t *sA = smem;                                   // [NSA][a_stage]
  uint8_t *sB = smem + NSA * a_stage;                   // [P.bst][b_stage]
  uint64_t *fullA = (uint64_t *)(sB + P.bst * b_stage);
  uint64_t *emptyA = fullA + NSA;
  uint64_t *loaded = emptyA + NSA;                      // cp.async completion per A stage
  uint64_t *fullB = loaded + NSA;
  uint64_t *emptyB = fullB + NSB;
  uint64_t *tfull = emptyB + NSB;
  uint64_t *tempty = tfull + 2;
  uint32_t *tslot = (uint32_t *)(tempty + 2);
  float *epi = (float *)(smem + NSA * a_stage + P.bst * b_stage + 8 * (3 * NSA + 2 * NSB + 4) + 16);  // [8][32][33]
  // epilogue operand boxes [8 warps][TM.nbuf][32 x 32] (1024-B aligned TMA targets) + their barriers
  float *obuf0 = (float *)(((uintptr_t)(epi + (TM.tstore ? 0 : NEPI * 32 * 33)) + 1023) & ~(uintptr_t)1023);
  float *stg0 = obuf0 + NEPI * TM.nbuf * 1024;          // TMA-store staging [8 warps][TM.nst][32 x 32]
  uint64_t *ebar = (uint64_t *)(stg0 + (TM.tstore ? NEPI * TM.nst * 1024 : 0));
  const uint32_t tcols = P.tmem_cols;                   // per accumulator buffer
  __shared__ uint64_t tr_entry, tr_setup;               // debug trace: kernel entry, setup done
  if (TC_SKIP(32) && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_entry));

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(2 * tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __shared__ uint64_t trace_ts[32], trace_ld[32], trace_cv[32], trace_mw[32], trace_ep[48];
  int nep = 0;
  if (TC_SKIP(32) && tid < 48) trace_ep[tid] = 0;
  if (tid == 0) {
    for (int i = 0; i < NSA; ++i) {
      mbar_init(&fullA[i], P.lconv ? 8 : 4);
      mbar_init(&emptyA[i], 1);
      mbar_init(&loaded[i], P.lconv ? 1 : 128);
    }
    for (int i = 0; i < NSB; ++i) { mbar_init(&fullB[i], 1); mbar_init(&emptyB[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], NEPI); }
    for (int i = 0; i < 2 * NEPI; ++i) mbar_init(&ebar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (TC_SKIP(32) && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_setup));
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < g.A.nseg && TM.use[k]) prefetch_tmap(&TM.m[k]);
      if (k < g.nchunk && TM.tstore) prefetch_tmap(&TM.o[k]);
      if (k < g.nchunk && TM.use_e[k]) prefetch_tmap(&TM.e[k]);
    }
  }
  pdl_begin();                                    // the setup above overlaps the predecessor's tail
  const uint32_t tmem = *tslot;
  if (TC_SKIP(32) && tid == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    trace_ts[0] = t;
  }

  // K chunks of this CTA: all, or [kcb, kcb + nkc) under a split-K; kc below is local, kcb + kc global
  const int kcb = P.ksplit > 1 ? (int)blockIdx.y * P.kper : 0;
  const int nkc = P.ksplit > 1 ? min(P.kper, P.width / KC - kcb) : P.width / KC;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_tiles * nkc;

  if (warp < 4 && !P.lconv) {
    // ---------------- A loaders (4 warps): cp.async 16 B straight into the 128B-swizzled slots ----------------
    // A stage layout (SWIZZLE_128B, K-major): row r's 32 tf32 occupy bytes [r*128, r*128+128),
    // 16-B unit u stored at unit u ^ (r & 7).  Thread = (q: unit, rb); rows rb + 16 i.
    // Row indices are loaded once per tile, so a chunk issues without dependent loads.
    const int q = tid & 7, rb = tid >> 3;
    int cur_tile = -1;
    int ridx[8][4];
    for (int gi = 0; gi < total; ++gi) {
      const int tl = gi / nkc, kc = gi % nkc;
      const int tile = blockIdx.x + tl * gridDim.x;
      const int sa = gi % NSA, ua = gi / NSA;
      if (tile != cur_tile) {
        cur_tile = tile;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int m = tile * TCM + rb + 16 * i;
#pragma unroll
          for (int sg = 0; sg < 4; ++sg)
            ridx[i][sg] = (sg < g.A.nseg && m < g.M) ? (g.A.seg[sg].idx ? __ldg(g.A.seg[sg].idx + m) : m) : -1;
        }
      }
      if (ua > 0) mbar_wait(&emptyA[sa], (ua - 1) & 1);
      const int col = P.lo + (kcb + kc) * KC;
      int seg = 0, start = 0;
      bool found = false;
#pragma unroll
      for (int sg = 0; sg < 4; ++sg)
        if (sg < g.A.nseg && !found) {
          if (col < start + g.A.seg[sg].width) { seg = sg; found = true; }
          else start += g.A.seg[sg].width;
        }
      const ASeg S = g.A.seg[seg];
      const int cin = col - start + 4 * q;
      const uint32_t dst0 = smem_u32(sA + sa * a_stage);
      bool tma = false;
#pragma unroll
      for (int sg = 0; sg < 4; ++sg)
        if (sg == seg) tma = TM.use[sg] != 0;
      if (tma) {                                       // one 16 KB box; the other 127 threads just arrive
        if (tid == 0) {
          mbar_expect_tx(&loaded[sa], a_bytes);
#pragma unroll
          for (int sg = 0; sg < 4; ++sg)
            if (sg == seg) tma_load_2d(dst0, &TM.m[sg], col - start, tile * TCM, &loaded[sa]);
        } else {
          mbar_arrive(&loaded[sa]);
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int r = -1;
#pragma unroll
        for (int sg = 0; sg < 4; ++sg)
          if (sg == seg) r = ridx[i][sg];
        if TC_SKIP(2) r = -1;                         // debug: no gather traffic
        const int row = rb + 16 * i;
        const uint32_t dst = dst0 + row * 128 + ((q ^ (row & 7)) << 4);
        if (r >= 0) cp_async16(dst, S.base + (size_t)r * S.ld + cin, 16);
        else cp_async16(dst, g.A.seg[0].base, 0);     // zero fill
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&loaded[sa])) : "memory");
      if (TC_SKIP(32) && tid == 0 && gi < 30) {       // debug trace: loader cadence
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace_ld[gi] = t;
      }
    }
  } else if (warp < 8) {
    // ---------------- A converters: thread = row; SiLU (GEMM2 input) + TF32 RN in place ----------------
    // warps 4-7 (the whole row), or warps 0-7 when every A box arrives by TMA (lconv: half a row
    // each — two warps per SMSP share the latency-bound conversion)
    const int r = tid & 127;
    const int sw = r & 7;
    const int hb = P.lconv ? (tid >> 7) * 4 : 0;      // first logical 16-B unit of this thread's part
    for (int gi = 0; gi < (P.noconv ? 0 : total); ++gi) {
      const int sa = gi % NSA, ua = gi / NSA;
      mbar_wait(&loaded[sa], ua & 1);
      uint4 *row = (uint4 *)(sA + sa * a_stage + r * 128);
      uint4 *row_lo = (uint4 *)(sA + sa * a_stage + a_bytes + r * 128);
      if (P.lconv) {
        // logical units hb..hb+3 (physical u ^ sw): SiLU, then TF32 (hi | lo) in place or the BF16 copy
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = *(const float4 *)&row[(hb + k) ^ sw];
        if (g.A.act == 1) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            v[k].x = silu_fast(v[k].x); v[k].y = silu_fast(v[k].y); v[k].z = silu_fast(v[k].z); v[k].w = silu_fast(v[k].w);
          }
        }
        if (P.bf16) {
          uint8_t *brow = sA + sa * a_stage + a_bytes + r * 64;
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = (hb >> 1) + c2;
            const float4 x = v[2 * c2], y = v[2 * c2 + 1];
            *reinterpret_cast<uint4 *>(brow + ((c ^ ((r >> 1) & 3)) << 4)) =
                make_uint4(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w), pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int pu = (hb + k) ^ sw;
            const float4 x = v[k];
            const uint4 h = make_uint4(to_tf32(x.x), to_tf32(x.y), to_tf32(x.z), to_tf32(x.w));
            row[pu] = h;
            if (P.split)
              row_lo[pu] = make_uint4(to_tf32(x.x - __uint_as_float(h.x)), to_tf32(x.y - __uint_as_float(h.y)),
                                      to_tf32(x.z - __uint_as_float(h.z)), to_tf32(x.w - __uint_as_float(h.w)));
          }
        }
      } else if (P.bf16) {
        // logical 16-B unit u of the row sits at u ^ (r & 7); BF16 unit c (k = 8c..8c+7) of the
        // copy goes to row r of the SWIZZLE_64B region at c ^ ((r >> 1) & 3)
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = *(const float4 *)&row[u ^ sw];
        uint8_t *brow = sA + sa * a_stage + a_bytes + r * 64;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float4 x = v[2 * c], y = v[2 * c + 1];
          if (g.A.act == 1) {
            x.x = silu_fast(x.x); x.y = silu_fast(x.y); x.z = silu_fast(x.z); x.w = silu_fast(x.w);
            y.x = silu_fast(y.x); y.y = silu_fast(y.y); y.z = silu_fast(y.z); y.w = silu_fast(y.w);
          }
          *reinterpret_cast<uint4 *>(brow + ((c ^ ((r >> 1) & 3)) << 4)) =
              make_uint4(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w), pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
        }
      } else if (!TC_SKIP(16)) {
        // all 8 loads first (independent: the row's 128 B), then convert and store — the
        // stores may alias later loads for the compiler, so interleaving would serialise them
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = *(const float4 *)&row[(k + sw) & 7];   // rotated: conflict-free
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int kk = (k + sw) & 7;
          float4 x = v[k];
          if (g.A.act == 1) { x.x = silu_fast(x.x); x.y = silu_fast(x.y); x.z = silu_fast(x.z); x.w = silu_fast(x.w); }
          const uint4 h = make_uint4(to_tf32(x.x), to_tf32(x.y), to_tf32(x.z), to_tf32(x.w));
          row[kk] = h;
          if (P.split)                                // exact remainder, rounded to TF32 again
            row_lo[kk] = make_uint4(to_tf32(x.x - __uint_as_float(h.x)), to_tf32(x.y - __uint_as_float(h.y)),
                                    to_tf32(x.z - __uint_as_float(h.z)), to_tf32(x.w - __uint_as_float(h.w)));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> async proxy (MMA)
      __syncwarp();
      if (lane == 0) mbar_arrive(&fullA[sa]);        // one arrival per converter warp
      if (TC_SKIP(32) && tid == 128 && gi < 30) {     // debug trace: converter cadence
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace_cv[gi] = t;
      }
    }
  } else if (warp == 8) {
    // ---------------- B producer (and, for lconv, the A TMA producer) ----------------
    auto issue_a = [&](int gi) {                        // lconv: stage gi's A box by TMA (one thread)
      const int tl = gi / nkc, kc = gi % nkc;
      const int tile = blockIdx.x + tl * gridDim.x;
      const int sa = gi % NSA, ua = gi / NSA;
      if (ua > 0) mbar_wait(&emptyA[sa], (ua - 1) & 1);
      const int col = P.lo + (kcb + kc) * KC;
      int start = 0;
      mbar_expect_tx(&loaded[sa], a_bytes);
#pragma unroll
      for (int sg = 0; sg < 4; ++sg) {
        if (sg >= g.A.nseg) break;
        const int w = g.A.seg[sg].width;
        if (col >= start && col < start + w)
          tma_load_2d(smem_u32(sA + sa * a_stage), &TM.m[sg], col - start, tile * TCM, &loaded[sa]);
        start += w;
      }
    };
    // weight chunk kc -> dst (hi, then lo in split mode): one bulk copy, or under a column split
    // the slice's columns, one copy per 16-B k group (image rows [kc][q][n] are column-contiguous)
    auto load_b = [&](uint8_t *dst, int kc, uint64_t *bar) {
      for (int h = 0; h <= P.split; ++h) {
        const uint32_t *src = (h ? bimg_lo : bimg) + (size_t)kc * NTg * KC;
        uint8_t *d = dst + h * b_bytes;
        if (P.csplit <= 1) {
          bulk_g2s(d, src, b_bytes, bar);
        } else {
          const int nq = P.bf16 ? KC / 8 : KC / 4;
          for (int q = 0; q < nq; ++q)
            bulk_g2s(d + q * NT * 16, reinterpret_cast<const uint8_t *>(src) + ((size_t)q * NTg + P.cs_n0[part]) * 16,
                     NT * 16, bar);
        }
      }
    };
    if (lane == 0 && P.lconv && P.bres) {               // resident image first, then the A stream
      if (total > 0) {
        mbar_expect_tx(&fullB[0], b_stage * nkc);
        for (int kc = 0; kc < nkc; ++kc) load_b(sB + kc * b_stage, kcb + kc, &fullB[0]);
      }
      for (int gi = 0; gi < total; ++gi) issue_a(gi);
    } else if (lane == 0 && P.lconv) {                  // A box and weight chunk of each stage in order
      for (int gi = 0; gi < total; ++gi) {
        issue_a(gi);
        const int kc = gi % nkc, sb = gi % NSBr, ub = gi / NSBr;
        if (ub > 0) mbar_wait(&emptyB[sb], (ub - 1) & 1);
        mbar_expect_tx(&fullB[sb], b_stage);
        load_b(sB + sb * b_stage, kcb + kc, &fullB[sb]);
      }
    } else if (lane == 0 && P.bres) {                   // whole image once: one barrier, nkc bulk copies
      if (total > 0) {
        if TC_SKIP(4) {
          mbar_arrive(&fullB[0]);
        } else {
          mbar_expect_tx(&fullB[0], b_stage * nkc);
          for (int kc = 0; kc < nkc; ++kc) load_b(sB + kc * b_stage, kcb + kc, &fullB[0]);
        }
      }
    } else if (lane == 0) {
      for (int gi = 0; gi < total; ++gi) {
        const int kc = gi % nkc, sb = gi % NSBr, ub = gi / NSBr;
        if (ub > 0) mbar_wait(&emptyB[sb], (ub - 1) & 1);
        if TC_SKIP(4) {                                 // debug: no weight traffic
          mbar_arrive(&fullB[sb]);
        } else {
          mbar_expect_tx(&fullB[sb], b_stage);
          load_b(sB + sb * b_stage, kcb + kc, &fullB[sb]);
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int gi = 0;
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int a = tl & 1, ua2 = tl >> 1;
        if (ua2 > 0) mbar_wait(&tempty[a], (ua2 - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        bool started[4] = {false, false, false, false};
        for (int kc = 0; kc < nkc; ++kc, ++gi) {
          const int sa = gi % NSA, ua = gi / NSA, sb = P.bres ? kc : gi % NSBr, ub = gi / NSBr;
          mbar_wait(P.noconv ? &loaded[sa] : &fullA[sa], ua & 1);
          if (!P.bres) mbar_wait(&fullB[sb], ub & 1);
          else if (gi == 0) mbar_wait(&fullB[0], 0);
          if (TC_SKIP(32) && gi < 30) {                // debug trace: operands ready
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace_mw[gi] = t;
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = smem_u32(sA + sa * a_stage), b_base = smem_u32(sB + sb * b_stage);
          const int col0 = P.lo + (kcb + kc) * KC;
          // MMA groups; under a column split one group: this CTA's chunks, N = its slice width
          const int ngr = P.csplit > 1 ? 1 : P.ngrp;
          for (int gr = 0; gr < ngr; ++gr) {
            const int c = P.csplit > 1 ? cb0 : P.gfirst[gr];
            const int gnv = P.csplit > 1 ? NT : P.gn[gr];
            const int boff = P.csplit > 1 ? 0 : P.bcoff[kcb + kc][c];
            const int kk = col0 - g.ch[c].a_k0;
            if (kk < 0 || kk >= g.K) continue;
            if (P.bf16) {                                 // BF16: K = 16 per MMA, A from the SWIZZLE_64B copy
              const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(gnv >> 3) << 17) |
                                     ((uint32_t)(TCM >> 4) << 24);
#pragma unroll
              for (int j = 0; j < KC / 16; ++j) {
                const uint64_t ad = make_desc(a_base + a_bytes + j * 32, 16, 512) | ((uint64_t)4 << 61);   // SWIZZLE_64B
                const uint64_t bd = make_desc(b_base + j * 2 * (NT * 16) + boff * 16, NT * 16, 128);
                if (TC_SKIP(8)) continue;
                mma_bf16(tmem + a * tcols + P.coff[c], ad, bd, idesc, (started[gr] || j > 0) ? 1u : 0u);
              }
              started[gr] = true;
              continue;
            }
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(gnv >> 3) << 17) |
                                   ((uint32_t)(TCM >> 4) << 24);
#pragma unroll
            for (int j = 0; j < KC / 8; ++j) {
              uint64_t ad = make_desc(a_base + j * 32, 16, 1024) | ((uint64_t)2 << 61);   // SWIZZLE_128B
              uint64_t bd = make_desc(b_base + j * 2 * (NT * 16) + boff * 16, NT * 16, 128);
              const uint32_t acc = (started[gr] || j > 0) ? 1u : 0u;
              if (TC_SKIP(8)) continue;                   // debug: no tensor-core work
              if (P.split) {                              // 3xTF32: small terms first, then hi·hi
                const uint64_t ad_lo = make_desc(a_base + a_bytes + j * 32, 16, 1024) | ((uint64_t)2 << 61);
                const uint64_t bd_lo = make_desc(b_base + b_bytes + j * 2 * (NT * 16) + boff * 16, NT * 16, 128);
                mma_tf32(tmem + a * tcols + P.coff[c], ad_lo, bd, idesc, acc);
                mma_tf32(tmem + a * tcols + P.coff[c], ad, bd_lo, idesc, 1u);
                mma_tf32(tmem + a * tcols + P.coff[c], ad, bd, idesc, 1u);
              } else {
                mma_tf32(tmem + a * tcols + P.coff[c], ad, bd, idesc, acc);
              }
            }
            started[gr] = true;
          }
          mma_commit(&emptyA[sa]);
          if (!P.bres) mma_commit(&emptyB[sb]);
          if (TC_SKIP(32) && gi < 30) {                // debug trace: MMA-side cadence
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace_ts[gi + 1] = t;
          }
        }
        mma_commit(&tfull[a]);
      }
      if TC_SKIP(32) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace_ts[31] = t;
      }
    }
  } else {
    // ---------------- epilogue (warps 10-17) ----------------
    const int lq = warp & 3;
    const uint32_t lane_base = (uint32_t)(lq * 32) << 16;
    float *stile = epi + (warp - 10) * (32 * 33);
    const int half = (warp - 10) >> 2;                // two warps per TMEM lane quarter split the blocks
    // this warp's 32x32 blocks (chunk, first column), the same in every tile
    int nmy = 0, mc[8], mj[8];
    {
      int blk = 0;
      for (int c = cb0; c < cb1; ++c)
        for (int j0 = 0; j0 < P.cpad[c]; j0 += 32, ++blk)
          if ((blk & 1) == half && nmy < 8) { mc[nmy] = c; mj[nmy] = j0; ++nmy; }
    }
    // mul / resid operand boxes arrive by TMA into per-warp buffers, issued ahead of use
    const int NB = TM.nbuf;
    float *obuf = obuf0 + (warp - 10) * (NB > 0 ? NB : 1) * 1024;
    uint64_t *obar = ebar + (warp - 10) * 2;
    uint32_t ophase = 0;                              // bit s: parity of slot s
    // blocks with a TMA operand, in list order: operand k of a tile uses slot k % NB
    int nop = 0, oi[8], kord[8];
    for (int i = 0; i < nmy; ++i) {
      kord[i] = -1;
      if (NB > 0 && TM.use_e[mc[i]]) { kord[i] = nop; oi[nop++] = i; }
    }
    auto issue_op = [&](int k, int row0) {            // operand k of this warp's list -> slot k % NB
      if (k >= nop || lane != 0) return;
      const int i = oi[k], c = mc[i], sl = k % NB;
      mbar_expect_tx(&obar[sl], 4096);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
        if (cc == c) tma_load_2d(smem_u32(obuf + sl * 1024), &TM.e[cc], mj[i], row0, &obar[sl]);
    };
    auto ep_mark = [&]() {
      if (TC_SKIP(32) && warp == 10 && lane == 0 && nep < 48) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace_ep[nep++] = t;
      }
    };
    if (TM.tstore) {
      // lane = row: the accumulator row as tcgen05.ld leaves it, bias / dSiLU(mul) / resid in
      // registers (operand box 128B-swizzled, conflict-free row reads), result written to a
      // swizzled staging box and stored by TMA (one bulk store per 32 x 32 block)
      float *stg = stg0 + (warp - 10) * TM.nst * 1024;
      int sc = 0;
      const int sw = lane & 7;
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int a = tl & 1;
        const int tile = blockIdx.x + tl * gridDim.x;
        const int row0 = tile * TCM + lq * 32;
        for (int k = 0; k < NB; ++k) issue_op(k, row0);
        // gather indices of this lane's row for the epilogue additions (shared by all chunks),
        // loaded while the accumulator is still being computed
        int gr[2] = {row0 + lane, row0 + lane};
        if (g.ch[0].ngadd && row0 + lane < g.M) {
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (k < g.ch[0].ngadd && g.ch[0].gidx[k]) gr[k] = __ldg(g.ch[0].gidx[k] + row0 + lane);
        }
        mbar_wait(&tfull[a], (tl >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        ep_mark();
        for (int i = 0; i < nmy; ++i) {
          const int c = mc[i], j0 = mj[i];
          const Chunk &C = g.ch[c];
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + a * tcols + P.coff[c] + j0, r);
          float *v = reinterpret_cast<float *>(r);
          if (C.bias) {
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] += __ldg(C.bias + j0 + q);
          }
          const int m = row0 + lane;
          if (C.ngadd && m < g.M) {                     // gathered row additions (factorised layer 1)
            // row indices hoisted per tile (gr); every table's 16 columns of a half-block are in
            // flight together: one memory latency per half-block, not one per table
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float4 u[2][4];
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                if (k >= C.ngadd) break;
                const float4 *src = reinterpret_cast<const float4 *>(C.gadd[k] + (size_t)gr[k] * C.ldga[k] + j0) + 4 * h;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) u[k][q4] = __ldg(src + q4);
              }
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                if (k >= C.ngadd) break;
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  float *w = v + 16 * h + 4 * q4;
                  w[0] += u[k][q4].x; w[1] += u[k][q4].y; w[2] += u[k][q4].z; w[3] += u[k][q4].w;
                }
              }
            }
          }
          if (kord[i] >= 0) {
            const int sl = kord[i] % NB;
            mbar_wait(&obar[sl], (ophase >> sl) & 1);
            ophase ^= 1u << sl;
            const float4 *ob = reinterpret_cast<const float4 *>(obuf + sl * 1024) + lane * 8;
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
              const float4 u = ob[q4 ^ sw];
              if (C.mul) {
                v[4 * q4] *= dsilu_fast(u.x); v[4 * q4 + 1] *= dsilu_fast(u.y);
                v[4 * q4 + 2] *= dsilu_fast(u.z); v[4 * q4 + 3] *= dsilu_fast(u.w);
              } else {
                v[4 * q4] += u.x; v[4 * q4 + 1] += u.y; v[4 * q4 + 2] += u.z; v[4 * q4 + 3] += u.w;
              }
            }
            __syncwarp();
            issue_op(kord[i] + NB, row0);                // slot consumed: next box of this tile
          } else if ((C.mul || C.resid) && !TM.radd[c] && m < g.M) {   // operand without a TMA map: own row
            const float *op = C.mul ? C.mul + (size_t)m * C.ldm + j0 : C.resid + (size_t)m * C.ldr + j0;
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = C.mul ? v[q] * dsilu_fast(__ldg(op + q)) : v[q] + __ldg(op + q);
          }
          if TC_SKIP(1) continue;                       // debug: no epilogue stores
          // pass 0: out (TF32-rounded if round_out); pass 1: sout = tf32(SiLU(v))
          for (int pass = 0; pass < (C.sout ? 2 : 1); ++pass) {
            float *st = stg + (sc % TM.nst) * 1024;
            if (lane == 0) {                            // staging box free (its previous store has read it)
              if (TM.nst > 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
            float4 *srow = reinterpret_cast<float4 *>(st) + lane * 8;
            if (pass == 0 && C.round_out) {
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4)
                srow[q4 ^ sw] = make_float4(tf32_round(v[4 * q4]), tf32_round(v[4 * q4 + 1]), tf32_round(v[4 * q4 + 2]),
                                            tf32_round(v[4 * q4 + 3]));
            } else if (pass == 0) {
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) srow[q4 ^ sw] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
            } else {
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4)
                srow[q4 ^ sw] = make_float4(tf32_round(silu_fast(v[4 * q4])), tf32_round(silu_fast(v[4 * q4 + 1])),
                                            tf32_round(silu_fast(v[4 * q4 + 2])), tf32_round(silu_fast(v[4 * q4 + 3])));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && row0 < g.M) {
#pragma unroll
              for (int cc = 0; cc < 4; ++cc)
                if (cc == c) {
                  if (TM.radd[cc]) tma_store_add_2d(&TM.o[cc], smem_u32(st), j0, row0);
                  else tma_store_2d(pass ? &TM.o2[cc] : &TM.o[cc], smem_u32(st), j0,
                                    row0 + (P.ksplit > 1 ? (int)blockIdx.y * P.kmpad : 0));
                }
            }
            ++sc;
          }
          ep_mark();
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    } else
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int a = tl & 1;
      const int tile = blockIdx.x + tl * gridDim.x;
      const int row0 = tile * TCM + lq * 32;
      const int nrows = min(32, g.M - row0);
      for (int k = 0; k < NB; ++k) issue_op(k, row0);   // overlaps the accumulator wait
      mbar_wait(&tfull[a], (tl >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      ep_mark();
      // 32x32 blocks go TMEM -> registers (lane = row) -> smem -> registers
      // (lane = column) so that every global access is a coalesced 128-B row run
      for (int i = 0; i < nmy; ++i) {
        const int c = mc[i], j0 = mj[i];
        const Chunk &C = g.ch[c];
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + a * tcols + P.coff[c] + j0, r);
        if TC_SKIP(1) continue;                         // debug: no epilogue stores
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) stile[lane * 33 + qq] = __uint_as_float(r[qq]);
        __syncwarp();
        const int n = j0 + lane;
        const bool opd = kord[i] >= 0;
        if (opd) {                                    // operand box of this block has landed
          const int sl = kord[i] % NB;
          mbar_wait(&obar[sl], (ophase >> sl) & 1);
          ophase ^= 1u << sl;
        }
        ep_mark();
        if (n < C.ncols) {
          const float bn = C.bias ? __ldg(C.bias + n) : 0.f;
          if (opd) {
            const float *ob = obuf + (kord[i] % NB) * 1024;
            if (C.mul) epi_rows_op<true>(C, stile, ob, lane, row0, nrows, n, bn);
            else epi_rows_op<false>(C, stile, ob, lane, row0, nrows, n, bn);
          } else {
            // flags are uniform per 32x32 block: one specialised row loop per combination
            const int code = (C.pre ? 1 : 0) | (C.mul ? 2 : 0) | (C.resid ? 4 : 0) | (g.act == 1 ? 8 : 0) |
                             (C.ngadd ? 16 : 0);
            switch (code) {
              case 0: epi_rows<false, false, false, false>(C, stile, lane, row0, nrows, n, bn); break;
              case 2: epi_rows<false, true, false, false>(C, stile, lane, row0, nrows, n, bn); break;
              case 4: epi_rows<false, false, true, false>(C, stile, lane, row0, nrows, n, bn); break;
              default: epi_rows_any(C, g.act, stile, lane, row0, nrows, n, bn); break;
            }
          }
        }
        __syncwarp();
        ep_mark();
        if (opd) issue_op(kord[i] + NB, row0);          // slot free again: next box of this tile
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);        // one arrival per epilogue warp
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (TC_SKIP(32) && blockIdx.x == 0 && tid == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    printf("TRACE tiles %d nkc %d grid %d | entry->setup %.2f ->pdl %.2f | start->chunk ends (us):", my_tiles, nkc,
           (int)gridDim.x, (tr_setup - tr_entry) * 1e-3, (trace_ts[0] - tr_setup) * 1e-3);
    for (int i = 1; i <= min(30, total); ++i) printf(" %.2f", (trace_ts[i] - trace_ts[0]) * 1e-3);
    printf(" | loader issued:");
    for (int i = 0; i < min(30, total); ++i) printf(" %.2f", (trace_ld[i] - trace_ts[0]) * 1e-3);
    printf(" | converted:");
    for (int i = 0; i < min(30, total); ++i) printf(" %.2f", (trace_cv[i] - trace_ts[0]) * 1e-3);
    printf(" | mma ready:");
    for (int i = 0; i < min(30, total); ++i) printf(" %.2f", (trace_mw[i] - trace_ts[0]) * 1e-3);
    printf(" | mma_done %.2f end %.2f", (trace_ts[31] - trace_ts[0]) * 1e-3, (t - trace_ts[0]) * 1e-3);
    printf(" | epi(w10):");
    for (int i = 0; i < 48 && trace_ep[i] > trace_ts[0]; ++i) printf(" %.2f", (trace_ep[i] - trace_ts[0]) * 1e-3);
    printf("\n");
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * tcols) : "memory");
}


// ---------------------------------------------------------------------------
// tcgen05 weight-gradient GEMM:  G[k, n] = Σ_m A(m, k) · D(m, n)
//   UMMA view: D_mma[M = k][N = n] = Σ_{K = m} A_mma[k][m] · B_mma[n][m].  Both
//   operands are staged K-MAJOR (MN-major tf32 operands read as zeros on this
//   part, tools/mma_probe.cu): producer lanes own one row m each, load 4
//   consecutive columns with one ld.global.v4 (gathered row, TF32-rounded in
//   registers, SiLU for A when act) and scatter them as 4-byte stores into 4
//   swizzled K-major rows (k or n) at column m — a free transpose, conflict-free.
//   Stage = 32 rows m: A_T [Kpad rows][128 B], D_T [N rows][128 B], SWIZZLE_128B.
//   Rows are split across persistent CTAs; each CTA accumulates its k tiles
//   (M = 128, ≤ 2) × N in TMEM and writes one partial [Kp][N] (TMA bulk stores of 32 x 32
//   blocks staged in the idle stage buffers); partials are reduced in a fixed order by the
//   batched reduction (reduce.cu).  The bias (column sums of D) is summed by the producers
//   from the staged K-major D rows.  Warps 0-14 produce, warp 15 issues MMAs, warps 0-3 run
//   the epilogue.
// ---------------------------------------------------------------------------
constexpr int WG_NST = 3;
constexpr int WG_NPW = 15;                 // producer warps
constexpr int WG_THREADS = (WG_NPW + 1) * 32;

struct WgPlan {
  int Kpad;        // rows of A_T (multiple of 128)
  int ktiles;      // Kpad / 128
  int Npad;        // N
  int Kp;          // rows written to the partial (K or K+1 with bias)
  int ones_col;    // K if the bias ones row is used, else -1
  int rows_per_cta;
  uint32_t tmem_cols;
  int split;       // 1: 3xTF32 — stage = [A_T hi | D_T hi | A_T lo | D_T lo], three MMAs per K step
  int nst;         // stages in the ring (<= WG_NST)
};

__device__ __forceinline__ uint32_t kmaj_swz(int r, int m) {   // byte offset of element (row r, K index m)
  return (uint32_t)(r * 128 + ((((m >> 2) ^ (r & 7))) << 4) + (m & 3) * 4);
}

__global__ void __launch_bounds__(WG_THREADS, 1) k_wgrad_tc(const __grid_constant__ WGrad g, const WgPlan P, float *__restrict__ partial,
                                                             int skip, const __grid_constant__ CUtensorMap pmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t a_bytes = P.Kpad * 128, d_bytes = P.Npad * 128;
  const uint32_t lo_off = a_bytes + d_bytes;                  // split: lo half of a stage
  const uint32_t st_bytes = lo_off << P.split;
  const int NST = P.nst;
  uint64_t *full = (uint64_t *)(smem + NST * st_bytes);
  uint64_t *empty = full + WG_NST;
  uint64_t *done = empty + WG_NST;
  uint32_t *tslot = (uint32_t *)(done + 1);
  float *sbias = (float *)(smem + NST * st_bytes + 8 * (2 * WG_NST + 1) + 16);   // [WG_NPW][256]
  __shared__ int s_seg[8], s_col[8];        // A block -> segment, column within the segment

  const int r0 = blockIdx.x * P.rows_per_cta;
  const int r1 = min(g.M, r0 + P.rows_per_cta);
  const int nchunks = r1 > r0 ? (r1 - r0 + 31) / 32 : 0;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) { mbar_init(&full[i], g.K / 32 + g.N / 32); mbar_init(&empty[i], 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 8) {
    int q = 0, start = 0;
    while (q < g.A.nseg - 1 && 32 * tid >= start + g.A.seg[q].width) start += g.A.seg[q++].width;
    s_seg[tid] = q;
    s_col[tid] = 32 * tid - start;
  }
  for (int i = tid; i < WG_NPW * 256; i += blockDim.x) sbias[i] = 0.f;
  // constant rows k = K..Kpad of A_T: zeros, and the ones row for the bias
  for (int s = 0; s < NST; ++s)
    for (int idx = tid; idx < (P.Kpad - g.K) * 32; idx += blockDim.x) {
      const int r = g.K + idx / 32, m = idx % 32;
      *(float *)(smem + s * st_bytes + kmaj_swz(r, m)) = (r == P.ones_col) ? 1.0f : 0.0f;
      if (P.split) *(float *)(smem + s * st_bytes + lo_off + kmaj_swz(r, m)) = 0.0f;
    }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  pdl_begin();                                    // the setup above overlaps the predecessor's tail
  const uint32_t tmem = *tslot;

  if (warp < WG_NPW) {
    // ---------------- producers: lane = row m of the chunk ----------------
    // Jobs are (chunk c, 32-column block b) over [A columns | D columns], j = c·nb + b,
    // dealt round-robin to the WG_NPW producer warps.  A job loads its lane's 128-B row
    // segment (8 x ld.v4), rounds to TF32 (SiLU first for A when act) and scatters it
    // into 32 K-major rows at column `lane`.  The next job's data and the row index of
    // the one after are loaded while the current job is being stored.
    const int nba = g.K / 32, nbd = g.N / 32, nb = nba + nbd;   // 32-column blocks
    const int njobs = nchunks * nb;
    auto row_of = [&](int j) -> int {
      if (j >= njobs || TC_SKIP(2)) return -1;
      const int c = j / nb, b = j - c * nb;
      const int m = r0 + c * 32 + lane;
      if (m >= r1) return -1;
      if (b < nba) {
        const int32_t *ix = g.A.seg[s_seg[b]].idx;
        return ix ? __ldg(ix + m) : m;
      }
      return g.didx ? __ldg(g.didx + m) : m;
    };
    auto load = [&](int j, int row, float4 (&v)[8]) {
      const float *src = nullptr;
      if (j < njobs && row >= 0) {
        const int b = j % nb;
        if (b < nba) {
          const ASeg &S = g.A.seg[s_seg[b]];
          src = S.base + (size_t)row * S.ld + s_col[b];
        } else {
          src = g.D + (size_t)row * g.ldd + 32 * (b - nba);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = src ? __ldg((const float4 *)src + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    int j = warp;
    int row_n = row_of(j + WG_NPW);
    float4 cur[8];
    load(j, row_of(j), cur);
    for (; j < njobs; j += WG_NPW) {
      float4 nxt[8];
      load(j + WG_NPW, row_n, nxt);
      row_n = row_of(j + 2 * WG_NPW);
      const int c = j / nb, b = j - c * nb, s = c % NST, u = c / NST;
      if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
      uint8_t *stA = smem + s * st_bytes;
      const bool isA = b < nba;
      uint8_t *base = isA ? stA : stA + a_bytes;
      const int r0b = isA ? 32 * b : 32 * (b - nba);
      const bool act = isA && g.A.act == 1;
      if (P.split) {                                   // 3xTF32: hi and the rounded remainder lo
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float v = act ? silu_fast(x[q]) : x[q];
            const uint32_t h = to_tf32(v);
            const uint32_t o = kmaj_swz(r0b + 4 * k + q, lane);
            *(uint32_t *)(base + o) = h;
            *(uint32_t *)(base + lo_off + o) = to_tf32(v - __uint_as_float(h));
          }
        }
      } else if (act) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) *(uint32_t *)(base + kmaj_swz(r0b + 4 * k + q, lane)) = to_tf32(silu_fast(x[q]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) *(uint32_t *)(base + kmaj_swz(r0b + 4 * k + q, lane)) = to_tf32(x[q]);
        }
      }
      if (!isA && g.bias) {
        // lane n sums K-major row r0b + n (the 32 rows m of this chunk), read back from smem
        __syncwarp();
        const uint8_t *row = base + (r0b + lane) * 128;
        float acc = 0.f;
#pragma unroll
        for (int uu = 0; uu < 8; ++uu) {
          float4 v = *(const float4 *)(row + (uu << 4));
          if (P.split) {                               // hi + lo: the value to 22 bits
            const float4 w = *(const float4 *)(row + lo_off + (uu << 4));
            v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
          }
          acc += (v.x + v.y) + (v.z + v.w);
        }
        sbias[warp * 256 + r0b + lane] += acc;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
#pragma unroll
      for (int k = 0; k < 8; ++k) cur[k] = nxt[k];
    }
    if (g.bias) {                                       // bias row K of this CTA's partial
      asm volatile("bar.sync 1, %0;" ::"r"(WG_NPW * 32) : "memory");
      float *Pout = partial + (size_t)blockIdx.x * P.Kp * g.N;
      for (int n = tid; n < g.N; n += WG_NPW * 32) {
        float t = 0.f;
        for (int w = 0; w < WG_NPW; ++w) t += sbias[w * 256 + n];   // fixed order: deterministic
        Pout[(size_t)g.K * g.N + n] = t;
      }
    }
  } else {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(P.Npad >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % NST, u = c / NST;
        mbar_wait(&full[s], u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t baseA = smem_u32(smem + s * st_bytes), baseD = baseA + a_bytes;
        for (int tt = 0; tt < P.ktiles; ++tt) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint64_t ad = make_desc(baseA + tt * 16384 + j * 32, 16, 1024) | ((uint64_t)2 << 61);
            uint64_t bd = make_desc(baseD + j * 32, 16, 1024) | ((uint64_t)2 << 61);
            const uint32_t acc = (c > 0 || j > 0) ? 1u : 0u;
            if (TC_SKIP(8)) continue;
            if (P.split) {                             // 3xTF32: A_lo·D_hi + A_hi·D_lo + A_hi·D_hi
              const uint64_t ad_lo = make_desc(baseA + lo_off + tt * 16384 + j * 32, 16, 1024) | ((uint64_t)2 << 61);
              const uint64_t bd_lo = make_desc(baseD + lo_off + j * 32, 16, 1024) | ((uint64_t)2 << 61);
              mma_tf32(tmem + tt * P.Npad, ad_lo, bd, idesc, acc);
              mma_tf32(tmem + tt * P.Npad, ad, bd_lo, idesc, 1u);
              mma_tf32(tmem + tt * P.Npad, ad, bd, idesc, 1u);
            } else {
              mma_tf32(tmem + tt * P.Npad, ad, bd, idesc, acc);
            }
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(done);
    }
  }

  // ---------------- epilogue: TMEM -> partial rows ----------------
  // thread = gradient row k (as tcgen05.ld leaves it): each 32 x 32 block goes to a swizzled
  // staging box in the now idle stage buffers and leaves by one TMA bulk store (rows >= K are
  // clipped by the map, so the producers' bias row K is untouched)
  if (warp < 4) {
    if (nchunks > 0) mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float *stg = (float *)(smem + warp * 4096);
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int sw = lane & 7;
    for (int tt = 0; tt < P.ktiles; ++tt) {
      const int k0 = tt * 128 + warp * 32;
      for (int j0 = 0; j0 < P.Npad; j0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + tt * P.Npad + j0, r);
        if (k0 >= g.K) continue;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        float4 *srow = reinterpret_cast<float4 *>(stg) + lane * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          srow[q ^ sw] = nchunks > 0 ? make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                   __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                           reinterpret_cast<uint64_t>(&pmap)),
                       "r"(j0), "r"(k0), "r"((int)blockIdx.x), "r"(smem_u32(stg))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05 weight-gradient GEMM with MN-major operands (k_wgrad_mn):
//   G[k, n] = Σ_m A(m, k) · D(m, n) as the UMMA D_mma[M = k][N = n] = Σ_{K = m} A_mma · B_mma
//   where A_mma (k × m) and B_mma (n × m) are read MN-MAJOR: the smem tile of 32 rows m ×
//   32 features holds each row's features contiguously — exactly the row-major layout of the
//   activations — so TMA loads the rows as they are (SWIZZLE_128B boxes of RS rows × 32 fp32)
//   and gathered rows arrive by 16-B cp.async into the same swizzled slots; no transpose.
//   MN-major TF32 operands need the 128B_BASE32B smem layout (descriptor layout type 1; TMA
//   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 32 features per 128-B row, the 32-B chunk c of row r
//   stored at chunk c ^ (r & 3) (a 512-B swizzle atom of 4 rows); canonical form (16-B units)
//   ((8, n), (4, k)) : ((1, LBO), (8, SBO)) — the next 32 features at LBO = one box (RS·128 B),
//   the next 4 rows at SBO = 512 B; an MMA K step (8 rows) advances 1 KB.
//   Warps 0-3 load (TMA by thread 0, gathers by all 128), warps 4-11 convert in place (lane =
//   column: SiLU for act, TF32 rounding or the 3xTF32 split hi | lo, and the column sums of D
//   = the bias gradient, one D box per warp for the whole kernel), warp 12 issues the MMAs,
//   warps 0-3 drain TMEM into the CTA's partial (TMA bulk stores; reduce.cu sums the partials).
// ---------------------------------------------------------------------------
#ifdef CHG_TC_DEBUG
__device__ int g_trace_wg = 0;
__device__ __forceinline__ int getenv_trace_wg() { return g_trace_wg; }
#endif
constexpr int MN_RS = 32;                  // rows m per stage
#define MN_RS_ 32
constexpr int MN_NLW = 4, MN_NCW = 12;     // loader / converter warps
constexpr int MN_THREADS = (MN_NLW + MN_NCW + 1) * 32;
constexpr int MN_NST = 3;

struct WmPlan {
  int Kpad, ktiles, nA, nD, Kp, rows_per_cta, split, nst;
  int bf16;                                // BF16 operands: stage = [fp32 boxes | bf16 boxes (SWIZZLE_64B)]
  uint32_t tmem_cols;
  int abox_seg[8], abox_col[8];            // A box b: segment, first column within the segment
  int tma_bytes;                           // TMA bytes per stage (direct A boxes + D boxes)
  int any_gather;
};
struct WmMaps { CUtensorMap a[4]; CUtensorMap d; };

// one 32 x 32 MN-major box, lane = column: (SiLU), TF32 rounding in place (+ the lo part), column
// sum (bias).  All loads first, then the stores (they may alias later loads for the compiler).
template <bool SPLIT, bool ACT, bool SUM>
__device__ __forceinline__ float convert_box(uint8_t *box, uint32_t lo_off, int ch, int hu, int e) {
  float x[MN_RS_];
#pragma unroll
  for (int r = 0; r < MN_RS_; ++r)
    x[r] = *reinterpret_cast<const float *>(box + r * 128 + (((ch ^ (r & 3)) << 1 | hu) << 4) + e * 4);
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < MN_RS_; ++r) {
    const uint32_t off = r * 128 + (((ch ^ (r & 3)) << 1 | hu) << 4) + e * 4;
    const float y = ACT ? silu_fast(x[r]) : x[r];
    if (SUM) acc += y;
    const uint32_t h = to_tf32(y);
    *reinterpret_cast<uint32_t *>(box + off) = h;
    if (SPLIT) *reinterpret_cast<uint32_t *>(box + lo_off + off) = to_tf32(y - __uint_as_float(h));
  }
  return acc;
}

// BF16 mode: the box's column `lane` (SiLU for act) rounded to BF16 into the MN-major SWIZZLE_64B
// copy (32 rows x 64 B; the 16-B unit c of row r at c ^ ((r >> 1) & 3)); returns its column sum
template <bool ACT, bool SUM>
__device__ __forceinline__ float convert_box_bf16(const uint8_t *box, uint8_t *bbox, int ch, int hu, int e, int lane) {
  float x[MN_RS_];
#pragma unroll
  for (int r = 0; r < MN_RS_; ++r)
    x[r] = *reinterpret_cast<const float *>(box + r * 128 + (((ch ^ (r & 3)) << 1 | hu) << 4) + e * 4);
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < MN_RS_; ++r) {
    const float y = ACT ? silu_fast(x[r]) : x[r];
    if (SUM) acc += y;
    *reinterpret_cast<__nv_bfloat16 *>(bbox + r * 64 + ((((lane >> 3) ^ ((r >> 1) & 3))) << 4) + (lane & 7) * 2) =
        __float2bfloat16_rn(y);
  }
  return acc;
}

__device__ __forceinline__ void mbar_expect_tx_only(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(MN_THREADS, 1) k_wgrad_mn(const __grid_constant__ WGrad g, const WmPlan P,
                                                            float *__restrict__ partial,
                                                            const __grid_constant__ WmMaps TM,
                                                            const __grid_constant__ CUtensorMap pmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t BOX = MN_RS * 128;                       // one box: RS rows x 32 fp32
  const int nbox = P.nA + P.nD;
  const uint32_t half_bytes = nbox * BOX;                     // hi part of a stage
  // [A hi | D hi] (| [A lo | D lo]); BF16: [A | D] as loaded, then their BF16 copies (BOX / 2 each)
  const uint32_t st_bytes = P.bf16 ? half_bytes + half_bytes / 2 : half_bytes << P.split;
  const int NST = P.nst;
  uint64_t *loaded = (uint64_t *)(smem + NST * st_bytes);
  uint64_t *full = loaded + MN_NST;
  uint64_t *empty = full + MN_NST;
  uint64_t *done = empty + MN_NST;
  uint32_t *tslot = (uint32_t *)(done + 1);

  const int r0 = blockIdx.x * P.rows_per_cta;
  const int r1 = min(g.M, r0 + P.rows_per_cta);
  const int nchunks = r1 > r0 ? (r1 - r0 + MN_RS - 1) / MN_RS : 0;
#ifdef CHG_TC_DEBUG
  // per-CTA timeline of CTA 0 (debug builds, CHG_WG_TRACE=1): load issued, converted, MMA issued
  __shared__ uint64_t tr_t0, tr_ld[16], tr_cv[16], tr_mm[16];
  auto now = []() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  if (tid == 0) tr_t0 = now();
#endif

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&loaded[i], MN_NLW * 32);
      mbar_init(&full[i], MN_NCW);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // padding feature boxes (k >= K, never loaded) are zero in every stage, hi and lo
  for (int s = 0; s < NST; ++s)
    for (int b = g.K / 32; b < P.nA; ++b) {
      if (P.bf16) {
        for (int i = tid; i < (int)(BOX / 32); i += blockDim.x)
          reinterpret_cast<uint4 *>(smem + s * st_bytes + half_bytes + b * (BOX / 2))[i] = make_uint4(0, 0, 0, 0);
        continue;
      }
      for (int h = 0; h <= P.split; ++h)
        for (int i = tid; i < (int)(BOX / 16); i += blockDim.x)
          reinterpret_cast<uint4 *>(smem + s * st_bytes + h * half_bytes + b * BOX)[i] = make_uint4(0, 0, 0, 0);
    }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < g.A.nseg && !g.A.seg[k].idx) prefetch_tmap(&TM.a[k]);
    prefetch_tmap(&TM.d);
    prefetch_tmap(&pmap);
  }
  pdl_begin();
  const uint32_t tmem = *tslot;
  const int nAk = g.K / 32;                                   // loaded A boxes

  if (warp < MN_NLW) {
    // ---------------- loaders ----------------
    const int q = tid & 7, rb = tid >> 3;                     // 16-B unit, row (rows rb, rb + 16)
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % NST, u = c / NST;
      if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
      const int m0 = r0 + c * MN_RS;
      uint8_t *st = smem + s * st_bytes;
      if (tid == 0) {
        if (P.tma_bytes) mbar_expect_tx_only(&loaded[s], P.tma_bytes);
        for (int b = 0; b < nAk; ++b) {
          const int sg = P.abox_seg[b];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k == sg && !g.A.seg[k].idx) tma_load_2d(smem_u32(st + b * BOX), &TM.a[k], P.abox_col[b], m0, &loaded[s]);
        }
        for (int b = 0; b < P.nD; ++b) tma_load_2d(smem_u32(st + (P.nA + b) * BOX), &TM.d, 32 * b, m0, &loaded[s]);
      }
      if (P.any_gather) {
        for (int b = 0; b < nAk; ++b) {
          const ASeg &S = g.A.seg[P.abox_seg[b]];
          if (!S.idx) continue;
          const uint32_t dst0 = smem_u32(st + b * BOX);
#pragma unroll
          for (int i = 0; i < MN_RS / 16; ++i) {
            const int row = rb + 16 * i, m = m0 + row;
            const int r = (m < r1) ? __ldg(S.idx + m) : -1;
            const uint32_t dst = dst0 + row * 128 + ((((q >> 1) ^ (row & 3)) << 1 | (q & 1)) << 4);
            if (r >= 0) cp_async16(dst, S.base + (size_t)r * S.ld + P.abox_col[b] + 4 * q, 16);
            else cp_async16(dst, S.base, 0);
          }
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&loaded[s])) : "memory");
#ifdef CHG_TC_DEBUG
      if (tid == 0 && c < 16) tr_ld[c] = now();
#endif
    }
  } else if (warp < MN_NLW + MN_NCW) {
    // ---------------- converters: lane = column of a box, rows in order ----------------
    const int cw = warp - MN_NLW;
    const int sw_lane = lane >> 2, e = lane & 3;              // 16-B unit and element of column `lane`
    const int ch = sw_lane >> 1, hu = sw_lane & 1;            // its 32-B chunk and half
    float bsum[2] = {0.f, 0.f};                               // column sums of my D boxes (bias)
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % NST, u = c / NST;
      mbar_wait(&loaded[s], u & 1);
      uint8_t *st = smem + s * st_bytes;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int b = cw + MN_NCW * t;
#ifdef CHG_TC_DEBUG
        if (g_trace_wg & 2) break;                           // timing study: no conversion
#endif
        if (b >= nbox || (b < P.nA && b >= nAk)) continue;    // no box / padding features
        const bool isA = b < P.nA;
        const bool act = isA && g.A.act == 1;
        uint8_t *box = st + b * BOX;
        if (P.bf16) {
          uint8_t *bbox = st + half_bytes + b * (BOX / 2);
          if (act) convert_box_bf16<true, false>(box, bbox, ch, hu, e, lane);
          else if (isA) convert_box_bf16<false, false>(box, bbox, ch, hu, e, lane);
          else bsum[t] += convert_box_bf16<false, true>(box, bbox, ch, hu, e, lane);
        } else if (P.split) {
          if (act) convert_box<true, true, false>(box, half_bytes, ch, hu, e);
          else if (isA) convert_box<true, false, false>(box, half_bytes, ch, hu, e);
          else bsum[t] += convert_box<true, false, true>(box, half_bytes, ch, hu, e);
        } else {
          if (act) convert_box<false, true, false>(box, half_bytes, ch, hu, e);
          else if (isA) convert_box<false, false, false>(box, half_bytes, ch, hu, e);
          else bsum[t] += convert_box<false, false, true>(box, half_bytes, ch, hu, e);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
#ifdef CHG_TC_DEBUG
      if (cw == 0 && lane == 0 && c < 16) tr_cv[c] = now();
#endif
    }
    if (g.bias) {                                            // bias row K of this CTA's partial
      float *Pout = partial + (size_t)blockIdx.x * P.Kp * g.N + (size_t)g.K * g.N;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int b = cw + MN_NCW * t;
        if (b >= P.nA && b < nbox) Pout[32 * (b - P.nA) + lane] = bsum[t];
      }
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(g.N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc_bf = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                              ((uint32_t)(g.N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    constexpr uint32_t BOXB = BOX / 2;                          // one BF16 box: RS rows x 64 B
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % NST, u = c / NST;
      mbar_wait(&full[s], u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = smem_u32(smem + s * st_bytes);
      if (P.bf16) {
        // MN-major SWIZZLE_64B: the next 32 features at LBO = one BF16 box, the next 8 rows at
        // SBO = 512 B; an MMA K step (16 rows) advances 1 KB
        const uint32_t bb = base + half_bytes;
        for (int tt = 0; tt < P.ktiles; ++tt) {
#pragma unroll
          for (int j = 0; j < MN_RS / 16; ++j) {
            const uint64_t ad = make_desc(bb + tt * 4 * BOXB + j * 1024, BOXB, 512) | ((uint64_t)4 << 61);
            const uint64_t bd = make_desc(bb + P.nA * BOXB + j * 1024, BOXB, 512) | ((uint64_t)4 << 61);
            mma_bf16(tmem + tt * g.N, ad, bd, idesc_bf, (c > 0 || j > 0) ? 1u : 0u);
          }
        }
        mma_commit(&empty[s]);
        continue;
      }
      for (int tt = 0; tt < P.ktiles; ++tt) {
#pragma unroll
        for (int j = 0; j < MN_RS / 8; ++j) {
          const uint32_t a0 = base + tt * 4 * BOX + j * 1024, d0 = base + P.nA * BOX + j * 1024;
          const uint64_t ad = make_desc(a0, BOX, 512) | ((uint64_t)1 << 61);     // SWIZZLE_128B_BASE32B
          const uint64_t bd = make_desc(d0, BOX, 512) | ((uint64_t)1 << 61);
          const uint32_t acc = (c > 0 || j > 0) ? 1u : 0u;
          if (P.split) {
            const uint64_t ad_lo = make_desc(a0 + half_bytes, BOX, 512) | ((uint64_t)1 << 61);
            const uint64_t bd_lo = make_desc(d0 + half_bytes, BOX, 512) | ((uint64_t)1 << 61);
            mma_tf32(tmem + tt * g.N, ad_lo, bd, idesc, acc);
            mma_tf32(tmem + tt * g.N, ad, bd_lo, idesc, 1u);
            mma_tf32(tmem + tt * g.N, ad, bd, idesc, 1u);
          } else {
            mma_tf32(tmem + tt * g.N, ad, bd, idesc, acc);
          }
        }
      }
      mma_commit(&empty[s]);
#ifdef CHG_TC_DEBUG
      if (c < 16) tr_mm[c] = now();
#endif
    }
    mma_commit(done);
  }

  // ---------------- epilogue: TMEM -> partial rows (thread = gradient row k) ----------------
  if (warp < 4) {
    if (nchunks > 0) mbar_wait(done, 0);
#ifdef CHG_TC_DEBUG
    if (tid == 0 && blockIdx.x == 0 && getenv_trace_wg()) {
      const uint64_t t = now();
      printf("WGTRACE K %d N %d chunks %d nst %d split %d | mma_done %.2f us |", g.K, g.N, nchunks, NST, P.split,
             (t - tr_t0) * 1e-3);
      for (int c = 0; c < min(16, nchunks); ++c)
        printf(" [%d ld %.2f cv %.2f mm %.2f]", c, (tr_ld[c] - tr_t0) * 1e-3, (tr_cv[c] - tr_t0) * 1e-3,
               (tr_mm[c] - tr_t0) * 1e-3);
      printf("\n");
    }
#endif
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float *stg = (float *)(smem + warp * 4096);
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int sw = lane & 7;
    for (int tt = 0; tt < P.ktiles; ++tt) {
      const int k0 = tt * 128 + warp * 32;
      for (int j0 = 0; j0 < g.N; j0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + tt * g.N + j0, r);
        if (k0 >= g.K) continue;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        float4 *srow = reinterpret_cast<float4 *>(stg) + lane * 8;
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          srow[q4 ^ sw] = nchunks > 0 ? make_float4(__uint_as_float(r[4 * q4]), __uint_as_float(r[4 * q4 + 1]),
                                                    __uint_as_float(r[4 * q4 + 2]), __uint_as_float(r[4 * q4 + 3]))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                           reinterpret_cast<uint64_t>(&pmap)),
                       "r"(j0), "r"(k0), "r"((int)blockIdx.x), "r"(smem_u32(stg))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols) : "memory");
}

struct TcCache {
  std::map<std::string, int> index;
  std::vector<PackJob> jobs;
  std::vector<uint64_t> gen;     // forward generation the image was packed for
  uint64_t cur_gen = 0;
  PackJob *d_jobs = nullptr;
  size_t d_cap = 0;
  bool dirty = false;
};

}  // namespace

// start of a forward: new generation; re-pack every cached image of the model in one launch
void tc_repack_all(chg_ctx *ctx, chg_model *m) {
  TcCache *c = (TcCache *)m->tc_cache;
  if (!c) {
    c = new TcCache();
    m->tc_cache = c;
  }
  ++c->cur_gen;
  if (c->jobs.empty()) return;
  if (c->dirty || c->d_cap < c->jobs.size()) {
    if (c->d_cap < c->jobs.size()) {
      if (c->d_jobs) CUDA_OK(cudaFree(c->d_jobs));
      c->d_cap = c->jobs.size() + 8;
      CUDA_OK(cudaMalloc(&c->d_jobs, c->d_cap * sizeof(PackJob)));
    }
    CUDA_OK(cudaMemcpyAsync(c->d_jobs, c->jobs.data(), c->jobs.size() * sizeof(PackJob), cudaMemcpyHostToDevice,
                            ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));   // pageable source: keep it simple, happens once per new site
    c->dirty = false;
  }
  double bytes = 0;
  for (auto &J : c->jobs) bytes += (double)J.nkc * J.P.bnt * KC * 8.0 * (1 + J.P.split);
  ProfScope ps(ctx, "tc_pack", 0.0, bytes);
  launch_k(ctx, k_pack_all, dim3(148, (unsigned)c->jobs.size()), 256, 0, ctx->stream, c->d_jobs);
  check_launch(ctx);
  for (auto &g : c->gen) g = c->cur_gen;
}

void tc_cache_free(chg_model *m) {
  TcCache *c = (TcCache *)m->tc_cache;
  if (!c) return;
  for (auto &J : c->jobs) cudaFree(J.img);
  if (c->d_jobs) cudaFree(c->d_jobs);
  delete c;
  m->tc_cache = nullptr;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}
// 2-D fp32 map over a row-major [rows][width] table (row stride ld floats): box = 32 columns x
// 128 rows, SWIZZLE_128B (the K-major UMMA layout), rows past the end read as zeros.
static int encode_a_map(CUtensorMap *m, const float *base, int width, int rows, int ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || rows <= 0 || ((uintptr_t)base & 15) || (ld * 4) % 16) return 0;
  cuuint64_t dim[2] = {(cuuint64_t)width, (cuuint64_t)rows};
  cuuint64_t stride[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {KC, TCM}, es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dim, stride, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

// 2-D fp32 map of an epilogue operand [rows][ncols] (row stride ld): 32 x 32 boxes, no swizzle
static int encode_op_map(CUtensorMap *m, const float *base, int ncols, int rows, int ld, bool swz = false) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || rows <= 0 || ncols % 32 || ((uintptr_t)base & 15) || (ld * 4) % 16) return 0;
  cuuint64_t dim[2] = {(cuuint64_t)ncols, (cuuint64_t)rows};
  cuuint64_t stride[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dim, stride, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

// Returns false if the GEMM does not fit this path (caller uses the SIMT kernel).
// ksplit > 1: g is the partial-output GEMM of a split-K (raw accumulators stored at rows
// y·kmpad + m of g.ch[0].out, k_splitk_sum finishes it; see rowgemm_tc below)
static bool rowgemm_tc_impl(chg_ctx *ctx, const RowGemm &g, int ksplit, int kper, int kmpad) {
  if (g.M <= 0 || g.K % KC != 0 || g.nchunk < 1) return false;
  const int split = ctx->tc_split ? 1 : 0;
  // small problems (at most one 128-row tile per SM: the per-atom / per-bond products) need no
  // A pipeline: one stage, which leaves room for a 256-column [hi | lo] weight image
  const bool one_wave = ceil_div(g.M, TCM) <= device_sm_count();
  if (split && g.nchunk > 1) {
    // 3xTF32 stages hold [hi | lo] operands: at most 128 output columns per launch, so wider
    // GEMMs (bc_f1, bc_dX, ac_dX) run as launches over groups of their output chunks
    int cols = 0;
    for (int c = 0; c < g.nchunk; ++c) cols += (g.ch[c].ncols + 31) / 32 * 32;
    if (cols > 128 && !(one_wave && g.K <= 64)) {
      int c0 = 0;
      while (c0 < g.nchunk) {
        RowGemm h = g;
        int w = 0, n = 0;
        while (c0 + n < g.nchunk && w + (g.ch[c0 + n].ncols + 31) / 32 * 32 <= 128) {
          h.ch[n] = g.ch[c0 + n];
          w += (g.ch[c0 + n].ncols + 31) / 32 * 32;
          ++n;
        }
        h.nchunk = n;
        if (!rowgemm_tc_impl(ctx, h, 1, 0, 0))
          CHG_THROW(CHG_ERR_STATE, "rowgemm_tc %s: 3xTF32 column group does not fit", g.tag);
        c0 += n;
      }
      return true;
    }
  }
  TcPlan P{};
  P.split = split;
  P.bf16 = ctx->tc_bf16 ? 1 : 0;
  P.ksplit = ksplit > 1 ? ksplit : 1;
  P.kper = kper;
  P.kmpad = kmpad;
  int lo = 1 << 30, hi = 0, off = 0;
  for (int c = 0; c < g.nchunk; ++c) {
    const Chunk &C = g.ch[c];
    if (C.a_k0 % KC) return false;
    for (int b = 0; b < C.nwb; ++b)
      if (!C.Wk[b]) return false;
    lo = std::min(lo, C.a_k0);
    hi = std::max(hi, C.a_k0 + g.K);
    P.cpad[c] = std::max(16, (C.ncols + 15) / 16 * 16);
    P.coff[c] = off;
    off += (C.ncols + 31) / 32 * 32;
  }
  int tot = 0;
  for (int s = 0; s < g.A.nseg; ++s) {
    const ASeg &S = g.A.seg[s];
    if (S.width % KC || S.ld % 4 || ((uintptr_t)S.base & 15)) return false;
    tot += S.width;
  }
  if (hi > tot) return false;
  for (int c = 0; c < g.nchunk; ++c) {                // gathered additions: 16-B rows, no TMA-operand chunk,
    if (g.ch[c].ngadd != g.ch[0].ngadd || g.ch[c].ngadd > 2) return false;  // <= 2, the same indices in every chunk
    for (int k = 0; k < g.ch[c].ngadd; ++k)
      if (((uintptr_t)g.ch[c].gadd[k] & 15) || (g.ch[c].ldga[k] & 3) || g.ch[c].mul || g.ch[c].resid ||
          g.ch[c].gidx[k] != g.ch[0].gidx[k])
        return false;
  }
  P.lo = lo;
  P.width = hi - lo;
  P.ntot = off;
  // adjacent chunks reading the same A window (same a_k0, contiguous TMEM columns) share one
  // MMA of N = their total width: fewer, wider tensor-core instructions
  P.ngrp = 0;
  for (int c = 0; c < g.nchunk; ++c) {
    const bool join = P.ngrp > 0 && g.ch[c].a_k0 == g.ch[P.gfirst[P.ngrp - 1]].a_k0 &&
                      P.coff[c] == P.coff[P.gfirst[P.ngrp - 1]] + P.gn[P.ngrp - 1] &&
                      P.coff[c] - P.coff[P.gfirst[P.ngrp - 1]] + P.cpad[c] <= 256;
    if (join) {
      P.gn[P.ngrp - 1] = P.coff[c] - P.coff[P.gfirst[P.ngrp - 1]] + P.cpad[c];
    } else {
      P.gfirst[P.ngrp] = c;
      P.gn[P.ngrp] = P.cpad[c];
      ++P.ngrp;
    }
  }
  if (P.ntot > 256) return false;
  P.tmem_cols = P.ntot <= 32 ? 32 : P.ntot <= 64 ? 64 : P.ntot <= 128 ? 128 : 256;
  {  // compact weight image: per K chunk only the chunks whose window covers it
    const int nkc0 = P.width / KC;
    if (nkc0 > 16) return false;
    P.bnt = 0;
    for (int kc = 0; kc < nkc0; ++kc) {
      int w = 0;
      for (int c = 0; c < 4; ++c) P.bcoff[kc][c] = -1;
      for (int c = 0; c < g.nchunk; ++c) {
        const int kk = P.lo + kc * KC - g.ch[c].a_k0;
        if (kk < 0 || kk >= g.K) continue;
        P.bcoff[kc][c] = (int16_t)w;
        w += (g.ch[c].ncols + 31) / 32 * 32;
      }
      P.bnt = std::max(P.bnt, w);
    }
  }
  const int nkc = P.width / KC;
  // column split (one-wave, dense: one MMA group, every chunk active in every K chunk): parts of
  // whole chunks on blockIdx.y, as many as fit one wave (<= 4)
  P.csplit = 1;
  static const bool no_csplit = getenv("CHG_TC_NO_CSPLIT") != nullptr;   // A/B knob
  {
    const int ntl = ceil_div(g.M, TCM), sms = device_sm_count();
    bool dense = P.ngrp == 1 && g.nchunk >= 2 && !no_csplit;
    for (int kc = 0; kc < nkc && dense; ++kc)
      for (int c = 0; c < g.nchunk; ++c) dense &= P.bcoff[kc][c] == P.bcoff[0][c] && P.bcoff[kc][c] >= 0;
    int G = 1;
    while (dense && G * 2 <= g.nchunk && g.nchunk % (G * 2) == 0 && ntl * G * 2 <= sms) G *= 2;
    if (G > 1) {
      P.csplit = G;
      const int per = g.nchunk / G;
      for (int y = 0; y < G; ++y) {
        P.cs_c0[y] = y * per;
        P.cs_c1[y] = (y + 1) * per;
        P.cs_n0[y] = P.bcoff[0][y * per];
        int w = 0;
        for (int c = y * per; c < (y + 1) * per; ++c) w += (g.ch[c].ncols + 31) / 32 * 32;
        P.cs_nt[y] = w;
      }
    }
  }
  int bnt_s = P.bnt;                                  // weight-image columns per CTA in shared memory
  if (P.csplit > 1) {
    bnt_s = 0;
    for (int y = 0; y < P.csplit; ++y) bnt_s = std::max(bnt_s, P.cs_nt[y]);
  }
  const size_t bchunk = P.bf16 ? (size_t)KC * bnt_s * 2 : ((size_t)KC * bnt_s * 4) << split;
  const size_t achunk = P.bf16 ? (size_t)KC * TCM * 6 : ((size_t)KC * TCM * 4) << split;
  const int nsa_min = split ? (one_wave ? 1 : 2) : 4;
  // TMA-store epilogue (lane = row) when every chunk's output is a plain [M][32k] table
  static const bool no_tstore = getenv("CHG_TC_NO_TSTORE") != nullptr;   // A/B knob
  TcMaps TM;
  memset(&TM, 0, sizeof(TM));
  TM.tstore = !no_tstore && g.act == 0 && encode_fn() != nullptr;
  for (int c = 0; c < g.nchunk && TM.tstore; ++c) {
    const Chunk &C = g.ch[c];
    if (C.pre || C.ncols % 32 || !C.out) TM.tstore = 0;
    else if (!encode_op_map(&TM.o[c], C.out, C.ncols, P.ksplit > 1 ? P.ksplit * P.kmpad : g.M, C.ldo, true)) TM.tstore = 0;
    else if (C.sout && !encode_op_map(&TM.o2[c], C.sout, C.ncols, g.M, C.ldso, true)) TM.tstore = 0;
  }
  for (int c = 0; c < g.nchunk && TM.tstore; ++c)
    TM.radd[c] = g.ch[c].resid == g.ch[c].out && g.ch[c].ldr == g.ch[c].ldo && !g.ch[c].mul;
  bool has_sout = false, has_round = false;
  for (int c = 0; c < g.nchunk; ++c) { has_sout |= g.ch[c].sout != nullptr; has_round |= g.ch[c].round_out != 0; }
  if ((has_sout || has_round) && !TM.tstore) return false;          // only the TMA-store epilogue writes sout / rounded out
  const size_t epi_b = TM.tstore ? 0 : (size_t)NEPI * 32 * 33 * 4;
  auto fixed_of = [&](int nsa) {
    return 1024 + nsa * achunk + 8 * (3 * nsa + 2 * NSB + 4) + 16 + epi_b;
  };
  // keep the whole weight image resident when it fits (no per-stage B round trips), then as
  // many A stages as the remaining shared memory holds (the A ring is latency-bound)
  static const bool no_bres = getenv("CHG_TC_NO_BRES") != nullptr;   // A/B knobs (timing studies)
  static const int nsa_cap = getenv("CHG_TC_NSA") ? atoi(getenv("CHG_TC_NSA")) : NSA_MAX;
  // epilogue operands (mul / resid of a chunk) by TMA when the GEMM has them: 2 boxes in flight
  // per epilogue warp if shared memory allows (else 1); with the TMA-store epilogue one
  // operand box and one staging box per warp take precedence over a resident weight image
  static const bool no_etma = getenv("CHG_TC_NO_ETMA") != nullptr;   // A/B knob
  int has_op = 0;
  for (int c = 0; c < g.nchunk; ++c)
    has_op |= ((g.ch[c].mul != nullptr) != (g.ch[c].resid != nullptr)) && !g.ch[c].pre && !TM.radd[c];
  int nbuf = (has_op && !no_etma) ? 2 : 0;
  static const int nst_cap = getenv("CHG_TC_NST") ? atoi(getenv("CHG_TC_NST")) : 1;
  TM.nst = TM.tstore ? ((has_sout || nst_cap >= 2) ? 2 : 1) : 0;
  auto opbytes = [&](int nb) { return (size_t)1024 + (size_t)NEPI * (nb + TM.nst) * 4096 + 2 * NEPI * 8; };
  const int nb_min = TM.tstore ? std::min(nbuf, 1) : 0;
  P.bres = !no_bres && fixed_of(nsa_min + 1) + nkc * bchunk + (TM.tstore ? opbytes(nb_min) : 0) <= 224 * 1024;
  P.nsb = split ? 2 : NSB;
  P.bst = P.bres ? nkc : P.nsb;
  if (nbuf == 2 && fixed_of(nsa_min) + P.bst * bchunk + opbytes(2) > 224 * 1024) nbuf = 1;
  if (nbuf == 1 && fixed_of(nsa_min) + P.bst * bchunk + opbytes(1) > 224 * 1024) nbuf = 0;
  if (TM.nst == 2 && fixed_of(nsa_min) + P.bst * bchunk + opbytes(nbuf) > 224 * 1024) TM.nst = 1;
  P.nsa = nsa_min;
  while (P.nsa < std::min(nsa_cap, NSA_MAX) && fixed_of(P.nsa + 1) + P.bst * bchunk + opbytes(nbuf) <= 224 * 1024)
    ++P.nsa;
  size_t smem = fixed_of(P.nsa) + P.bst * bchunk + opbytes(nbuf);
  if (smem > 224 * 1024) {
    fprintf(stderr, "rowgemm_tc %s: shared memory plan %zu B exceeds 224 KB\n", g.tag ? g.tag : "?", smem);
    return false;
  }
  smem_optin((const void *)k_rowgemm_tc, 224 * 1024);
  double cols = 0;
  for (int c = 0; c < g.nchunk; ++c) cols += g.ch[c].ncols;
  // weight image: cached per (model, call site); all of a model's images are re-packed in
  // one launch at the start of each forward (tc_repack_all) — only a new site packs here
  uint32_t *img = nullptr;
  TcCache *cache = ctx->cur_model ? (TcCache *)ctx->cur_model->tc_cache : nullptr;
  std::string key;
  if (cache) {
    char kb[64];
    key = g.tag ? g.tag : "";
    for (int c = 0; c < g.nchunk; ++c)
      for (int b = 0; b < g.ch[c].nwb; ++b) {
        snprintf(kb, sizeof(kb), "|%p", (const void *)g.ch[c].Wk[b]);
        key += kb;
      }
    auto it = cache->index.find(key);
    if (it != cache->index.end() && cache->gen[it->second] == cache->cur_gen) img = cache->jobs[it->second].img;
  }
  if (!img) {
    const size_t bytes = ((size_t)nkc * P.bnt * KC * 4) << split;    // hi image (+ lo image)
    if (cache) {
      auto it = cache->index.find(key);
      int id;
      if (it == cache->index.end()) {
        id = (int)cache->jobs.size();
        PackJob J{};
        J.g = g; J.P = P; J.nkc = nkc;
        CUDA_OK(cudaMalloc(&J.img, bytes));
        cache->jobs.push_back(J);
        cache->gen.push_back(0);
        cache->index[key] = id;
        cache->dirty = true;
      } else {
        id = it->second;
      }
      img = cache->jobs[id].img;
      cache->gen[id] = cache->cur_gen;
    } else {
      img = (uint32_t *)ctx->get("tc_bimg", bytes);
    }
    ProfScope ps(ctx, "tc_pack", 0.0, (double)nkc * P.bnt * KC * 8.0);
    dim3 grid(ceil_div((int64_t)P.bnt * KC, 256), nkc);
    launch_k(ctx, k_pack_b, grid, 256, 0, ctx->stream, g, P, img);
    check_launch(ctx);
  }
  const int ntiles = ceil_div(g.M, TCM);
  const int sms = device_sm_count();
  const int grid = std::min(ntiles, sms);
  double outb = 0;
  for (int c = 0; c < g.nchunk; ++c) {
    const Chunk &C = g.ch[c];
    outb += C.ncols * (1.0 + (C.pre != nullptr) + (C.mul != nullptr) + (C.resid != nullptr) + (C.sout != nullptr));
  }
  ProfScope ps(ctx, g.tag ? g.tag : "rowgemm_tc", 2.0 * g.M * (double)g.K * cols,
               gemm_a_bytes(g.A, g.M, P.lo, P.lo + P.width) + (double)g.M * 4.0 * outb + 4.0 * g.K * cols);
#ifdef CHG_TC_DEBUG
  static int skip = getenv("CHG_TC_SKIP") ? atoi(getenv("CHG_TC_SKIP")) : 0;   // debug knob (timing studies)
#else
  const int skip = 0;
#endif
  static const bool no_tma = getenv("CHG_TC_NO_TMA") != nullptr;            // A/B knob (timing studies)
  for (int s = 0; s < g.A.nseg && !no_tma; ++s) {
    const ASeg &S = g.A.seg[s];
    if (S.idx) continue;                              // gathered rows stay on cp.async (tile::gather4 measured slower)
    TM.use[s] = encode_a_map(&TM.m[s], S.base, S.width, g.M, S.ld);
  }
  static const bool no_noconv = getenv("CHG_TC_NO_NOCONV") != nullptr;    // A/B knob
  P.noconv = g.A.rounded && g.A.act == 0 && !no_noconv && !split && !P.bf16;
  for (int s = 0; s < g.A.nseg; ++s) P.noconv &= TM.use[s];
  static const bool no_lconv = getenv("CHG_TC_NO_LCONV") != nullptr;      // A/B knob
  P.lconv = !P.noconv && !no_lconv && g.A.nseg > 0;
  for (int s = 0; s < g.A.nseg; ++s) P.lconv &= TM.use[s];
  TM.nbuf = nbuf;
  for (int c = 0; c < g.nchunk && nbuf > 0; ++c) {
    const Chunk &C = g.ch[c];
    if ((C.mul != nullptr) == (C.resid != nullptr) || C.pre || TM.radd[c]) continue;
    const float *op = C.mul ? C.mul : C.resid;
    TM.use_e[c] = encode_op_map(&TM.e[c], op, C.ncols, g.M, C.mul ? C.ldm : C.ldr, TM.tstore != 0);
  }
  static const bool verbose = getenv("CHG_TC_VERBOSE") != nullptr;
  if (verbose)
    fprintf(stderr, "rowgemm_tc %s: M %d K %d nseg %d tma %d%d%d%d nsa %d bres %d tstore %d nst %d nbuf %d noconv %d lconv %d csplit %d smem %zu\n",
            g.tag ? g.tag : "?", g.M, g.K, g.A.nseg, TM.use[0], TM.use[1], TM.use[2], TM.use[3], P.nsa, P.bres,
            TM.tstore, TM.nst, nbuf, P.noconv, P.lconv, P.csplit, smem);
  if (P.ksplit > 1 && (!TM.tstore || P.csplit > 1)) CHG_THROW(CHG_ERR_STATE, "rowgemm_tc %s: split-K plan", g.tag);
  launch_k(ctx, k_rowgemm_tc, dim3(grid, P.ksplit > 1 ? P.ksplit : P.csplit), WS_THREADS, smem, ctx->stream, g, P, img,
           ntiles, skip, TM);
  check_launch(ctx);
  return true;
}


namespace {
// out[m][n] = resid[m][n] + bias[n] + Σ_y part[y·mpad + m][n]  (fixed order: deterministic)
__global__ void k_splitk_sum(int M, int ncols, int G, const float *__restrict__ part, int mpad, int ldp,
                             const float *__restrict__ bias, const float *__restrict__ resid, int ldr,
                             float *__restrict__ out, int ldo) {
  pdl_begin();
  const int nq = ncols >> 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)M * nq; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / nq), q = (int)(i % nq);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int y = 0; y < G; ++y) {
      const float4 v = *reinterpret_cast<const float4 *>(part + ((size_t)y * mpad + m) * ldp + 4 * q);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (bias) {
      const float4 b = *reinterpret_cast<const float4 *>(bias + 4 * q);
      acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
    }
    if (resid) {
      const float4 r = *reinterpret_cast<const float4 *>(resid + (size_t)m * ldr + 4 * q);
      acc.x += r.x; acc.y += r.y; acc.z += r.z; acc.w += r.w;
    }
    *reinterpret_cast<float4 *>(out + (size_t)m * ldo + 4 * q) = acc;
  }
}
}  // namespace

// Split-K for one-wave single-chunk GEMMs with a long K and a plain epilogue (bias / residual
// only: the per-atom / per-bond adjoint GEMMs, K = 256-512 on a few tiles): G CTAs per tile
// each sum K / G, raw partial tiles are stored by TMA and added in a fixed order by
// k_splitk_sum — more SMs busy, each with a fraction of the MMA / load / conversion chain.
bool rowgemm_tc(chg_ctx *ctx, const RowGemm &g) {
  static const bool no_ksplit = getenv("CHG_TC_NO_KSPLIT") != nullptr;   // A/B knob
  const Chunk &C = g.ch[0];
  const int ntiles = g.M > 0 ? ceil_div(g.M, TCM) : 0, sms = device_sm_count();
  const int nkc = g.K / KC;
  const bool plain = g.nchunk == 1 && g.act == 0 && !C.mul && !C.pre && !C.sout && !C.round_out && C.ngadd == 0 &&
                     C.out && C.ncols % 32 == 0 && C.ldo % 4 == 0 && (!C.resid || C.ldr % 4 == 0) &&
                     C.a_k0 == 0 && g.K % KC == 0;
  int G = 1;
  while (plain && !no_ksplit && ntiles > 0 && nkc / (G * 2) >= 2 && ntiles * G * 2 <= sms) G *= 2;
  if (G == 1) return rowgemm_tc_impl(ctx, g, 1, 0, 0);
  const int kper = (nkc + G - 1) / G;
  G = (nkc + kper - 1) / kper;
  const int mpad = ntiles * TCM, ldp = C.ncols;
  float *part = ctx->getf(ctx->ws_name("tc_ksplit"), (size_t)G * mpad * ldp);   // stream-private (forked branches)
  RowGemm h = g;
  Chunk &H = h.ch[0];
  H.out = part; H.ldo = ldp; H.bias = nullptr; H.resid = nullptr; H.ldr = 0;
  if (!rowgemm_tc_impl(ctx, h, G, kper, mpad)) return false;
  const int64_t n4 = (int64_t)g.M * (C.ncols / 4);
  ProfScope ps(ctx, g.tag ? g.tag : "rowgemm_tc", 0.0, 4.0 * g.M * C.ncols * (G + 1 + (C.resid ? 1 : 0)));
  launch_k(ctx, k_splitk_sum, (unsigned)std::min<int64_t>(ceil_div(n4, 256), 4 * sms), 256, 0, ctx->stream, g.M,
           C.ncols, G, (const float *)part, mpad, ldp, C.bias, C.resid, C.ldr, C.out, C.ldo);
  check_launch(ctx);
  return true;
}

// MN-major weight gradient (k_wgrad_mn): false when an operand cannot be TMA / cp.async staged
static bool wgrad_mn(chg_ctx *ctx, const WGrad &g, float **partial_out, int *Kp_out, int *splits_out) {
  static const bool off = getenv("CHG_WG_TRANSPOSE") != nullptr;   // A/B knob: the transposing producers
  EncodeTiledFn fn = encode_fn();
  if (off || !fn || g.didx || (g.ldd % 4) || ((uintptr_t)g.D & 15) || g.K > 256 || g.N > 256 || g.K % 32 || g.N % 32)
    return false;
  WmPlan P{};
  P.Kpad = (g.K + 127) / 128 * 128;
  P.ktiles = P.Kpad / 128;
  P.nA = P.Kpad / 32;
  P.nD = g.N / 32;
  P.Kp = g.K + (g.bias ? 1 : 0);
  P.split = ctx->tc_split ? 1 : 0;
  P.bf16 = ctx->tc_bf16 ? 1 : 0;
  const int cols = P.ktiles * g.N;
  if (cols > 512) return false;
  P.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  WmMaps TM;
  memset(&TM, 0, sizeof(TM));
  int direct_boxes = 0;
  {
    int sg = 0, start = 0;
    for (int b = 0; b < g.K / 32; ++b) {
      while (sg < g.A.nseg && 32 * b >= start + g.A.seg[sg].width) start += g.A.seg[sg++].width;
      if (sg >= g.A.nseg) return false;
      P.abox_seg[b] = sg;
      P.abox_col[b] = 32 * b - start;
      if (g.A.seg[sg].idx) P.any_gather = 1;
      else ++direct_boxes;
    }
    for (int s = 0; s < g.A.nseg; ++s) {
      const ASeg &S = g.A.seg[s];
      if (S.width % 32 || S.ld % 4 || ((uintptr_t)S.base & 15)) return false;
      if (S.idx) continue;
      cuuint64_t dim[2] = {(cuuint64_t)S.width, (cuuint64_t)g.M};
      cuuint64_t stride[1] = {(cuuint64_t)S.ld * 4};
      cuuint32_t box[2] = {32, MN_RS}, es[2] = {1, 1};
      if (fn(&TM.a[s], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)S.base, dim, stride, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    }
    cuuint64_t dim[2] = {(cuuint64_t)g.N, (cuuint64_t)g.M};
    cuuint64_t stride[1] = {(cuuint64_t)g.ldd * 4};
    cuuint32_t box[2] = {32, MN_RS}, es[2] = {1, 1};
    if (fn(&TM.d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)g.D, dim, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  P.tma_bytes = (direct_boxes + P.nD) * MN_RS * 128;
  const size_t st_half = (size_t)(P.nA + P.nD) * MN_RS * 128;
  const size_t st_bytes = P.bf16 ? st_half + st_half / 2 : st_half << P.split;
  const size_t fixed = 1024 + 8 * (3 * MN_NST + 1) + 16;
  P.nst = (int)std::min<size_t>(MN_NST, (224 * 1024 - fixed) / st_bytes);
  if (P.nst < 2) return false;
  const size_t smem = fixed + P.nst * st_bytes;
  const int sms = device_sm_count();
  const int chunks = (g.M + MN_RS - 1) / MN_RS;
  const int grid = std::max(1, std::min(sms, chunks));
  P.rows_per_cta = (chunks + grid - 1) / grid * MN_RS;
  const int splits = (g.M + P.rows_per_cta - 1) / P.rows_per_cta;
  float *partial = red_partial(ctx, (size_t)splits * P.Kp * g.N);
  if ((uintptr_t)partial & 15) return false;
  CUtensorMap pmap;
  {
    cuuint64_t dim[3] = {(cuuint64_t)g.N, (cuuint64_t)g.K, (cuuint64_t)splits};
    cuuint64_t stride[2] = {(cuuint64_t)g.N * 4, (cuuint64_t)P.Kp * g.N * 4};
    cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
    if (fn(&pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, partial, dim, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  smem_optin((const void *)k_wgrad_mn, 224 * 1024);
#ifdef CHG_TC_DEBUG
  static const int trace = getenv("CHG_WG_TRACE") ? atoi(getenv("CHG_WG_TRACE")) : 0;
  static bool set = false;
  if (!set) { cudaMemcpyToSymbol(g_trace_wg, &trace, sizeof(int)); set = true; }
#endif
  ProfScope ps(ctx, g.tag ? g.tag : "wgrad_tc", 2.0 * g.M * (double)P.Kp * g.N,
               gemm_a_bytes(g.A, g.M, 0, g.K) + (double)g.M * 4.0 * g.N + 4.0 * P.Kp * g.N);
  launch_k(ctx, k_wgrad_mn, splits, MN_THREADS, smem, ctx->stream, g, P, partial, TM, pmap);
  check_launch(ctx);
  *partial_out = partial;
  *Kp_out = P.Kp;
  *splits_out = splits;
  return true;
}

// Weight gradient on tcgen05 (TF32).  Returns false when the shape does not fit
// (caller uses the SIMT kernel).  Writes partials [splits][Kp][N] for the batched reduction (reduce.cu).
bool wgrad_tc(chg_ctx *ctx, const WGrad &g, float **partial_out, int *Kp_out, int *splits_out, bool *bias_done) {
  if (g.M <= 0 || g.K <= 0 || g.K % 32 || g.N % 32 || g.N > 256 || g.K > 256 || (g.ldd % 4)) return false;
  if (wgrad_mn(ctx, g, partial_out, Kp_out, splits_out)) {
    *bias_done = true;
    return true;
  }
  if ((uintptr_t)g.D & 15) return false;
  for (int s = 0; s < g.A.nseg; ++s) {
    const ASeg &S = g.A.seg[s];
    if (S.width % 32 || S.ld % 4 || ((uintptr_t)S.base & 15)) return false;
  }
  WgPlan P{};
  P.Kpad = (g.K + 127) / 128 * 128;
  P.ktiles = P.Kpad / 128;
  P.Npad = g.N;
  P.ones_col = -1;                                    // bias is summed by the producers
  P.Kp = g.K + (g.bias ? 1 : 0);
  const int cols = P.ktiles * P.Npad;
  if (cols > 512) return false;
  P.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  const int sms = device_sm_count();
  const int chunks = (g.M + 31) / 32;
  const int grid = std::max(1, std::min(sms, chunks));
  P.rows_per_cta = (chunks + grid - 1) / grid * 32;
  const int splits = (g.M + P.rows_per_cta - 1) / P.rows_per_cta;
  float *partial = red_partial(ctx, (size_t)splits * P.Kp * g.N);
  P.split = ctx->tc_split ? 1 : 0;
  const size_t st_bytes = ((size_t)(P.Kpad + P.Npad) * 128) << P.split;
  const size_t fixed = 1024 + 8 * (2 * WG_NST + 1) + 16 + WG_NPW * 256 * 4;
  P.nst = (int)std::min<size_t>(WG_NST, (224 * 1024 - fixed) / st_bytes);
  if (P.nst < (P.split ? 2 : 1)) return false;        // caller splits K (3xTF32) or uses the SIMT kernel
  const size_t smem = fixed + P.nst * st_bytes;
  smem_optin((const void *)k_wgrad_tc, 224 * 1024);
#ifdef CHG_TC_DEBUG
  static int skip = getenv("CHG_TC_SKIP") ? atoi(getenv("CHG_TC_SKIP")) : 0;
#else
  const int skip = 0;
#endif
  ProfScope ps(ctx, g.tag ? g.tag : "wgrad_tc", 2.0 * g.M * (double)P.Kp * g.N,
               gemm_a_bytes(g.A, g.M, 0, g.K) + (double)g.M * (4.0 * g.N + (g.didx ? 4.0 : 0.0)) + 4.0 * P.Kp * g.N);
  // partial as a 3-D tensor [splits][K][N] (row stride N, split stride Kp·N): TMA-store epilogue
  CUtensorMap pmap;
  memset(&pmap, 0, sizeof(pmap));
  int use_pmap = 0;
  if (EncodeTiledFn fn = encode_fn(); fn && ((uintptr_t)partial & 15) == 0) {
    cuuint64_t dim[3] = {(cuuint64_t)g.N, (cuuint64_t)g.K, (cuuint64_t)splits};
    cuuint64_t stride[2] = {(cuuint64_t)g.N * 4, (cuuint64_t)P.Kp * g.N * 4};
    cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
    use_pmap = fn(&pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, partial, dim, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (!use_pmap) return false;                        // SIMT weight gradient instead
  launch_k(ctx, k_wgrad_tc, splits, WG_THREADS, smem, ctx->stream, g, P, partial, skip, pmap);
  check_launch(ctx);
  *partial_out = partial;
  *Kp_out = P.Kp;
  *splits_out = splits;
  *bias_done = true;
  return true;
}
