// Probe: tcgen05.mma issue/execution rate in isolation (one CTA, operands resident in smem).
// For each (kind, N, B layout, accumulators): R rounds of `per` MMAs (M = 128, K = 32 B of K)
// chained into TMEM, one commit at the end; prints cycles per MMA.  Compare with the
// tcgen05 floor max(M,128)·N/256 cycles (B300_MICROARCH.md) to see what the row GEMM's
// measured ~0.5-1 us per 32-wide K stage is made of.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)lay << 61);
}

// mode bit 0: B SW128 (else interleaved / SWIZZLE_NONE); bit 1: bf16 (kind::f16) else tf32;
// bit 2: alternate between 2 accumulators (independent chains); nis: issuing warps (lane 0 of
// warps 0..nis-1, each into its own TMEM columns)
__global__ void rate(long long *out, int N, int mode, int rounds, int per, int nis) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *sm = raw + ((1024 - (su(raw) & 1023)) & 1023);
  uint8_t *sA = sm, *sB = sm + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (16384 + 32768) / 4; i += blockDim.x) ((uint32_t *)sm)[i] = 0x3f800000u;   // 1.0f
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(nis));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if ((tid & 31) == 0 && tid / 32 < nis) {
    const int w = tid / 32;
    const bool bsw = mode & 1, bf = mode & 2, two = mode & 4;
    const uint32_t idesc = (1u << 4) | (bf ? (1u << 7) | (1u << 10) : (2u << 7) | (2u << 10)) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    // descriptors precomputed (the loop issues only MMAs); K steps jj = j & 3 advance 32 B
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      ad[jj] = desc(su(sA) + jj * 32, 16, 1024, 2);
      bd[jj] = bsw ? desc(su(sB) + jj * 32, 16, 1024, 2) : desc(su(sB) + jj * 2 * (N * 16), N * 16, 128, 0);
    }
    const uint32_t d0 = tm + (nis > 1 ? w * (512 / nis) : 0), d1 = tm + (nis > 1 ? w * (512 / nis) : (two ? 256 : 0));
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const uint32_t d = (j & 1) ? d1 : d0;
        const uint32_t acc = (r > 0 || j > 1) ? 1u : 0u;
        if (mode & 8)   // A from TMEM (columns 384 + 8 jj), B from smem
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                       "r"(tm + 384 + 8 * (j & 3)), "l"(bd[j & 3]), "r"(idesc), "r"(acc));
        else if (bf)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(ad[j & 3]), "l"(bd[j & 3]), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(ad[j & 3]), "l"(bd[j & 3]), "r"(idesc), "r"(acc));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"((uint64_t)__cvta_generic_to_shared(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(&bar)));
    long long t2 = clock64();
    if (w == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  const int Ns[3] = {64, 128, 256};
  for (int nis = 1; nis <= 2; nis *= 2)
    for (int mode = 0; mode <= 8; mode += 8)
      for (int ni = 0; ni < 3; ++ni) {
        const int N = Ns[ni], rounds = 200, per = 12;
        if (nis == 2 && N > 128) continue;
        rate<<<1, 128, 52000>>>(d, N, mode, rounds, per, nis);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double n = (double)rounds * per;
        printf("%s N=%3d issuers=%d: per issuer %.1f cyc/MMA issue, %.1f complete; all issuers: %.1f cyc/MMA (floor %d) %s\n",
               (mode & 8) ? "tf32 A-in-TMEM" : (mode & 2) ? "bf16" : "tf32", N, nis, h[0] / n, h[1] / n, h[1] / (n * nis), 128 * N / 256, cudaGetErrorString(e));
      }
  return 0;
}
