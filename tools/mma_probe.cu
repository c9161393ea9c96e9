// Probe: one tcgen05.mma.kind::tf32, M=128 N=32 K=8, operands MN-major SWIZZLE_128B.
// A[m][k] = (m == k) ? 1 : 0 ; B[n][k] = n + 100 k  ->  D[m][n] = B[n][m] for m < 8, else 0.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)lay << 61);
}
__device__ __forceinline__ uint32_t mn_swz(int mn, int kk) {
  return (uint32_t)((mn >> 5) * 4096 + (kk >> 3) * 1024 + (kk & 7) * 128 + ((((mn & 31) >> 2) ^ (kk & 7)) << 4) + (mn & 3) * 4);
}
__global__ void probe(float *out, int mode) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *sm = raw + ((1024 - (su(raw) & 1023)) & 1023);
  uint8_t *sA = sm, *sB = sm + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  int tid = threadIdx.x;
  for (int i = tid; i < 16384 / 4 * 2; i += blockDim.x) ((float *)sm)[i] = 0.f;
  __syncthreads();
  if (tid < 128) {
    int m = tid;
    for (int k = 0; k < 8; ++k) {
      float v = (m == k) ? 1.f : 0.f;
      if (mode == 3) *(float *)(sA + (m >> 2) * 128 + (k & 7) * 16 + (m & 3) * 4) = v;   // MN-major INTERLEAVE
      else if (mode != 1) *(float *)(sA + mn_swz(m, k)) = v;                       // MN-major SW128
      else *(float *)(sA + m * 128 + ((((k >> 2)) ^ (m & 7)) << 4) + (k & 3) * 4) = v;  // K-major SW128
    }
  }
  if (tid < 32) {
    int n = tid;
    for (int k = 0; k < 8; ++k) {
      float v = n + 100.f * k;
      if (mode == 3) *(float *)(sB + (n >> 2) * 128 + (k & 7) * 16 + (n & 3) * 4) = v;
      else if (mode != 1) *(float *)(sB + mn_swz(n, k)) = v;
      else *(float *)(sB + n * 128 + ((((k >> 2)) ^ (n & 7)) << 4) + (k & 3) * 4) = v;
    }
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  if (tid == 0) {
    uint32_t idesc, mj = (mode != 1) ? 1u : 0u;
    idesc = (1u << 4) | (2u << 7) | (2u << 10) | (mj << 15) | (mj << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t ad, bd;
    if (mode == 0) { ad = desc(su(sA), 4096, 1024, 2); bd = desc(su(sB), 4096, 1024, 2); }
    else if (mode == 2) { ad = desc(su(sA), 1024, 4096, 2); bd = desc(su(sB), 1024, 4096, 2); }
    else if (mode == 3) { ad = desc(su(sA), 128 * 32, 128, 0); bd = desc(su(sB), 128 * 8, 128, 0); }
    else { ad = desc(su(sA), 16, 1024, 2); bd = desc(su(sB), 16, 1024, 2); }
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"((uint64_t)__cvta_generic_to_shared(&bar)));
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid < 128) {
    uint32_t r[32];
    uint32_t ta = tm + ((uint32_t)((tid / 32) * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) out[tid * 32 + j] = __uint_as_float(r[j]);
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  float *d, h[128 * 32];
  cudaMalloc(&d, sizeof(h));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(d, 0, sizeof(h));
    probe<<<1, 128, 36000>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d (%s) err=%s\n", mode, mode == 0 ? "MN-major" : mode == 1 ? "K-major" : mode == 2 ? "MN-major lbo/sbo swapped" : "MN-major interleave", cudaGetErrorString(e));
    for (int m = 0; m < 10; ++m) { printf(" D[%d][0..5] =", m); for (int n = 0; n < 6; ++n) printf(" %7.1f", h[m * 32 + n]); printf("\n"); }
  }
  return 0;
}
