// Latency probe: per-iteration cost of (a) mbarrier arrive + wait, (b) tcgen05.commit -> mbarrier
// + wait, (c) (b) + tcgen05.fence::after_thread_sync, for one thread of one CTA (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cp tools/commit_probe.cu && /tmp/cp
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}

__global__ void probe(long long *out, int iters) {
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {   // (a) plain arrive + wait
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
      wait(&bar, ph); ph ^= 1;
    }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) {   // (b) tcgen05.commit -> mbarrier + wait
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"((uint64_t)su32(&bar)) : "memory");
      wait(&bar, ph); ph ^= 1;
    }
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {   // (c) fence + commit + wait
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"((uint64_t)su32(&bar)) : "memory");
      wait(&bar, ph); ph ^= 1;
    }
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) {   // (d) commit only (no wait), then one wait at the end
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"((uint64_t)su32(&bar)) : "memory");
    }
    long long t4 = clock64();
    out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters; out[3] = (t4 - t3) / iters;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot) : "memory");
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, 32);
  probe<<<1, 128>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("%s | cycles/iter: arrive+wait %lld  commit+wait %lld  fence+commit+wait %lld  commit-only %lld\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  return 0;
}
