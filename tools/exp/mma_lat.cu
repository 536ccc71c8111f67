// Microbenchmark: cost of a chain of R tcgen05.mma (kind::f16, M = 128, K = 16)
// issued back to back by one thread, vs N, measured with clock64 from the
// first issue to the commit's mbarrier completion (one CTA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) | (uint64_t((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__global__ void k(int N, int R, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  uint16_t* A = (uint16_t*)sm;            // 128 x 16 bf16
  uint16_t* B = (uint16_t*)(sm + 4096);   // N x 16 bf16
  for (int i = threadIdx.x; i < (4096 + 256 * 32) / 2; i += blockDim.x) ((uint16_t*)sm)[i] = 0x3c00;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    uint64_t da = desc(sa(A), 128 * 16, 128), db = desc(sa(B), N * 16, 128);
    for (int warm = 0; warm < 2; ++warm) {
      long long t0 = clock64();
      for (int r = 0; r < R; ++r) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(r));
      }
      long long t1 = clock64();
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)sa(&bar)) : "memory");
      asm volatile("{\n.reg .pred d;\nW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n@!d bra W;\n}" ::"r"(sa(&bar)), "r"(warm));
      long long t2 = clock64();
      out[0] = t1 - t0; out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) { asm volatile("tcgen05.fence::after_thread_sync;"); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm)); }
}
int main() {
  long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (int N : {16, 32, 64, 128, 256})
    for (int R : {1, 8, 16, 32}) {
      k<<<1, 128, 16384>>>(N, R, d);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("N %3d R %2d: issue %5lld cycles, to completion %5lld cycles (%.0f per MMA)\n", N, R, h[0], h[1], double(h[1]) / R);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
