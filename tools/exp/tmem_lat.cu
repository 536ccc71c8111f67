// Microbenchmark: latency of tcgen05.ld.32x32b.x16 + tcgen05.wait::ld with 4 or
// 16 warps loading at once (clock64 per warp), and of a 10-MMA chain issued
// from an elected lane (M = 128, N = 64, K = 16, SS operands).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3fff) | (uint64_t((lbo >> 4) & 0x3fff) << 16) | (uint64_t((sbo >> 4) & 0x3fff) << 32) |
         (1ull << 46);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "+r"(pred));
  return pred != 0;
}
__global__ void k(int nw_load, long long* out, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (4096 * 10 + 2048 * 10) / 2; i += blockDim.x) ((uint16_t*)sm)[i] = 0x3c00;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  float acc = 0.f;
  for (int rep = 0; rep < 3; ++rep) {
    // MMA chain: 10 x (M128 N64 K16), A 4 KB + B 2 KB per MMA from smem
    long long t0 = clock64(), t1 = 0;
    if (warp == 0 && elect_one()) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(64 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
      uint64_t da = desc(sa(sm), 128 * 16 * 10, 128), db = desc(sa(sm + 40960), 64 * 16 * 10, 128);
#pragma unroll
      for (int r = 0; r < 10; ++r) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                     "l"(da + r * 16), "l"(db + r * 16), "r"(idesc), "r"(r));
      }
      t1 = clock64();
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)sa(&bar)) : "memory");
    }
    __syncwarp();
    asm volatile("{\n.reg .pred d;\nW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n@!d bra W;\n}" ::"r"(sa(&bar)),
                 "r"(rep & 1));
    asm volatile("tcgen05.fence::after_thread_sync;");
    long long t2 = clock64();
    // TMEM loads: nw_load warps at once (warp w reads lanes 32 (w % 4)..)
    long long t3 = t2, t4 = t2;
    if (warp < nw_load) {
      uint32_t r[16];
      const uint32_t ta = tm + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 16);
      t3 = clock64();
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      t4 = clock64();
      for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if ((threadIdx.x & 31) == 0 && rep == 2) {
      long long* o = out + warp * 4;
      o[0] = t1 - t0; o[1] = t2 - t0; o[2] = t4 - t3; o[3] = t4 - t2;
    }
  }
  sink[threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}
int main() {
  long long* out;
  float* sink;
  cudaMalloc(&out, 16 * 4 * 8);
  cudaMalloc(&sink, 512 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int nw : {1, 4, 16}) {
    k<<<1, 512, 64 * 1024>>>(nw, out, sink);
    long long h[64];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("load warps %2d: mma issue %lld cyc, mma done %lld cyc; tmem ld+wait per warp:", nw, h[0], h[1]);
    for (int w = 0; w < nw; ++w) printf(" %lld", h[w * 4 + 2]);
    printf("\n");
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
