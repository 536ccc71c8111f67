// Microbenchmark + check: tcgen05.mma kind::f16 with A (128 x K bf16) from
// shared memory (SS) vs from tensor memory (TS: tcgen05.st of each row,
// lane = row m, column c = bf16 pair (k = 2c, 2c + 1)); B = X^T MN-major in
// shared memory exactly as K4 builds it (N = 64).  Prints max |D - D_ref|
// for both and the clock cycles of a 16-MMA chain (issue -> commit done).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
constexpr int M = 128, N = 64, K = 256, KS = K / 16;
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
// A: [M][K] row-major bf16 (global); B: [K][N] row-major bf16 (global); D: [M][N] f32 out (2 copies)
__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  __nv_bfloat16* As = (__nv_bfloat16*)sm;            // K-major core matrices: [K/8][M][8]
  __nv_bfloat16* Bs = (__nv_bfloat16*)(sm + M * K * 2);  // MN-major: chunk (n/8)*K + k holds n..n+7 of row k
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, kk = i % K;
    As[((kk / 8) * M + m) * 8 + kk % 8] = A[i];
  }
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int kk = i / N, n = i % N;
    Bs[((n / 8) * K + kk) * 8 + n % 8] = B[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t0 = tm;
  const uint32_t a_tm = t0 + 2 * N;  // A in TMEM at columns [2N, 2N + K/2)
  // rows of A into TMEM: warp w (of 4) = lanes 32w..; thread = row m, K/2 columns in chunks of 32
  if (warp < 4) {
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 32) {
      uint32_t r[32];
      for (int c = 0; c < 32; ++c) {
        __nv_bfloat162 p = __halves2bfloat162(A[m * K + 2 * (c0 + c)], A[m * K + 2 * (c0 + c) + 1]);
        r[c] = *reinterpret_cast<uint32_t*>(&p);
      }
      const uint32_t ta = a_tm + (uint32_t(warp * 32) << 16) + uint32_t(c0);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(ta),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(N >> 3) << 17) |
                         (uint32_t(M >> 4) << 24);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      long long c0 = 0, c1 = 0;
      if (warp == 0 && elect_one()) {
        c0 = clock64();
        for (int ks = 0; ks < KS; ++ks) {
          const uint64_t db = desc(sa(Bs) + ks * 256, 128, K * 16);
          const uint32_t dt = t0 + uint32_t(mode * N);
          if (mode == 0) {
            const uint64_t da = desc(sa(As) + ks * 2 * M * 16, M * 16, 128);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(dt),
                         "l"(da), "l"(db), "r"(idesc), "r"(ks));
          } else {
            const uint32_t at = a_tm + uint32_t(ks * 8);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(dt),
                         "r"(at), "l"(db), "r"(idesc), "r"(ks));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)sa(&bar)) : "memory");
      }
      __syncwarp();
      asm volatile("{\n.reg .pred d;\nW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n@!d bra W;\n}" ::"r"(sa(&bar)),
                   "r"((mode * 2 + rep) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (warp == 0 && lane == 0) c1 = clock64();
      if (tid == 0) cyc[mode] = c1 - c0;
    }
  }
  // read back both accumulators: warp w of 4 = lanes 32w.., 2 x N columns
  if (warp < 4) {
    const int m = warp * 32 + lane;
    for (int c = 0; c < 2 * N; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(t0 + (uint32_t(warp * 32) << 16) + uint32_t(c)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 16; ++i) {
        const int col = c + i, mode = col / N, n = col % N;
        D[(mode * M + m) * N + n] = __uint_as_float(r[i]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  std::vector<__nv_bfloat16> A(M * K), B(K * N);
  std::vector<float> Af(M * K), Bf(K * N);
  srand(1);
  for (int i = 0; i < M * K; ++i) { A[i] = __float2bfloat16(rand() / float(RAND_MAX) - 0.5f); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < K * N; ++i) { B[i] = __float2bfloat16(rand() / float(RAND_MAX) - 0.5f); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dD; long long* dc;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, K * N * 2); cudaMalloc(&dD, 2 * M * N * 4); cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), K * N * 2, cudaMemcpyHostToDevice);
  const int smem = M * K * 2 + K * N * 2;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(dA, dB, dD, dc);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> D(2 * M * N); long long cyc[2];
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
  for (int mode = 0; mode < 2; ++mode) {
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int kk = 0; kk < K; ++kk) r += double(Af[m * K + kk]) * Bf[kk * N + n];
        err = fmax(err, fabs(r - D[(mode * M + m) * N + n]));
      }
    printf("%s: max |D - ref| %.3e, %d-MMA chain %lld cycles\n", mode ? "TS (A in TMEM)" : "SS (A in smem)", err, KS, cyc[mode]);
  }
}
