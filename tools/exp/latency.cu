// Dependent-chain latency of the instructions the PCR loop is built from
// (one warp, clock64 around N chained ops).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void k(float* out, long long* cyc, float seed) {
  __shared__ float sm[64];
  const int lane = threadIdx.x;
  float v = seed + lane;
  unsigned u = __float_as_uint(v);
  sm[lane] = v;
  sm[lane + 32] = v;
  __syncwarp();
  long long t0, t1;
  int slot = 0;
#define TIME(body)                                        \
  t0 = clock64();                                         \
  _Pragma("unroll 16") for (int i = 0; i < N; ++i) { body; } \
  t1 = clock64();                                         \
  if (lane == 0) cyc[slot] = t1 - t0;                     \
  ++slot;
  TIME(v = fmaf(v, 1.0001f, 0.5f))                                  // 0 FFMA
  TIME(v = v + 0.25f)                                               // 1 FADD
  TIME(v += __shfl_xor_sync(0xffffffffu, v, 1))                     // 2 SHFL.BFLY + FADD
  TIME(v += __shfl_sync(0xffffffffu, v, (lane + 1) & 31))           // 3 SHFL.IDX + FADD
  TIME(u = __reduce_add_sync(0xffffffffu, u))                       // 4 REDUX.SUM
  TIME(u = __reduce_max_sync(0xffffffffu, u) ^ lane)                // 5 REDUX.MAX + LOP
  TIME(v = __frcp_rn(v) + 1.0f)                                     // 6 MUFU.RCP (+ fixup) + FADD
  TIME(v = __fdividef(1.0f, v) + 1.0f)                              // 7 fast div
  TIME(v = __int2float_rn(__float2int_rn(v) + 1))                   // 8 F2I + IADD + I2F
  TIME(v = sm[(__float_as_uint(v) & 31u)] + 1.0f)                   // 9 LDS + FADD
  TIME(sm[lane] = v; __syncwarp(); v = sm[lane ^ 1] + 1.0f; __syncwarp())  // 10 STS + LDS
  TIME(v = sqrtf(v) + 1.0f)                                         // 11 sqrt
  float2 v2 = make_float2(v, v + 1.f);
  TIME(v2 = __ffma2_rn(v2, make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f)))  // 12 FFMA2
  out[threadIdx.x] = v + __uint_as_float(u) + v2.x + v2.y;
}

template <bool PACKED>
__global__ void thr(float* out, long long* cyc, float seed) {
  float a[8];
  float2 b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = make_float2(a[2 * j], a[2 * j + 1]);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    if (PACKED) {
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = __ffma2_rn(b[j], make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f));
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 1.0001f, 0.5f);
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
#pragma unroll
  for (int j = 0; j < 4; ++j) s += b[j].x + b[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(float));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  k<<<1, 32>>>(out, cyc, 1.0f);  // warm
  k<<<1, 32>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  const char* names[] = {"FFMA", "FADD", "SHFL.BFLY+FADD", "SHFL.IDX+FADD", "REDUX.SUM", "REDUX.MAX+LOP",
                         "RCP+FADD", "fdividef+FADD", "F2I+IADD+I2F", "LDS+FADD", "STS+LDS+FADD (2 syncwarp)",
                         "sqrt+FADD", "FFMA2"};
  for (int i = 0; i < 13; ++i) printf("%-28s %6.1f cycles\n", names[i], double(cyc[i]) / N);
  float* o2;
  cudaMalloc(&o2, 148 * 1024 * sizeof(float));
  for (int w : {4, 8, 16, 32}) {
    thr<false><<<148, 32 * w>>>(o2, cyc, 1.0f);
    thr<false><<<148, 32 * w>>>(o2, cyc, 1.0f);
    cudaDeviceSynchronize();
    const double cf = double(cyc[0]);
    thr<true><<<148, 32 * w>>>(o2, cyc, 1.0f);
    thr<true><<<148, 32 * w>>>(o2, cyc, 1.0f);
    cudaDeviceSynchronize();
    const double cp = double(cyc[0]);
    // 8 fp32 FMA per thread-iteration either way
    printf("warps/SM %2d: FFMA %.2f FMA/clk/SM, FFMA2 %.2f FMA/clk/SM\n", w, 8.0 * N * 32 * w / cf, 8.0 * N * 32 * w / cp);
  }
  return 0;
}
