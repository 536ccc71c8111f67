// Auxiliary device kernels of the C-ABI: bench random actions, the PPO
// learner's GAE and the fp32 math self-test (compiled with the fp32 step
// kernel's flags, build.py; GAE uses no division / sqrt).
#include <cuda_runtime.h>

#include "stampede_sim.h"
#include "sim_device.cuh"
#include "sim_launch.h"
#include "stp_error.h"
#include "stp_rng.h"

struct stp_sim;

namespace {

// i.i.d. U[-1,1] actions keyed by derive_seed(seed, TAG_ACTION, env<<32|step)
// (rng.hpp:35-37; SURVEY §8(d) synthetic inputs).
__global__ void k_random_actions(float* out, int n, int J, uint64_t seed, long long env_offset, uint64_t step) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * J) return;
  const int e = int(i / J), j = int(i % J);
  const uint64_t genv = uint64_t(env_offset + e);
  const uint64_t s = stp_derive_seed(seed, STP_TAG_ACTION, (genv << 32) | uint32_t(step));
  out[i] = 2.0f * stp_uniformf(s, uint32_t(j)) - 1.0f;
}

// The fp32-only elementary functions of the step kernel, evaluated on
// caller arrays (DESIGN.md §2 "fp32-only paths"): fn 0 = sincos_(x) ->
// (sin, cos); fn 1 = unit_dir(y = x, x = y) -> (sin, cos) of atan2(x, y).
__global__ void k_debug_math(int fn, const float* x, const float* y, float* o0, float* o1, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s, c;
  if (fn == 0) stp::sincos_(x[i], &s, &c);
  else stp::unit_dir(x[i], y[i], &s, &c);
  o0[i] = s;
  o1[i] = c;
}

// compute_gae for the PPO learner's rollout buffer [T][N]:
// one thread per environment runs the backward recursion
//   delta_t = r_t + gamma V_{t+1} (1 - done_t) - V_t
//   A_t = delta_t + gamma lambda (1 - done_t) A_{t+1},  R_t = A_t + V_t
// (V_T = the bootstrap value), in fp32 like the learner; each block adds its
// advantages' count, sum and sum of squares (double) to stats[3] for the
// global advantage normalisation, so no host round trip.
__global__ void k_gae(const float* __restrict__ rew, const float* __restrict__ val, const uint8_t* __restrict__ done,
                      const float* __restrict__ last_val, int T, int N, float gamma, float lam, float* __restrict__ adv,
                      float* __restrict__ ret, double* __restrict__ stats) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0, sq = 0.0;
  if (e < N) {
    float next_v = last_val[e], a = 0.f;
    for (int t = T - 1; t >= 0; --t) {
      const size_t i = size_t(t) * N + e;
      const float nonterm = done[i] ? 0.f : 1.f;
      const float v = val[i];
      const float delta = rew[i] + gamma * next_v * nonterm - v;
      a = delta + gamma * lam * nonterm * a;
      adv[i] = a;
      ret[i] = a + v;
      s += double(a);
      sq += double(a) * double(a);
      next_v = v;
    }
  }
  if (stats) {
    for (int off = 16; off > 0; off >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, off);
      sq += __shfl_xor_sync(0xffffffffu, sq, off);
    }
    __shared__ double ws[2][32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
      ws[0][w] = s;
      ws[1][w] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bs = 0.0, bq = 0.0;
      for (int k = 0; k < int(blockDim.x >> 5); ++k) {
        bs += ws[0][k];
        bq += ws[1][k];
      }
      const int n_here = min(int(blockDim.x), N - int(blockIdx.x * blockDim.x));
      atomicAdd(stats, double(n_here) * T);
      atomicAdd(stats + 1, bs);
      atomicAdd(stats + 2, bq);
    }
  }
}

}  // namespace

extern "C" int stp_gae(const float* rewards, const float* values, const uint8_t* dones, const float* last_value,
                       int32_t T, int32_t N, float gamma, float lam, float* advantages, float* returns,
                       double* stats, void* stream) {
  if (T < 0 || N < 0 || (T > 0 && N > 0 && (!rewards || !values || !dones || !last_value || !advantages || !returns)))
    return stp::fail(STP_EINVAL, "stp_gae: bad arguments");
  if (T == 0 || N == 0) return STP_OK;
  const int threads = 256;
  k_gae<<<(N + threads - 1) / threads, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      rewards, values, dones, last_value, T, N, gamma, lam, advantages, returns, stats);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_gae: ") + cudaGetErrorString(e));
  return STP_OK;
}

extern "C" int stp_debug_math(int32_t fn, const float* x, const float* y, float* out0, float* out1, int64_t n,
                              void* stream) {
  if (fn < 0 || fn > 1 || n < 0 || (n > 0 && (!x || !out0 || !out1 || (fn == 1 && !y))))
    return stp::fail(STP_EINVAL, "stp_debug_math: bad arguments");
  if (n == 0) return STP_OK;
  const int threads = 256;
  k_debug_math<<<int((n + threads - 1) / threads), threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      fn, x, y, out0, out1, (long long)n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_debug_math: ") + cudaGetErrorString(e));
  return STP_OK;
}

namespace stp {
int sim_dims(const stp_sim* s, int* n, int* J, uint64_t* seed, long long* off, void** stream);
int sim_device(const stp_sim* s);
int sim_order(stp_sim* s, void* stream);
int sim_mark(stp_sim* s, void* stream);
}

extern "C" int stp_random_actions(stp_sim* sim, float* actions, uint64_t step, void* stream) {
  int n = 0, J = 0;
  uint64_t seed = 0;
  long long off = 0;
  void* own = nullptr;
  if (!sim || !actions || stp::sim_dims(sim, &n, &J, &seed, &off, &own) != STP_OK)
    return stp::fail(STP_EINVAL, "stp_random_actions: bad arguments");
  const long long total = (long long)n * J;
  if (total == 0) return STP_OK;
  const stp::DeviceGuard dg_(stp::sim_device(sim));
  const int threads = 256;
  const int blocks = int((total + threads - 1) / threads);
  void* sv = stream ? stream : own;
  if (const int rc = stp::sim_order(sim, sv)) return rc;  // in call order with the handle's other work
  k_random_actions<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(sv)>>>(actions, n, J, seed, off, step);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_random_actions: ") + cudaGetErrorString(e));
  return stp::sim_mark(sim, sv);
}
