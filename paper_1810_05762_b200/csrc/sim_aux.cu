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

// ppo_update's minibatch loss head and its gradient with
// respect to the networks' outputs, one thread per sample i of the minibatch:
//   logp_i = sum_j -z_ij^2 / 2 - ls_j - log(2 pi) / 2,  z = (a - mu) / sigma
//   r_i = exp(logp_i - logp_old),  Ahat = (A - mean) / std (global stats)
//   L = -mean_i min(r Ahat, clip(r, 1-eps, 1+eps) Ahat) + c_v mean_i (V - R)^2
// dL/dmu_ij = g_i z_ij / sigma_j, dL/dls_j = sum_i g_i (z_ij^2 - 1) with
// g_i = dL/dlogp_i; dL/dV_i = 2 c_v (V_i - R_i) / B.  The min / clamp
// derivatives follow autograd's (ties split the gradient in half; the clamp
// passes it on [lo, hi]).  Rollout columns (actions, old log-prob, A, R) are
// read through the minibatch's permutation idx, so the gather is fused.
// Block partials [2A + 3] (dL/dls, the column sums of dL/dmu and dL/dV —
// the heads' bias gradients — the surrogate sum, the value-error sum) go to
// scratch and are summed in a fixed order by k_ppo_finish: deterministic.
// The tile's mu rows (contiguous), gathered action rows and the d_mu
// result move through shared memory with coalesced loads / stores (row
// stride A | 1 words: conflict-free column reads); the per-sample math reads
// the tiles.
constexpr int kPpoThreads = 128;
constexpr int kPpoMaxA = 32;

__global__ void __launch_bounds__(kPpoThreads) k_ppo_head(
    const float* __restrict__ mu, const float* __restrict__ log_std, const float* __restrict__ value,
    const float* __restrict__ actions, const float* __restrict__ old_logp, const float* __restrict__ adv,
    const float* __restrict__ ret, const int64_t* __restrict__ idx, int B, int A, const double* __restrict__ adv_stats,
    float clip, float vf_coef, float* __restrict__ d_mu, float* __restrict__ d_value, double* __restrict__ partials) {
  __shared__ float s_ls[kPpoMaxA], s_isig[kPpoMaxA];
  __shared__ float s_mu[kPpoThreads * (kPpoMaxA + 1)], s_a[kPpoThreads * (kPpoMaxA + 1)];
  __shared__ long long s_row[kPpoThreads];
  __shared__ double s_red[kPpoThreads / 32][3];
  const int SA = A | 1;
  const int i0 = blockIdx.x * kPpoThreads;
  const int nrow = min(kPpoThreads, B - i0);
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    s_ls[j] = log_std[j];
    s_isig[j] = expf(-log_std[j]);
  }
  if (threadIdx.x < nrow) s_row[threadIdx.x] = idx ? (long long)idx[i0 + threadIdx.x] : (long long)(i0 + threadIdx.x);
  __syncthreads();
  for (int e = threadIdx.x; e < nrow * A; e += kPpoThreads) {  // coalesced tile loads
    const int r = e / A, c = e - r * A;
    s_mu[r * SA + c] = mu[(long long)i0 * A + e];
    s_a[r * SA + c] = actions[s_row[r] * A + c];
  }
  __syncthreads();
  double an_mean = 0.0, an_inv = 1.0;
  if (adv_stats) {  // global_normalize, in double like the host
    const double n = adv_stats[0], mean = adv_stats[1] / n;
    an_mean = mean;
    an_inv = 1.0 / (sqrt(fmax(adv_stats[2] / n - mean * mean, 0.0)) + 1e-8);
  }
  const float inv_b = 1.0f / float(B);
  const float kHalfLog2Pi = 0.91893853320467274f;
  const int t = threadIdx.x, i = i0 + t;
  const int lane = t & 31, warp = t >> 5;
  double acc_pg = 0.0, acc_vf = 0.0, acc_dv = 0.0;
  float g = 0.f;
  float* a_row = s_a + t * SA;
  float* mu_row = s_mu + t * SA;
  if (t < nrow) {
    const long long k = s_row[t];
    float logp = 0.f;
    for (int j = 0; j < A; ++j) {
      const float z = (a_row[j] - mu_row[j]) * s_isig[j];
      logp += -0.5f * z * z - s_ls[j] - kHalfLog2Pi;
    }
    const float r = expf(logp - old_logp[k]);
    const float ah = float((double(adv[k]) - an_mean) * an_inv);
    const float lo = 1.f - clip, hi = 1.f + clip;
    // clamp and min propagate NaN like torch's (fminf / fmaxf would drop it)
    const float c = r != r ? r : fminf(fmaxf(r, lo), hi);
    const float s1 = r * ah, s2 = c * ah;
    const float pass = (r >= lo && r <= hi) ? 1.f : 0.f;
    const float dmin_dr = s1 < s2 ? ah : (s1 == s2 ? 0.5f * ah + 0.5f * ah * pass : ah * pass);
    g = -inv_b * dmin_dr * r;  // dL/dlogp_i
    acc_pg = (s1 != s1 || s2 != s2) ? double(s1 + s2) : double(fminf(s1, s2));
    const float dv = value[i] - ret[k];
    acc_vf = double(dv) * double(dv);
    const float dvo = 2.f * vf_coef * dv * inv_b;
    d_value[i] = dvo;
    acc_dv = double(dvo);
  }
  // per output column: d_mu into the mu tile and g (z^2 - 1) into the action
  // tile, in place (each entry is read before it is overwritten)
  if (t < nrow) {
    for (int j = 0; j < A; ++j) {
      const float z = (a_row[j] - mu_row[j]) * s_isig[j];
      mu_row[j] = g * z * s_isig[j];
      a_row[j] = g * (z * z - 1.f);
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    acc_pg += __shfl_xor_sync(0xffffffffu, acc_pg, off);
    acc_vf += __shfl_xor_sync(0xffffffffu, acc_vf, off);
    acc_dv += __shfl_xor_sync(0xffffffffu, acc_dv, off);
  }
  if (lane == 0) {
    s_red[warp][0] = acc_dv;
    s_red[warp][1] = acc_pg;
    s_red[warp][2] = acc_vf;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nrow * A; e += kPpoThreads) {  // coalesced d_mu store
    const int r = e / A, c = e - r * A;
    d_mu[(long long)i0 * A + e] = s_mu[r * SA + c];
  }
  // column sums of the two tiles (dL/dls, then dL/dmu): warp w takes columns
  // w, w + 4, ...; lane l adds rows l, l + 32, ... in double, then a fixed tree
  double* out = partials + (long long)blockIdx.x * (2 * A + 3);
  for (int col = warp; col < 2 * A; col += kPpoThreads / 32) {
    const float* tile = col < A ? s_a + col : s_mu + (col - A);
    double sm = 0.0;
    for (int r = lane; r < nrow; r += 32) sm += double(tile[r * SA]);
    for (int off = 16; off > 0; off >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, off);
    if (lane == 0) out[col] = sm;
  }
  if (threadIdx.x < 3) {
    double sm = 0.0;
    for (int w = 0; w < kPpoThreads / 32; ++w) sm += s_red[w][threadIdx.x];
    out[2 * A + threadIdx.x] = sm;
  }
}

// Sums the block partials: d_log_std[A], the heads' bias gradients, loss[3]
// = (total, surrogate, value error) and bad = max(bad, loss not finite)
// (ppo.py's abort flag, read once after the epochs).  Block c < 2A + 1 owns
// column c, the last block the two loss columns; each column is summed by
// 256 threads in a fixed order (strided partial sums, then a fixed tree):
// deterministic.
__device__ double colsum_fixed(const double* __restrict__ partials, int nblk, int ncol, int c, double* s_tree) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partials[(long long)b * ncol + c];
  s_tree[threadIdx.x] = s;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) s_tree[threadIdx.x] += s_tree[threadIdx.x + h];
    __syncthreads();
  }
  const double r = s_tree[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) k_ppo_finish(const double* __restrict__ partials, int nblk, int A, int B,
                                                    float vf_coef, float* __restrict__ d_log_std,
                                                    float* __restrict__ d_mu_bias, float* __restrict__ d_value_bias,
                                                    float* __restrict__ loss, float* __restrict__ bad) {
  __shared__ double s_tree[256];
  const int ncol = 2 * A + 3, c = blockIdx.x;
  if (c < 2 * A + 1) {
    const double s = colsum_fixed(partials, nblk, ncol, c, s_tree);
    if (threadIdx.x == 0) {
      if (c < A) d_log_std[c] = float(s);
      else if (c < 2 * A) { if (d_mu_bias) d_mu_bias[c - A] = float(s); }
      else if (d_value_bias) *d_value_bias = float(s);
    }
    return;
  }
  const double pg = colsum_fixed(partials, nblk, ncol, 2 * A + 1, s_tree);
  const double vf = colsum_fixed(partials, nblk, ncol, 2 * A + 2, s_tree);
  if (threadIdx.x == 0) {
    loss[1] = float(-pg / B);
    loss[2] = float(vf / B);
    const float total = loss[1] + vf_coef * loss[2];
    loss[0] = total;
    if (bad && !isfinite(total)) *bad = 1.f;
  }
}

// KL(old || new) of the diagonal Gaussian policies averaged over the batch
// (kl_diag_gaussian; the learning-rate rule's input,
// :468-475): one thread per state, per-block double sums, then a fixed-order
// sum in k_kl_finish (deterministic).
constexpr int kKlThreads = 256;

__global__ void __launch_bounds__(kKlThreads) k_kl(const float* __restrict__ mu0, const float* __restrict__ ls0,
                                                   const float* __restrict__ mu1, const float* __restrict__ ls1,
                                                   int B, int A, double* __restrict__ partials) {
  __shared__ double s_w[kKlThreads / 32];
  const int i = blockIdx.x * kKlThreads + threadIdx.x;
  double kl = 0.0;
  if (i < B) {
    float acc = 0.f;
    for (int j = 0; j < A; ++j) {
      const float v0 = expf(2.f * ls0[j]), v1 = expf(2.f * ls1[j]);
      const float d = mu0[(long long)i * A + j] - mu1[(long long)i * A + j];
      acc += ls1[j] - ls0[j] + (v0 + d * d) / (2.f * v1) - 0.5f;
    }
    kl = double(acc);
  }
  for (int off = 16; off > 0; off >>= 1) kl += __shfl_xor_sync(0xffffffffu, kl, off);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = kl;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kKlThreads / 32; ++w) t += s_w[w];
    partials[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) k_kl_finish(const double* __restrict__ partials, int nblk, int B,
                                                   float* __restrict__ out) {
  __shared__ double s_tree[256];
  const double s = colsum_fixed(partials, nblk, 1, 0, s_tree);
  if (threadIdx.x == 0) *out = float(s / B);
}

// Backward of one hidden layer's SELU for the learner (§4.4 SELU
// networks): g = dy * selu'(z) from the layer's OUTPUT y (y > 0: lambda;
// else y + lambda alpha = lambda alpha e^z, autograd's result form), written
// over dy, and the bias gradient db = sum over rows of g.  One pass over the
// [rows][H] activations (float4 along H); each block reduces its row range
// per column in registers + shared memory and writes one partial row, which
// k_colsum_finish adds in block order (deterministic).
constexpr int kSeluThreads = 256;
constexpr int kSeluBlocks = 148 * 4;  // 4 blocks per SM; the row split depends only on rows and H

__global__ void __launch_bounds__(kSeluThreads) k_selu_bwd_bias(float* __restrict__ g, const float* __restrict__ y,
                                                               long long rows, int H, long long rows_per_block,
                                                               float* __restrict__ partials) {
  extern __shared__ float s_part[];  // [kSeluThreads / (H/4)][H]
  const float kL = 1.0507009873554805f, kLA = 1.0507009873554805f * 1.6732632423543772f;
  const int q = H >> 2;                       // float4 per row
  const int c4 = threadIdx.x % q, rlane = threadIdx.x / q, rpar = kSeluThreads / q;
  const long long r0 = (long long)blockIdx.x * rows_per_block;
  const long long r1 = min(rows, r0 + rows_per_block);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (rlane < rpar) {
#pragma unroll 4
    for (long long r = r0 + rlane; r < r1; r += rpar) {
      float4* gp = reinterpret_cast<float4*>(g + r * H) + c4;
      const float4 yv = __ldcs(reinterpret_cast<const float4*>(y + r * H) + c4);
      float4 d = *gp;
      d.x *= yv.x > 0.f ? kL : yv.x + kLA;
      d.y *= yv.y > 0.f ? kL : yv.y + kLA;
      d.z *= yv.z > 0.f ? kL : yv.z + kLA;
      d.w *= yv.w > 0.f ? kL : yv.w + kLA;
      *gp = d;
      acc.x += d.x;
      acc.y += d.y;
      acc.z += d.z;
      acc.w += d.w;
    }
    reinterpret_cast<float4*>(s_part + rlane * H)[c4] = acc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += kSeluThreads) {
    float s = 0.f;
    for (int k = 0; k < rpar; ++k) s += s_part[k * H + c];
    partials[(long long)blockIdx.x * H + c] = s;
  }
}

// Column sums of partials [nblk][H]: a block per 32 columns, warp w adds
// the rows b = w, w + 8, ... in order, then the 8 warp sums in order
// (coalesced, deterministic).
__global__ void __launch_bounds__(256) k_colsum_finish(const float* __restrict__ partials, int nblk, int H,
                                                       float* __restrict__ out) {
  __shared__ float s_w[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < H)
    for (int b = w; b < nblk; b += 8) s += partials[(long long)b * H + c];
  s_w[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < H) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += s_w[k][lane];
    out[c] = t;
  }
}

// Forward epilogue of a learner layer: z += bias (+ SELU) in place over the
// GEMM's [rows][H] output, float4 along H (the bias / SELU of the forward
// as one pass instead of a GEMM epilogue plus an elementwise pass).
// e^x - 1 for x <= 0 without expm1f's slow path: a degree-7 Taylor polynomial
// on [-1/2, 0] (truncation < |x|^8 / 40320: < 2.5e-7 relative), else the
// MUFU exponential minus 1 (|e^x - 1| >= 0.39 there, so the subtraction keeps
// ~4e-7 relative); branch-free.
__device__ __forceinline__ float expm1_neg(float x) {
  float p = fmaf(x, 1.f / 5040.f, 1.f / 720.f);
  p = fmaf(x, p, 1.f / 120.f);
  p = fmaf(x, p, 1.f / 24.f);
  p = fmaf(x, p, 1.f / 6.f);
  p = fmaf(x, p, 0.5f);
  p = fmaf(x, p, 1.f);
  const float small = x * p;
  const float big = __expf(x) - 1.f;
  return x > -0.5f ? small : big;
}

__global__ void k_bias_selu(float* __restrict__ z, const float* __restrict__ bias, long long n4, int q, int selu) {
  const float kL = 1.0507009873554805f, kLA = 1.0507009873554805f * 1.6732632423543772f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 b = reinterpret_cast<const float4*>(bias)[i % q];
    float4 v = reinterpret_cast<float4*>(z)[i];
    v.x += b.x;
    v.y += b.y;
    v.z += b.z;
    v.w += b.w;
    if (selu) {
      v.x = v.x > 0.f ? kL * v.x : kLA * expm1_neg(v.x);
      v.y = v.y > 0.f ? kL * v.y : kLA * expm1_neg(v.y);
      v.z = v.z > 0.f ? kL * v.z : kLA * expm1_neg(v.z);
      v.w = v.w > 0.f ? kL * v.w : kLA * expm1_neg(v.w);
    }
    reinterpret_cast<float4*>(z)[i] = v;
  }
}

}  // namespace

extern "C" int stp_bias_selu(float* z, const float* bias, int64_t rows, int32_t H, int32_t selu, void* stream) {
  if (rows < 0 || H <= 0 || (H & 3) || !bias || (rows > 0 && !z) || (reinterpret_cast<uintptr_t>(z) & 15) ||
      (reinterpret_cast<uintptr_t>(bias) & 15))
    return stp::fail(STP_EINVAL, "stp_bias_selu: bad arguments");
  const long long n4 = (long long)rows * (H / 4);
  if (n4 == 0) return STP_OK;
  const int threads = 256;
  const long long want = (n4 + threads - 1) / threads;
  const int blocks = int(want < 148LL * 16 ? want : 148LL * 16);
  k_bias_selu<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(z, bias, n4, H / 4, selu);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_bias_selu: ") + cudaGetErrorString(e));
  return STP_OK;
}

extern "C" int stp_ppo_kl(const float* mu_old, const float* log_std_old, const float* mu_new,
                          const float* log_std_new, int32_t B, int32_t A, float* kl_mean, double* scratch,
                          void* stream) {
  if (B <= 0 || A <= 0 || !mu_old || !log_std_old || !mu_new || !log_std_new || !kl_mean || !scratch)
    return stp::fail(STP_EINVAL, "stp_ppo_kl: bad arguments");
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nblk = (B + kKlThreads - 1) / kKlThreads;
  k_kl<<<nblk, kKlThreads, 0, st>>>(mu_old, log_std_old, mu_new, log_std_new, B, A, scratch);
  k_kl_finish<<<1, 256, 0, st>>>(scratch, nblk, B, kl_mean);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_kl: ") + cudaGetErrorString(e));
  return STP_OK;
}

extern "C" int stp_selu_backward_bias(float* grad, const float* out, int64_t rows, int32_t H, float* d_bias,
                                      float* scratch, void* stream) {
  if (rows < 0 || H <= 0 || (H & 3) || H > 4 * kSeluThreads || !d_bias || !scratch ||
      (rows > 0 && (!grad || !out)) || (reinterpret_cast<uintptr_t>(grad) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return stp::fail(STP_EINVAL, "stp_selu_backward_bias: bad arguments");
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int rpar = kSeluThreads / (H / 4) > 0 ? kSeluThreads / (H / 4) : 1;
  // rows per block: a multiple of the rows in flight, at most kSeluBlocks blocks
  long long rpb = (rows + kSeluBlocks - 1) / kSeluBlocks;
  rpb = (rpb + rpar - 1) / rpar * rpar;
  const int nblk = rows > 0 ? int((rows + rpb - 1) / rpb) : 0;
  if (nblk > 0) {
    k_selu_bwd_bias<<<nblk, kSeluThreads, size_t(rpar) * H * sizeof(float), st>>>(grad, out, rows, H, rpb, scratch);
    k_colsum_finish<<<(H + 31) / 32, 256, 0, st>>>(scratch, nblk, H, d_bias);
  } else {
    cudaMemsetAsync(d_bias, 0, size_t(H) * sizeof(float), st);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_selu_bwd_bias: ") + cudaGetErrorString(e));
  return STP_OK;
}

extern "C" int stp_ppo_surrogate(const float* mu, const float* log_std, const float* value, const float* actions,
                                 const float* old_logp, const float* advantages, const float* returns,
                                 const int64_t* idx, int32_t B, int32_t A, const double* adv_stats, float clip,
                                 float vf_coef, float* d_mu, float* d_value, float* d_log_std, float* d_mu_bias,
                                 float* d_value_bias, float* loss, float* bad, double* scratch, void* stream) {
  if (B < 0 || A <= 0 || A > kPpoMaxA || !log_std || !d_log_std || !loss || !scratch ||
      (B > 0 && (!mu || !value || !actions || !old_logp || !advantages || !returns || !d_mu || !d_value)))
    return stp::fail(STP_EINVAL, "stp_ppo_surrogate: bad arguments");
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nblk = (B + kPpoThreads - 1) / kPpoThreads;
  if (nblk > 0)
    k_ppo_head<<<nblk, kPpoThreads, 0, st>>>(mu, log_std, value, actions, old_logp, advantages, returns, idx, B, A,
                                             adv_stats, clip, vf_coef, d_mu, d_value, scratch);
  k_ppo_finish<<<2 * A + 2, 256, 0, st>>>(scratch, nblk, A, B > 0 ? B : 1, vf_coef, d_log_std, d_mu_bias,
                                          d_value_bias, loss, bad);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_ppo_head: ") + cudaGetErrorString(e));
  return STP_OK;
}

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
