// K4: rollout policy forward on the 5th-generation tensor cores.
//
// SPEC.md:366-409 (SELU MLP, Gaussian policy), :446-454 (observation
// whitening), Table 4 (Humanoid [256, 128, 64], Ant [128, 64, 32]).
//
// Swapped operands (the small-batch GEMM form): each layer computes
// D^T = W X^T, so the hidden units run along the UMMA M = 128 dimension
// (a 256-wide layer is two M blocks) and the environments along N.  A CTA owns
// NT = 16 / 32 / 64 environments of one net (blockIdx.y: 0 policy, 1 value),
// so a 4096-env forward is 128 CTAs on the 148 SMs instead of 64 CTAs of 128
// envs, and every epilogue thread handles one hidden unit x 16 environments
// (tcgen05.ld 32x32b: TMEM lane = hidden unit):
//   obs tile (fp32, TMA bulk copy) -> whiten + clip(+-10) -> bf16 B operand
//   -> per layer tcgen05.mma (W: bf16 K-major A operand from smem, X^T: bf16
//      MN-major B operand, fp32 accumulator in TMEM)
//   -> epilogue: bias + SELU -> bf16 -> the next layer's B operand (16-byte
//      stores of 8 consecutive environments, conflict-free)
//   -> last layer: mean (+ log_std, counter-based Gaussian sample, log-prob)
//      or value.
// Weights (packed bf16 [K/8][N_out][8], the K-major core-matrix layout) are
// staged into smem with TMA bulk copies (cp.async.bulk) completing on an
// mbarrier; nets whose weights do not fit next to the operands (the 241-wide
// terrain observation) stream each layer's weights in contiguous K-block
// chunks through one buffer, every chunk accumulating into the same TMEM
// accumulator.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "stampede_sim.h"
#include "stp_error.h"
#include "stp_rng.h"

namespace {

constexpr int kM = 128;        // UMMA M: hidden units per M block (TMEM lanes)
constexpr int kThreads = 512;  // 16 warps: warps w, w+4, w+8, w+12 share TMEM lanes 32(w%4).. (units round-robin)
constexpr int kMaxNT = 64;     // environments per CTA (UMMA N)
constexpr float kSeluL = 1.0507009873554805f, kSeluA = 1.6732632423543772f;

struct MlpDims {
  int k[4];  // padded input width of layer l (multiple of 16)
  int n[4];  // padded output width of layer l (multiple of 16)
  int out;   // real output width of the last layer
  int kb_chunk[4];  // streaming mode: 8-wide K blocks per weight chunk (even)
};

struct NetPtrs {
  const __nv_bfloat16* w[4];  // packed [k/8][n][8] bf16
  const float* bias[4];       // padded to n
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, SWIZZLE_NONE canonical layouts
// (cute/arch/mma_sm100_desc.hpp SmemDescriptor); core matrix = 8 x 16 B
// contiguous.  K-major (weights, [k/8][m][8]): LBO = stride between
// K-adjacent core matrices (m * 16 B), SBO = stride between 8-row groups
// (128 B).  MN-major (activations X^T, [n/8][k][8 envs]): LBO = stride between
// K-adjacent core matrices (128 B), SBO = stride between 8-environment groups
// (k * 16 B) (checked on B200 against the torch reference, tests/test_gpu_policy.py).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;  // version = 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor kind::f16: bf16 x bf16 -> f32, A K-major, B
// MN-major (cute/arch/mma_sm100_desc.hpp InstrDescriptor: b_major bit 16).
__device__ __forceinline__ uint32_t umma_idesc(int m, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format = F32
  d |= 1u << 7;                    // a_format = BF16
  d |= 1u << 10;                   // b_format = BF16
  d |= 1u << 16;                   // b_major = MN (environments contiguous)
  d |= uint32_t(n >> 3) << 17;     // n_dim
  d |= uint32_t(m >> 4) << 24;     // m_dim
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
// 1-D TMA bulk copy global -> shared, completing tx bytes on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// programmatic dependent launch (griddepcontrol): wait for the preceding
// grid's completion and memory; let the next grid launch
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// one lane of a converged warp (elect.sync): the MMA issue region, so that
// ptxas knows a single thread issues and keeps the descriptors in uniform
// registers (a `tid == 0` region makes it wrap every tcgen05.mma in an
// ELECT / R2UR.BROADCAST loop over the possibly active threads)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
      : "+r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"(
                   reinterpret_cast<uint64_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// 16 fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// SELU with the fast exponential: the result is rounded to bf16 for the next
// layer anyway (8 significant bits), so __expf's ~2 ulp fp32 error is invisible.
// Branch-free: the exponential of min(x, 0) is computed for every lane and
// selected, so a warp never splits on the sign.
// __expf(y) is ex2.approx(y * log2 e); the flush-to-zero form skips the
// denormal-range fixups, which only differ for y < -87 where SELU's negative
// branch rounds to -lambda*alpha either way.
#ifndef STP_K4_SELU
#define STP_K4_SELU 0
#endif
__device__ __forceinline__ float selu(float x) {
#if STP_K4_SELU == 2  // timing experiment only: identity
  return x;
#else
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fminf(x, 0.f) * 1.4426950408889634f));
  const float neg = kSeluL * kSeluA * (e - 1.f);
  return x > 0.f ? kSeluL * x : neg;
#endif
}

// bias + SELU on a thread's 16 accumulator columns.  STP_K4_SELU == 1
// (experiment): the exponentials as ex2.approx.f16x2, two per MUFU op.
__device__ __forceinline__ void selu16(float (&v)[16], float bias) {
#if STP_K4_SELU == 1
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float a = v[2 * i] + bias, b = v[2 * i + 1] + bias;
    const __half2 t = __floats2half2_rn(fminf(a, 0.f) * 1.4426950408889634f, fminf(b, 0.f) * 1.4426950408889634f);
    uint32_t e2;
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(e2) : "r"(*reinterpret_cast<const uint32_t*>(&t)));
    const float2 e = __half22float2(*reinterpret_cast<const __half2*>(&e2));
    v[2 * i] = a > 0.f ? kSeluL * a : kSeluL * kSeluA * (e.x - 1.f);
    v[2 * i + 1] = b > 0.f ? kSeluL * b : kSeluL * kSeluA * (e.y - 1.f);
  }
#else
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = selu(v[i] + bias);
#endif
}


// 8 bf16 = one 16-byte chunk of the MN-major operand X^T: row k (hidden unit
// or observation column), environments n0..n0+7 (n0 % 8 == 0).
__device__ __forceinline__ void st_xt(__nv_bfloat16* buf, int kpad, int k, int n0, const float* x8) {
  __nv_bfloat162 p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(x8[2 * i], x8[2 * i + 1]);
  *reinterpret_cast<uint4*>(buf + (size_t(n0 >> 3) * kpad + k) * 8) = *reinterpret_cast<uint4*>(p);
}

// Experiment-only phase timestamps (tools/exp/k4_phases.py builds with
// -DSTP_K4_PHASES): thread 0 of each CTA records %globaltimer (phase 0) and
// the SM clock (every phase) at phase ends.
#ifdef STP_K4_PHASES
constexpr int kPhases = 32;
__device__ unsigned long long g_k4_phase[1024 * kPhases];
__device__ __forceinline__ void phase(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    if (i == 0) {
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      g_k4_phase[(blockIdx.y * gridDim.x + blockIdx.x) * kPhases + 31] = t;
    }
    t = clock64();
    g_k4_phase[(blockIdx.y * gridDim.x + blockIdx.x) * kPhases + i] = t;
  }
}
#else
__device__ __forceinline__ void phase(int) {}
#endif

struct Smem {
  uint64_t bar_obs;    // observation tile landed (TMA path)
  uint64_t bar_w;      // weights landed
  uint64_t bar_mma;    // layer accumulator ready
  uint64_t bar_chunk;  // streaming mode: a chunk's MMAs done (weight buffer free)
  uint32_t tmem;
  alignas(16) float wmean[256];  // whitening: per-column mean and std (TMA bulk destinations: 16-byte aligned)
  alignas(16) float winv[256];
  uint64_t streams[kMaxNT];  // policy noise stream per environment of the tile
  float sdv[256];            // exp(log_std) per action
  float lsd[256];            // log_std per action
  alignas(16) float bias[4][256];  // the net's biases (TMA bulk copies, padded widths)
};
constexpr int kHeader = 9216;  // Smem, rounded to the operand alignment
static_assert(sizeof(Smem) <= kHeader, "Smem header");
constexpr int kTmemCols = 2 * kMaxNT;  // two M blocks x NT accumulator columns

// One 4-layer net over the CTA's NT environments; B operand of layer 0 already
// in xb0.  Returns with the last layer's accumulator (rows = outputs) in TMEM.
__device__ __forceinline__ void run_net(const MlpDims& D, const NetPtrs& P, __nv_bfloat16* wbase, __nv_bfloat16* xb0,
                        __nv_bfloat16* xb1, Smem* sh, uint32_t& wphase, uint32_t& mphase, int tid, bool stream,
                        int NT) {
  const int warp = tid >> 5, lane = tid & 31;
  const int sp = warp & 3;   // TMEM subpartition: lanes 32 sp ..
  const int wq = warp >> 2;  // 0..3: unit phase within the subpartition
  if (!stream) {
    mbar_wait(&sh->bar_w, wphase);
    wphase ^= 1;
  }
  phase(3);
  uint32_t cphase = 0;  // streaming mode, issuing thread only
  __nv_bfloat16* x_in = xb0;
  __nv_bfloat16* x_out = xb1;
  const uint32_t idesc = umma_idesc(kM, NT);
  uint32_t woff = 0;  // byte offset of layer l's resident weights
  for (int l = 0; l < 4; ++l) {
    const int mblocks = (D.n[l] + kM - 1) / kM;
    fence_async_smem();  // generic-proxy operand writes -> visible to the tensor core
    __syncthreads();
    phase(13 + l);
    if (warp == 0 && elect_one()) {
      tc_after_sync();
      const uint32_t xa = smem_u32(x_in);
      const uint32_t xsbo = uint32_t(D.k[l]) * 16;  // 8-environment group stride of X^T
      const uint32_t wlbo = uint32_t(D.n[l]) * 16;  // K-group stride of W
      auto issue = [&](uint32_t w0, int ks0, int nks, int kg0) {
        // K steps [ks0, ks0 + nks) of 16 for every M block; kg0 = global K step
        // of ks0.  The descriptors are linear in the start address (bits 0-13,
        // address >> 4), so each step adds a constant
        const uint64_t db0 = umma_desc(xa + uint32_t(kg0) * 256, 128, xsbo);
        for (int mb = 0; mb < mblocks; ++mb) {
          uint64_t da = umma_desc(w0 + uint32_t(mb) * kM * 16, wlbo, 128), db = db0;
          for (int ks = 0; ks < nks; ++ks) {
            mma_bf16(sh->tmem + uint32_t(mb * NT), da, db, idesc, kg0 + ks > 0);
            da += uint64_t(2 * wlbo) >> 4;
            db += 256 >> 4;
          }
        }
      };
      if (!stream) {
        issue(smem_u32(wbase) + woff, 0, D.k[l] / 16, 0);
      } else {
        // K blocks [kb0, kb0 + nb) of the packed [k/8][n][8] weight are one
        // contiguous range: stage it, accumulate its MMAs, free the buffer
        const int kbt = D.k[l] / 8, kbc = D.kb_chunk[l];
        for (int kb0 = 0; kb0 < kbt; kb0 += kbc) {
          const int nb = min(kbc, kbt - kb0);
          const uint32_t bytes = uint32_t(nb) * 8 * D.n[l] * 2;
          mbar_expect_tx(&sh->bar_w, bytes);
          bulk_g2s(wbase, P.w[l] + size_t(kb0) * 8 * D.n[l], bytes, &sh->bar_w);
          mbar_wait(&sh->bar_w, wphase);
          wphase ^= 1;
          issue(smem_u32(wbase), 0, nb / 2, kb0 / 2);
          if (kb0 + nb < kbt) {
            umma_commit(&sh->bar_chunk);
            mbar_wait(&sh->bar_chunk, cphase);
            cphase ^= 1;
          }
        }
      }
      umma_commit(&sh->bar_mma);
      phase(17 + l);
    }
    woff += uint32_t(D.k[l]) * D.n[l] * 2;
    phase(21 + l);
    mbar_wait(&sh->bar_mma, mphase);
    mphase ^= 1;
    tc_after_sync();
    phase(4 + 2 * l);
    if (l == 3) break;
    // epilogue: units (M block, 16-environment chunk) of this subpartition
    // round-robin over its 4 warps; lane = hidden unit h, 16 environments
    const int nch = NT / 16, units = mblocks * nch;
    const int kout = D.k[l + 1];  // = D.n[l] (padded width): K rows of the next operand
    for (int u = wq; u < units; u += 4) {
      const int mb = u / nch, ch = u - mb * nch;
      const int h = mb * kM + sp * 32 + lane;
      if (mb * kM + sp * 32 >= D.n[l]) continue;  // warp-uniform: no valid unit in this subpartition
      const float bias = h < D.n[l] ? sh->bias[l][h] : 0.f;
      float v[16];
      tmem_ld16(sh->tmem + (uint32_t(sp * 32) << 16) + uint32_t(mb * NT + ch * 16), v);
      if (l == 0 && u == wq) phase(28);
      selu16(v, bias);
      if (h < kout) {
        st_xt(x_out, kout, h, ch * 16, v);
        st_xt(x_out, kout, h, ch * 16 + 8, v + 8);
      }
    }
    tc_before_sync();
    phase(5 + 2 * l);
    __nv_bfloat16* t = x_in;
    x_in = x_out;
    x_out = t;
  }
}

// K4 kernel: blockIdx.x = NT-environment tile, blockIdx.y = net (0 policy, 1 value).
__global__ void __launch_bounds__(kThreads, 1)
    k_policy_mlp(const float* __restrict__ obs, int n_envs, int obs_dim, const float* __restrict__ mean,
                 const float* __restrict__ stdv, const __grid_constant__ MlpDims Dpi,
                 const __grid_constant__ NetPtrs Ppi, const __grid_constant__ MlpDims Dv,
                 const __grid_constant__ NetPtrs Pv,
                 const float* __restrict__ log_std, uint64_t seed, uint64_t step, long long env_offset,
                 float* __restrict__ mu_out, float* __restrict__ act_out, float* __restrict__ logp_out,
                 float* __restrict__ v_out, int x0_elems, int x1_elems, int wbuf_elems, int NT, int eps_elems) {
  extern __shared__ __align__(1024) unsigned char smem[];
  Smem* sh = reinterpret_cast<Smem*>(smem);
  phase(0);
  float* eps = reinterpret_cast<float*>(smem + kHeader);  // policy noise [env][out]
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(smem + kHeader + size_t(eps_elems) * 4);
  // operand ping-pong: xb0 holds layer 0/2 inputs, xb1 layer 1/3 inputs
  __nv_bfloat16* xb0 = base;
  __nv_bfloat16* xb1 = base + x0_elems;
  __nv_bfloat16* wbase = base + x0_elems + x1_elems;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const bool value_net = blockIdx.y == 1;
  const MlpDims& D = value_net ? Dv : Dpi;
  const NetPtrs& P = value_net ? Pv : Ppi;

  // The tile's observation rows are one contiguous block of global memory,
  // staged into the (still unused) layer-1 operand buffer by one TMA bulk copy
  // when its size and address allow (issued first, then the 4 weight blobs, all
  // completing on mbarriers), else by coalesced loads.
  float* stage = reinterpret_cast<float*>(xb1);
  const int tile0 = blockIdx.x * NT;
  const int rows = min(NT, n_envs - tile0);
  const float* src = obs + size_t(tile0) * obs_dim;
  const uint32_t tile_bytes = uint32_t(rows) * uint32_t(obs_dim) * 4u;
  const bool tma_obs = (tile_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  // the whitening statistics by TMA too when they are 16-byte multiples
  const uint32_t stat_bytes = uint32_t(obs_dim) * 4u;
  const bool tma_stat = tma_obs && (stat_bytes & 15) == 0 &&
                        ((reinterpret_cast<uintptr_t>(mean) | reinterpret_cast<uintptr_t>(stdv)) & 15) == 0;
  const bool stream = wbuf_elems > 0;
  // Programmatic dependent launch: everything up to griddep_wait() reads only
  // the network parameters (never written by a kernel that triggers early: the
  // step kernel and K4 itself), so it overlaps the tail of the preceding grid;
  // the observations, the whitening statistics and every output come after it.
  if (warp == 1 && elect_one()) {  // barriers + weight TMA (warp 0 allocates TMEM meanwhile)
    mbar_init(&sh->bar_obs, 1);
    mbar_init(&sh->bar_w, 1);
    mbar_init(&sh->bar_mma, 1);
    mbar_init(&sh->bar_chunk, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (!stream) {  // weights + biases (16-byte multiples: padded to 16 outputs) on bar_w
      uint32_t bytes = 0;
      for (int l = 0; l < 4; ++l) bytes += uint32_t(D.k[l]) * D.n[l] * 2 + uint32_t(D.n[l]) * 4;
      mbar_expect_tx(&sh->bar_w, bytes);
      for (int l = 0; l < 4; ++l) bulk_g2s(sh->bias[l], P.bias[l], uint32_t(D.n[l]) * 4, &sh->bar_w);
      for (int l = 0, off = 0; l < 4; off += D.k[l] * D.n[l], ++l)
        bulk_g2s(wbase + off, P.w[l], uint32_t(D.k[l]) * D.n[l] * 2, &sh->bar_w);
    }
  }
  if (warp == 0) {  // TMEM: two M blocks x NT columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&sh->tmem)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (!value_net && act_out) {
    for (int r = tid; r < rows; r += kThreads)
      sh->streams[r] = stp_derive_seed(seed, 6 /* policy noise */, (uint64_t(env_offset + tile0 + r) << 32) |
                                                                       uint32_t(step));
  }
  // policy noise [env][out] into shared memory, before the dependency wait
  // (it reads only the seed / step / env ids and log_std): Box-Muller pairs
  // (both the cosine and the sine branch) on two 24-bit counter-based
  // uniforms of one 64-bit hash per pair of actions, fast log / sincos on
  // [-pi, pi) (|err| ~1e-6)
  if (!value_net && act_out) {
    __syncthreads();  // streams
    for (int c = tid; c < D.out; c += kThreads) {
      const float ls = log_std[c];
      sh->lsd[c] = ls;
      sh->sdv[c] = expf(ls);
    }
    const int npair = (D.out + 1) / 2;
    for (int i = tid; i < rows * npair; i += kThreads) {
      const int r = i / npair, q = i - r * npair;
      const uint64_t z = stp_mix64(sh->streams[r] + uint64_t(q));  // bits 40-63: u1, 16-39: u2
      const float u1 = fmaxf(float(z >> 40) * (1.f / 16777216.f), 1e-7f);
      const float u2 = float((z >> 16) & 0xffffffu) * (1.f / 16777216.f);
      const float rad = sqrtf(-2.f * __logf(u1));
      float sn, cs;
      __sincosf(6.2831853071795865f * u2 - 3.14159265358979323f, &sn, &cs);
      float* e = eps + r * D.out + 2 * q;
      e[0] = rad * cs;
      if (2 * q + 1 < D.out) e[1] = rad * sn;
    }
  }
  griddep_wait();
  griddep_launch_dependents();
  if (warp == 1 && elect_one()) {  // observation tile + statistics (+ streaming mode: biases) on bar_obs
    uint32_t bias_bytes = 0;
    if (stream)
      for (int l = 0; l < 4; ++l) bias_bytes += uint32_t(D.n[l]) * 4;
    mbar_expect_tx(&sh->bar_obs, bias_bytes + (tma_obs ? tile_bytes : 0) + (tma_stat ? 2 * stat_bytes : 0));
    if (stream)
      for (int l = 0; l < 4; ++l) bulk_g2s(sh->bias[l], P.bias[l], uint32_t(D.n[l]) * 4, &sh->bar_obs);
    if (tma_obs) {
      bulk_g2s(stage, src, tile_bytes, &sh->bar_obs);
      if (tma_stat) {
        bulk_g2s(sh->wmean, mean, stat_bytes, &sh->bar_obs);
        bulk_g2s(sh->winv, stdv, stat_bytes, &sh->bar_obs);  // the standard deviations themselves
      }
    }
  }
  if (!tma_stat)
    for (int c = tid; c < obs_dim; c += kThreads) {
      sh->wmean[c] = __ldg(mean + c);
      sh->winv[c] = __ldg(stdv + c);
    }
  if (!tma_obs) {
    const int nf = rows * obs_dim;
    for (int i = tid; i < nf; i += kThreads) stage[i] = __ldg(src + i);
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  phase(1);
  // whitened, clipped observations (RunningStat) -> X^T:
  // one (observation column k, 8-environment group) chunk per thread and pass
  {
    mbar_wait(&sh->bar_obs, 0);
    for (int c = tid; c < obs_dim; c += kThreads) sh->winv[c] = 1.f / sh->winv[c];
    __syncthreads();
    phase(11);
    const int kpad = D.k[0], ngr = NT / 8;
    for (int u = tid; u < kpad * ngr; u += kThreads) {
      const int k = u % kpad, g = u / kpad;
      // branch-free: padded columns / rows read a clamped in-tile address and
      // are zeroed by the select, so the 8 loads issue back to back
      const bool kin = k < obs_dim;
      const int kc = kin ? k : 0;
      const float mk = sh->wmean[kc], ik = sh->winv[kc];
      float x8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = g * 8 + i;
        const bool in = kin && r < rows;
        const float x = (stage[(in ? r : 0) * obs_dim + kc] - mk) * ik;
        x8[i] = in ? fminf(fmaxf(x, -10.f), 10.f) : 0.f;
      }
      st_xt(xb0, kpad, k, g * 8, x8);
    }
  }
  phase(2);
  uint32_t wphase = 0, mphase = 0;
  run_net(D, P, wbase, xb0, xb1, sh, wphase, mphase, tid, stream, NT);
  // last layer: TMEM lane = output, columns = environments
  const int sp = warp & 3, wq = warp >> 2, nch = NT / 16;
  if (!value_net) {
    // policy head: the mean tile [env][out] through shared
    // memory (the operand buffers are free once the last MMA completed), then
    // 8 threads per environment write its mean / action row (8 consecutive
    // columns per pass) and sum its log-prob terms
    const int out = D.out;
    float* tile = reinterpret_cast<float*>(base);
    for (int u = wq; u < nch * ((out + 31) / 32); u += 4) {
      const int ch = u % nch, blk = u / nch;
      if (blk != sp) continue;  // outputs 32 sp .. of M block 0 live in subpartition sp
      float v[16];
      tmem_ld16(sh->tmem + (uint32_t(sp * 32) << 16) + uint32_t(ch * 16), v);
      const int c = sp * 32 + lane;
      if (c < out) {
        const float bias = sh->bias[3][c];
#pragma unroll
        for (int i = 0; i < 16; ++i) tile[(ch * 16 + i) * out + c] = v[i] + bias;
      }
    }
    phase(25);
    __syncthreads();
    phase(26);
    // 8 threads per environment: columns j, j + 8, ...; the log-prob terms
    // summed in that order, then a fixed shuffle tree (deterministic)
    static_assert(kThreads >= 8 * kMaxNT, "8 threads per environment");
    const int r = tid >> 3, j = tid & 7;
    float lp = 0.f;
    if (r < rows)
      for (int c = j; c < out; c += 8) {
        const float m = tile[r * out + c];
        const size_t g = (size_t(tile0) + r) * out + c;
        mu_out[g] = m;
        if (act_out) {
          const float ep = eps[r * out + c];  // drawn in the prologue (same [env][out] indexing)
          act_out[g] = m + sh->sdv[c] * ep;
          lp += -0.5f * ep * ep - sh->lsd[c] - 0.91893853320467274f;
        }
      }
    phase(27);
    if (logp_out) {
      lp += __shfl_xor_sync(0xffffffffu, lp, 4);
      lp += __shfl_xor_sync(0xffffffffu, lp, 2);
      lp += __shfl_xor_sync(0xffffffffu, lp, 1);
      if (j == 0 && r < rows) logp_out[tile0 + r] = lp;
    }
  } else if (sp == 0 && wq < nch) {
    float v[16];
    tmem_ld16(sh->tmem + uint32_t(wq * 16), v);
    if (lane == 0) {
      const float bias = sh->bias[3][0];
      for (int i = 0; i < 16; ++i)
        if (wq * 16 + i < rows) v_out[tile0 + wq * 16 + i] = v[i] + bias;
    }
  }
  tc_before_sync();
  __syncthreads();
  phase(12);
  if (warp == 0) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(sh->tmem), "n"(kTmemCols));
  }
}

}  // namespace

#ifdef STP_K4_PHASES
extern "C" int stp_k4_phases(unsigned long long* out, int n) {
  return int(cudaMemcpyFromSymbol(out, g_k4_phase, sizeof(unsigned long long) * size_t(n)));
}
#endif

extern "C" int stp_policy_forward(const float* obs, int32_t n_envs, int32_t obs_dim, const float* obs_mean,
                                  const float* obs_std, const int32_t* dims_pi, const void* const* w_pi,
                                  const float* const* b_pi, const int32_t* dims_v, const void* const* w_v,
                                  const float* const* b_v, const float* log_std, uint64_t seed, uint64_t step,
                                  int64_t env_offset, float* mean_out, float* action_out, float* logp_out,
                                  float* value_out, void* stream) {
  if (!obs || n_envs <= 0 || !dims_pi || !w_pi || !b_pi || !mean_out || !obs_mean || !obs_std)
    return stp::fail(STP_EINVAL, "stp_policy_forward: bad arguments");
  MlpDims Dpi{}, Dv{};
  NetPtrs Ppi{}, Pv{};
  // dims: [in, h1, h2, h3, out] real sizes
  auto fill = [](const int32_t* d, MlpDims& D) {
    auto pad16 = [](int x) { return (x + 15) / 16 * 16; };
    for (int l = 0; l < 4; ++l) {
      D.k[l] = pad16(d[l]);
      D.n[l] = pad16(d[l + 1]);
    }
    D.out = d[4];
  };
  fill(dims_pi, Dpi);
  for (int l = 0; l < 4; ++l) {
    Ppi.w[l] = static_cast<const __nv_bfloat16*>(w_pi[l]);
    Ppi.bias[l] = b_pi[l];
  }
  if (value_out) {
    if (!dims_v || !w_v || !b_v) return stp::fail(STP_EINVAL, "stp_policy_forward: value net missing");
    fill(dims_v, Dv);
    for (int l = 0; l < 4; ++l) {
      Pv.w[l] = static_cast<const __nv_bfloat16*>(w_v[l]);
      Pv.bias[l] = b_v[l];
    }
  }
  auto aligned = [](const NetPtrs& P) {  // TMA bulk sources, float4 bias loads
    for (int l = 0; l < 4; ++l)
      if ((reinterpret_cast<uintptr_t>(P.w[l]) | reinterpret_cast<uintptr_t>(P.bias[l])) & 15) return false;
    return true;
  };
  if (!aligned(Ppi) || (value_out && !aligned(Pv)))
    return stp::fail(STP_EINVAL, "stp_policy_forward: weights and biases must be 16-byte aligned");
  auto check = [](const MlpDims& D) {
    for (int l = 0; l < 4; ++l)
      if (D.n[l] > 256 || D.k[l] > 256) return false;  // one UMMA N per layer, 256 TMEM columns
    return true;
  };
  if (!check(Dpi) || (value_out && !check(Dv)))
    return stp::fail(STP_EINVAL, "stp_policy_forward: layer widths must be <= 256");
  if (Dpi.k[0] != (obs_dim + 15) / 16 * 16) return stp::fail(STP_EINVAL, "stp_policy_forward: obs_dim mismatch");
  auto welems = [](const MlpDims& D) {
    int s = 0;
    for (int l = 0; l < 4; ++l) s += D.k[l] * D.n[l];
    return s;
  };
  const int wmax = value_out ? (welems(Dpi) > welems(Dv) ? welems(Dpi) : welems(Dv)) : welems(Dpi);
  auto mx = [](int a, int b) { return a > b ? a : b; };
  if (Dpi.out > kM) return stp::fail(STP_EINVAL, "stp_policy_forward: at most 128 actions");
  // environments per CTA (UMMA N): the largest of 64 / 32 / 16 that still
  // gives ~one CTA per SM over both nets
  const int nets = value_out ? 2 : 1;
  const int NT = (n_envs + 63) / 64 * nets >= 120 ? 64 : (n_envs + 31) / 32 * nets >= 120 ? 32 : 16;
  int c0 = mx(Dpi.k[0], Dpi.k[2]), c1 = mx(Dpi.k[1], Dpi.k[3]);
  if (value_out) {
    c0 = mx(c0, mx(Dv.k[0], Dv.k[2]));
    c1 = mx(c1, mx(Dv.k[1], Dv.k[3]));
  }
  const int x0 = NT * c0;
  const int x1 = mx(NT * c1, (NT * obs_dim * 4 + 1) / 2);  // X^T operands; x1 also stages the fp32 obs tile
  const size_t kSmemMax = 227 * 1024;
  // + one M block of K-major rows (2 KB): a layer narrower than 128 outputs is
  // read as a full M = 128 block, the extra rows' results are never used
  const size_t kOverRead = size_t(kM) * 16;
  const int eps_elems = action_out ? ((NT * Dpi.out + 3) / 4 * 4) : 0;  // noise tile, 16-byte multiple
  const size_t base = kHeader + size_t(eps_elems) * 4 + size_t(x0 + x1) * 2;
  size_t smem = base + size_t(wmax) * 2 + kOverRead;
  int wbuf = 0;  // 0: all weights resident
  for (MlpDims* D : {&Dpi, &Dv})
    for (int l = 0; l < 4; ++l) D->kb_chunk[l] = D->k[l] / 8;
  if (smem > kSmemMax) {
    // stream: one weight buffer filling the rest of shared memory
    wbuf = int((kSmemMax - base - kOverRead) / 2) / 128 * 128;
    for (MlpDims* D : {&Dpi, &Dv}) {
      if (D == &Dv && !value_out) continue;
      for (int l = 0; l < 4; ++l) {
        D->kb_chunk[l] = (wbuf / (8 * D->n[l])) & ~1;
        if (D->kb_chunk[l] < 2)
          return stp::fail(STP_EINVAL, "stp_policy_forward: network too large for shared memory");
      }
    }
    smem = base + size_t(wbuf) * 2 + kOverRead;
  }
  static size_t configured[64] = {};  // per device (the attribute is)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || smem > configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_policy_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_policy_mlp attr: ") + cudaGetErrorString(e));
    if (dev >= 0 && dev < 64) configured[dev] = smem;
  }
  // programmatic dependent launch: the prologue (barriers, TMEM, weight TMA)
  // overlaps the tail of the preceding grid when that grid triggers early
  // (the step kernel, K4); STP_PDL=0 launches plainly (A/B timing)
  static const bool pdl = [] {
    const char* v = getenv("STP_PDL");
    return !(v && v[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n_envs + NT - 1) / NT, nets);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_policy_mlp, obs, n_envs, obs_dim, obs_mean, obs_std, Dpi, Ppi, Dv, Pv,
                                     log_std, seed, step, (long long)env_offset, mean_out, action_out, logp_out,
                                     value_out, x0, x1, wbuf, NT, eps_elems);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_policy_mlp: ") + cudaGetErrorString(e));
  return STP_OK;
}
