// K4: rollout policy forward on the 5th-generation tensor cores.
//
// SPEC.md:366-409 (SELU MLP, Gaussian policy), :446-454 (observation
// whitening), Table 4 (Humanoid [256, 128, 64], Ant [128, 64, 32]).
// One CTA = 128 environments = one M=128 tcgen05 tile:
//   obs (fp32, HBM) -> whiten + clip(+-10) -> bf16 operand in smem
//   -> 4 x tcgen05.mma (bf16 x bf16 -> fp32 accumulator in TMEM)
//   -> tcgen05.ld epilogue: bias + SELU -> bf16 -> next layer's smem operand
//   -> last layer: mean (+ log_std, counter-based Gaussian sample, log-prob)
// for the policy net, then the same chain for the value net.  Weights (packed
// bf16, K-major 8x16B core-matrix layout) are staged into smem with TMA bulk
// copies (cp.async.bulk) completing on an mbarrier; nets whose weights do not
// fit next to the operands (e.g. the 241-wide terrain observation) stream each
// layer's weights in contiguous K-block chunks through one buffer, every chunk
// accumulating into the same TMEM accumulator.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "stampede_sim.h"
#include "stp_error.h"
#include "stp_rng.h"

namespace {

constexpr int kM = 128;        // rows (envs) per CTA = UMMA M
constexpr int kThreads = 512;  // 16 warps: warps w, w+4, w+8, w+12 share TMEM lanes 32(w%4).. (16-column chunks round-robin)
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

// UMMA shared-memory descriptor, SWIZZLE_NONE K-major canonical layout
// (cute/arch/mma_sm100_desc.hpp SmemDescriptor): core matrix = 8 rows x 16 B
// contiguous; LBO = byte stride between K-adjacent core matrices, SBO = byte
// stride between 8-row groups.  Our packing [k/8][rows][8] gives SBO = 128 B
// and LBO = rows * 16 B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;  // version = 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor kind::f16: bf16 x bf16 -> f32, both K-major
// (cute/arch/mma_sm100_desc.hpp InstrDescriptor).
__device__ __forceinline__ uint32_t umma_idesc(int m, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format = F32
  d |= 1u << 7;                    // a_format = BF16
  d |= 1u << 10;                   // b_format = BF16
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
__device__ __forceinline__ float selu(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fminf(x, 0.f) * 1.4426950408889634f));
  const float neg = kSeluL * kSeluA * (e - 1.f);
  return x > 0.f ? kSeluL * x : neg;
}

// Write 8 bf16 (16 B) of row `row`, K-chunk `kc` into a [k/8][128][8] operand.
__device__ __forceinline__ int quarter_of(int warp) { return warp >> 2; }

__device__ __forceinline__ void st_chunk(__nv_bfloat16* buf, int kc, int row, const float* x8) {
  __nv_bfloat162 p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(x8[2 * i], x8[2 * i + 1]);
  *reinterpret_cast<uint4*>(buf + (size_t(kc) * kM + row) * 8) = *reinterpret_cast<uint4*>(p);
}

// Experiment-only phase timestamps (tools/exp/k4_phases.py builds with
// -DSTP_K4_PHASES): thread 0 of each CTA records %globaltimer at phase ends.
#ifdef STP_K4_PHASES
constexpr int kPhases = 16;
__device__ unsigned long long g_k4_phase[512 * kPhases];
__device__ __forceinline__ void phase(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
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
  float wmean[256];  // whitening: per-column mean and 1 / std of the observation
  float winv[256];
};
constexpr int kHeader = 3072;  // Smem, rounded to the operand alignment
static_assert(sizeof(Smem) <= kHeader, "Smem header");

// One 4-layer net over the CTA's 128 rows; A operand of layer 0 already in abuf0.
// Returns with the final accumulator (n[3] columns) in TMEM.
__device__ void run_net(const MlpDims& D, const NetPtrs& P, __nv_bfloat16* wsm[4], __nv_bfloat16* abuf0,
                        __nv_bfloat16* abuf1, Smem* sh, uint32_t& wphase, uint32_t& mphase, int tid,
                        bool stream) {
  const int warp = tid >> 5;
  const int row = (warp & 3) * 32 + (tid & 31);  // TMEM lane = tile row
  const int quarter = quarter_of(warp);          // epilogue chunk phase (0..3)
  // resident mode: the 4 weight blobs were issued by the caller
  if (!stream) {
    mbar_wait(&sh->bar_w, wphase);
    wphase ^= 1;
  }
  phase(3);
  uint32_t cphase = 0;  // streaming mode, issuing thread only
  __nv_bfloat16* a_in = abuf0;
  __nv_bfloat16* a_out = abuf1;
  for (int l = 0; l < 4; ++l) {
    fence_async_smem();  // generic-proxy operand writes -> visible to the tensor core
    __syncthreads();
    if (tid == 0) {
      tc_after_sync();
      const uint32_t idesc = umma_idesc(kM, D.n[l]);
      const uint32_t a0 = smem_u32(a_in), b0 = smem_u32(wsm[stream ? 0 : l]);
      if (!stream) {
        for (int ks = 0; ks < D.k[l] / 16; ++ks) {
          // K step of 16 = two 8-element core-matrix columns
          const uint64_t da = umma_desc(a0 + uint32_t(ks) * 2 * kM * 16, kM * 16, 128);
          const uint64_t db = umma_desc(b0 + uint32_t(ks) * 2 * D.n[l] * 16, uint32_t(D.n[l]) * 16, 128);
          mma_bf16(sh->tmem, da, db, idesc, ks > 0);
        }
      } else {
        // K blocks [kb0, kb0 + nb) of the packed [k/8][n][8] weight are one
        // contiguous range: stage it, accumulate its MMAs, free the buffer
        const int kbt = D.k[l] / 8, kbc = D.kb_chunk[l];
        for (int kb0 = 0; kb0 < kbt; kb0 += kbc) {
          const int nb = min(kbc, kbt - kb0);
          const uint32_t bytes = uint32_t(nb) * 8 * D.n[l] * 2;
          mbar_expect_tx(&sh->bar_w, bytes);
          bulk_g2s(wsm[0], P.w[l] + size_t(kb0) * 8 * D.n[l], bytes, &sh->bar_w);
          mbar_wait(&sh->bar_w, wphase);
          wphase ^= 1;
          for (int ks = 0; ks < nb / 2; ++ks) {
            const int kg = kb0 / 2 + ks;  // global K step of 16
            const uint64_t da = umma_desc(a0 + uint32_t(kg) * 2 * kM * 16, kM * 16, 128);
            const uint64_t db = umma_desc(b0 + uint32_t(ks) * 2 * D.n[l] * 16, uint32_t(D.n[l]) * 16, 128);
            mma_bf16(sh->tmem, da, db, idesc, kg > 0);
          }
          if (kb0 + nb < kbt) {
            umma_commit(&sh->bar_chunk);
            mbar_wait(&sh->bar_chunk, cphase);
            cphase ^= 1;
          }
        }
      }
      umma_commit(&sh->bar_mma);
    }
    mbar_wait(&sh->bar_mma, mphase);
    mphase ^= 1;
    tc_after_sync();
    phase(4 + 2 * l);
    if (l == 3) break;
    // epilogue: bias + SELU -> bf16 -> next operand (this thread's row, every
    // 4th 16-column chunk)
    const uint32_t tbase = sh->tmem + (uint32_t((warp & 3) * 32) << 16);
    const int nch = D.n[l] / 16;
    for (int j = quarter; j < nch; j += 4) {
      // bias loads first: their latency overlaps the TMEM load's
      const float4* b4 = reinterpret_cast<const float4*>(P.bias[l] + 16 * j);
      float4 bq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) bq[q] = __ldg(b4 + q);
      float v[16];
      tmem_ld16(tbase + uint32_t(16 * j), v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 b = bq[q];
        v[4 * q] = selu(v[4 * q] + b.x);
        v[4 * q + 1] = selu(v[4 * q + 1] + b.y);
        v[4 * q + 2] = selu(v[4 * q + 2] + b.z);
        v[4 * q + 3] = selu(v[4 * q + 3] + b.w);
      }
      st_chunk(a_out, 2 * j, row, v);
      st_chunk(a_out, 2 * j + 1, row, v + 8);
    }
    tc_before_sync();
    phase(5 + 2 * l);
    __nv_bfloat16* t = a_in;
    a_in = a_out;
    a_out = t;
  }
}

// K4 kernel: blockIdx.x = 128-env tile, blockIdx.y = net (0 policy, 1 value).
__global__ void __launch_bounds__(kThreads, 1)
    k_policy_mlp(const float* __restrict__ obs, int n_envs, int obs_dim, const float* __restrict__ mean,
                 const float* __restrict__ stdv, const __grid_constant__ MlpDims Dpi,
                 const __grid_constant__ NetPtrs Ppi, const __grid_constant__ MlpDims Dv,
                 const __grid_constant__ NetPtrs Pv,
                 const float* __restrict__ log_std, uint64_t seed, uint64_t step, long long env_offset,
                 float* __restrict__ mu_out, float* __restrict__ act_out, float* __restrict__ logp_out,
                 float* __restrict__ v_out, int a0_elems, int a1_elems, int wbuf_elems) {
  extern __shared__ __align__(1024) unsigned char smem[];
  Smem* sh = reinterpret_cast<Smem*>(smem);
  phase(0);
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(smem + kHeader);
  // operand ping-pong: abuf0 holds layer 0/2 inputs, abuf1 layer 1/3 inputs
  __nv_bfloat16* abuf0 = base;
  __nv_bfloat16* abuf1 = base + a0_elems;
  __nv_bfloat16* wbase = base + a0_elems + a1_elems;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool value_net = blockIdx.y == 1;
  const MlpDims& D = value_net ? Dv : Dpi;
  const NetPtrs& P = value_net ? Pv : Ppi;
  const int lrow = (warp & 3) * 32 + (tid & 31);  // TMEM lane / tile row of this thread
  const int row = blockIdx.x * kM + lrow;

  __nv_bfloat16* wsm[4];
  int off = 0;
  for (int l = 0; l < 4; ++l) {
    wsm[l] = wbase + off;
    off += D.k[l] * D.n[l];
  }
  // whitened, clipped observation rows -> bf16 operand (RunningStat,
  // SPEC.md:446-454).  The tile's rows are one contiguous block of global
  // memory staged into the (still unused) layer-1 operand buffer: by one TMA
  // bulk copy when its size and address allow (issued first, then the 4 weight
  // blobs, all completing on mbarriers while the CTA waits for the first),
  // else by coalesced loads in row passes that fit the buffer.  Each
  // (row, 8-column chunk) is then whitened and written as one 16-byte chunk.
  float* stage = reinterpret_cast<float*>(abuf1);
  const int tile0 = blockIdx.x * kM;
  const int rows = min(kM, n_envs - tile0);
  const float* src = obs + size_t(tile0) * obs_dim;
  const uint32_t tile_bytes = uint32_t(rows) * uint32_t(obs_dim) * 4u;
  const bool tma_obs = (tile_bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                       tile_bytes <= uint32_t(a1_elems) * 2u;
  const bool stream = wbuf_elems > 0;
  if (tid == 0) {
    mbar_init(&sh->bar_obs, 1);
    mbar_init(&sh->bar_w, 1);
    mbar_init(&sh->bar_mma, 1);
    mbar_init(&sh->bar_chunk, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (tma_obs) {
      mbar_expect_tx(&sh->bar_obs, tile_bytes);
      bulk_g2s(stage, src, tile_bytes, &sh->bar_obs);
    }
    if (!stream) {
      uint32_t bytes = 0;
      for (int l = 0; l < 4; ++l) bytes += uint32_t(D.k[l]) * D.n[l] * 2;
      mbar_expect_tx(&sh->bar_w, bytes);
      for (int l = 0; l < 4; ++l) bulk_g2s(wsm[l], P.w[l], uint32_t(D.k[l]) * D.n[l] * 2, &sh->bar_w);
    }
  }
  if (warp == 0) {  // TMEM: 256 columns (max layer width)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&sh->tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  for (int c = tid; c < obs_dim; c += kThreads) {
    sh->wmean[c] = __ldg(mean + c);
    sh->winv[c] = 1.f / __ldg(stdv + c);
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  phase(1);

  {
    const int pass_rows = tma_obs ? kM : min(kM, (a1_elems * 2) / (obs_dim * 4));
    const int kchunks = D.k[0] / 8;
    if (tma_obs) mbar_wait(&sh->bar_obs, 0);
    phase(11);
    for (int p0 = 0; p0 < kM; p0 += pass_rows) {
      const int pr = max(0, min(pass_rows, rows - p0));
      if (!tma_obs) {
        const int nf = pr * obs_dim;
        const float* s0 = src + size_t(p0) * obs_dim;
        const int nf4 = (reinterpret_cast<uintptr_t>(s0) & 15) == 0 ? nf / 4 : 0;  // float4 path when aligned
#pragma unroll 4
        for (int i = tid; i < nf4; i += kThreads)
          reinterpret_cast<float4*>(stage)[i] = __ldg(reinterpret_cast<const float4*>(s0) + i);
        for (int i = nf4 * 4 + tid; i < nf; i += kThreads) stage[i] = __ldg(s0 + i);
        __syncthreads();
      }
      const float* st = stage + (tma_obs ? size_t(p0) * obs_dim : 0);
      const int prow = min(pass_rows, kM - p0);
      for (int u = tid; u < prow * kchunks; u += kThreads) {
        const int r = u % prow, kc = u / prow;
        float x8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = kc * 8 + i;
          float x = 0.f;
          if (r < pr && c < obs_dim) {
            x = (st[r * obs_dim + c] - sh->wmean[c]) * sh->winv[c];
            x = fminf(fmaxf(x, -10.f), 10.f);
          }
          x8[i] = x;
        }
        st_chunk(abuf0, kc, p0 + r, x8);
      }
      __syncthreads();
    }
  }
  phase(2);
  uint32_t wphase = 0, mphase = 0;
  run_net(D, P, wsm, abuf0, abuf1, sh, wphase, mphase, tid, stream);
  const uint32_t tbase = sh->tmem + (uint32_t((warp & 3) * 32) << 16);
  if (!value_net) {
    // policy head in row passes through shared memory (the
    // operand buffers are free once the last MMA completed): TMEM -> mean
    // tile [rows][out]; then every thread takes consecutive tile elements, so
    // the mean / action stores are coalesced; the log-prob terms replace the
    // means in place and each row is summed in column order by one thread.
    // Per pass the buffer holds the tile, the rows' noise streams and the
    // columns' standard deviations.
    const int out = D.out;
    const int bytes = (a0_elems + a1_elems) * 2 - out * 4 - 8;
    const int cap = min(kM, bytes / (out * 4 + 8));
    float* tile = reinterpret_cast<float*>(abuf0);
    uint64_t* streams = reinterpret_cast<uint64_t*>(abuf0) + (cap * out + 1) / 2;
    float* sdv = reinterpret_cast<float*>(streams + cap);
    const int nch = D.n[3] / 16;
    if (act_out && tid < out) sdv[tid] = expf(log_std[tid]);
    for (int p0 = 0; p0 < rows; p0 += cap) {
      const int pr = min(cap, rows - p0);
      const bool mine = lrow >= p0 && lrow < p0 + pr;
      if (act_out && mine && quarter_of(warp) == 0) {
        const uint64_t genv = uint64_t(env_offset + row);
        streams[lrow - p0] = stp_derive_seed(seed, 6 /* policy noise */, (genv << 32) | uint32_t(step));
      }
      for (int j = quarter_of(warp); j < nch; j += 4) {
        float v[16];
        tmem_ld16(tbase + uint32_t(16 * j), v);
        if (mine)
          for (int i = 0; i < 16; ++i) {
            const int c = 16 * j + i;
            if (c < out) tile[(lrow - p0) * out + c] = v[i] + P.bias[3][c];
          }
      }
      __syncthreads();
      const size_t g0 = (size_t(tile0) + p0) * out;
      for (int i = tid; i < pr * out; i += kThreads) {
        const int r = i / out, c = i - r * out;
        const float m = tile[i];
        mu_out[g0 + i] = m;
        if (act_out) {
          // Box-Muller on two 24-bit counter-based uniforms
          const uint64_t ns = streams[r];
          const float u1 = fmaxf(stp_uniformf(ns, 2 * c), 1e-7f), u2 = stp_uniformf(ns, 2 * c + 1);
          const float eps = sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
          const float sd = sdv[c];
          act_out[g0 + i] = m + sd * eps;
          tile[i] = -0.5f * eps * eps - log_std[c] - 0.91893853320467274f;
        }
      }
      __syncthreads();
      if (logp_out && tid < pr) {
        float lp = 0.f;
        if (act_out)
          for (int c = 0; c < out; ++c) lp += tile[tid * out + c];
        logp_out[tile0 + p0 + tid] = lp;
      }
      __syncthreads();
    }
  } else if (warp < 4) {
    float v[16];
    tmem_ld16(tbase, v);
    if (row < n_envs) v_out[row] = v[0] + P.bias[3][0];
  }
  tc_before_sync();
  __syncthreads();
  phase(12);
  if (warp == 0) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(sh->tmem));
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
  int c0 = mx(Dpi.k[0], Dpi.k[2]), c1 = mx(Dpi.k[1], Dpi.k[3]);
  if (value_out) {
    c0 = mx(c0, mx(Dv.k[0], Dv.k[2]));
    c1 = mx(c1, mx(Dv.k[1], Dv.k[3]));
  }
  const int a0 = kM * c0, a1 = kM * c1;
  const size_t kSmemMax = 227 * 1024;
  const size_t base = kHeader + size_t(a0 + a1) * 2;
  size_t smem = base + size_t(wmax) * 2;
  int wbuf = 0;  // 0: all weights resident
  for (MlpDims* D : {&Dpi, &Dv})
    for (int l = 0; l < 4; ++l) D->kb_chunk[l] = D->k[l] / 8;
  if (smem > kSmemMax) {
    // stream: one weight buffer filling the rest of shared memory
    wbuf = int((kSmemMax - base) / 2) / 128 * 128;
    for (MlpDims* D : {&Dpi, &Dv}) {
      if (D == &Dv && !value_out) continue;
      for (int l = 0; l < 4; ++l) {
        D->kb_chunk[l] = (wbuf / (8 * D->n[l])) & ~1;
        if (D->kb_chunk[l] < 2)
          return stp::fail(STP_EINVAL, "stp_policy_forward: network too large for shared memory");
      }
    }
    smem = base + size_t(wbuf) * 2;
  }
  static size_t configured[64] = {};  // per device (the attribute is)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || smem > configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_policy_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_policy_mlp attr: ") + cudaGetErrorString(e));
    if (dev >= 0 && dev < 64) configured[dev] = smem;
  }
  const dim3 grid((n_envs + kM - 1) / kM, value_out ? 2 : 1);
  k_policy_mlp<<<grid, kThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      obs, n_envs, obs_dim, obs_mean, obs_std, Dpi, Ppi, Dv, Pv, log_std, seed, step, env_offset, mean_out,
      action_out, logp_out, value_out, a0, a1, wbuf);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return stp::fail(STP_ECUDA, std::string("k_policy_mlp: ") + cudaGetErrorString(e));
  return STP_OK;
}
