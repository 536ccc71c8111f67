// Fused environment-step kernel (K1 contacts + K2 solve + K3 epilogue).
//
// Execution model: one warp segment of W lanes = one env,
// lane b = body b.  Per-lane data that persists across the Newton loop but is
// read once per Newton iteration (constant part of the diagonal block and
// rhs, H(child, parent), limit / contact rows) lives in shared memory; rarely
// used rows (non-PD fallback, aliasing quirk, L) in a global scratch buffer.
// The PCR is run in split block-Jacobi form: per Newton iteration each lane
// factors its diagonal block H_bb = L L^T and forms the transformed block
// Hh = L_b^-1 H(b, parent) L_parent^-T in registers, so a CR iteration on
// Ahat = L^-1 H L^-T needs one 6x6 block product per lane (identity
// diagonal blocks), a 2-round shuffle schedule for the children's terms and
// two segment reductions.
//
// Instantiated per precision in sim_step_f32.cu / sim_step_f64.cu.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "sim_kernels.cuh"
#include "sim_launch.h"

namespace stp {

// Per-warp shared-memory rows; each row holds one T per warp lane.
constexpr int R_HOFF = 0;   // 36: H(child, parent), row-major 6x6
constexpr int R_SCAT = 36;  // 9: child -> parent gather buffer
constexpr int R_HEQ = 45;   // 27: constant diagonal block (21, packed) + rhs (6)
constexpr int R_LIM = 72;   // 7: limit axis (3), d_lo, d_hi, b_lo, b_hi
constexpr int R_QRK = 79;   // 7: quirk d0, ja angular (3), jb angular (3)
constexpr int R_CT = 86;    // 11 per contact slot: n(3) r(3) t1(3) d b
// Rarely used per-lane rows live in a global scratch buffer (L1-resident):
constexpr int G_QH = 0;     // 13: quirk in the transformed system: d0, qa (6), qc (6)
constexpr int G_HD = 13;    // 21: diagonal block, kept only when it is not positive definite
constexpr int G_LC = 34;    // 21: Cholesky factor L of the own block (exact residual test, back-substitution)
constexpr int G_CT = 55;    // 11 per overflow contact slot (terrain instantiation, slots CPB.. CPB+11)
// island mode, per cross-contact slot s at G_XS + kXSlotRows * s:
//   0 partner warp, 1 partner lane, 2 role, 3 r_own, 6 r_part, 9 normal,
//   12 tangent t1, 15 bias, 16 normal-row weight (kc m_eff), 17 active normal
//   weight, 18 friction weight (this Newton iterate), 19.. Hh_x (36, row-major),
//   55 partner's global body index
constexpr int G_XS = G_CT + 11 * kSpillSlots;
static_assert(G_XS + kXSlotRows * kXSlots == kScratchRows, "scratch layout");
template <int CPB>
__host__ __device__ constexpr int smem_rows() {
  return R_CT + 11 * CPB;
}

template <class T, int W>
struct Lane {
  T* sm;
  T* gs;  // global scratch rows of this env (kScratchRows x W)
  unsigned mask;
  int lane, base, b, par_src, maxc;
  int kid[4];  // child lanes (-1 = none)
  bool has_off, quirk, diag_h;
  bool any_quirk, any_diag;  // segment-uniform guards of the rare paths
  int grounds;               // child-gather schedule (DevModel::gather_*)
  unsigned gsrc;             // 8-bit source lane per round
  T gwy[4], gwt[4];
  int ghas_t[4];
  T lim_s;  // -(sum of active limit weights): angular rank-1 term of H(c,p)
  v3<T> lim_a;
  T Hh[36];  // transformed off-diagonal block L_b^-1 H(b, parent) L_parent^-T

  __device__ __forceinline__ T& at(int row) const { return sm[row * 32 + lane]; }
  __device__ __forceinline__ T at_kid(int row, int k) const { return sm[row * 32 + base + k]; }
  __device__ __forceinline__ T& g(int row) const { return gs[row * W + b]; }
  // rows [row, row + 2k) read as k float2 rows (fp32 packed coupling blocks)
  __device__ __forceinline__ float2& g2(int row, int k) const {
    return reinterpret_cast<float2*>(gs + row * W)[k * W + b];
  }

  // contact slot k of this lane: 11 rows n(3) r(3) t1(3) d b, in shared memory
  // for k < CPB, in the global overflow rows (G_CT) beyond (terrain only)
  struct Slot {
    T* p;
    int s;
    __device__ __forceinline__ T& operator[](int f) const { return p[f * s]; }
  };
  template <int CPB>
  __device__ __forceinline__ Slot slot(int k) const {
    if (k < CPB) return {sm + (R_CT + 11 * k) * 32 + lane, 32};
    return {gs + (G_CT + 11 * (k - CPB)) * W + b, W};
  }

  // out = sum over children of v (parent side of a child's contribution)
  template <int K>
  __device__ __forceinline__ void gather(const T (&v)[K], T (&out)[K]) const {
    static_assert(K <= 9, "scatter buffer holds 9 values");
#pragma unroll
    for (int k = 0; k < K; ++k) at(R_SCAT + k) = v[k];
    __syncwarp(mask);
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = T(0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < maxc && kid[i] >= 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] += at_kid(R_SCAT + k, kid[i]);
      }
    }
    __syncwarp(mask);
  }

  // y = Ahat v for the split-preconditioned system Ahat = L^-1 H L^-T:
  // identity diagonal blocks (the own block only when it was not positive
  // definite), Hh v_parent, and the children's Hh^T v_child.
  // RARE = false drops the not-positive-definite and aliasing-quirk terms
  // (caller checked any_diag / any_quirk); GR > 0 = exactly GR gather rounds.
  template <bool RARE = true, int GR = 0>
  __device__ __forceinline__ void apply_hat(const T (&v)[6], T (&y)[6]) const {
    T vp[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) vp[k] = __shfl_sync(mask, v[k], par_src, W);
#pragma unroll
    for (int k = 0; k < 6; ++k) y[k] = v[k];
    if (RARE && any_diag) {  // segment-uniform: some own block was not positive definite
      if (diag_h) {
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          T s = T(0);
#pragma unroll
          for (int c = 0; c < 6; ++c) s += g(G_HD + sidx(r, c)) * v[c];
          y[r] = s;
        }
      }
    }
    // Hh is zero on lanes without a parent block: no branch
    T t[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      T s = y[r];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        s += Hh[r * 6 + c] * vp[c];
        t[c] += Hh[r * 6 + c] * v[r];
      }
      y[r] = s;
    }
    if (RARE && any_quirk) {  // segment-uniform; Ahat(p,c) = Hh^T - d0 qa qc^T
      if (quirk) {
        T s0 = T(0);
#pragma unroll
        for (int k = 0; k < 6; ++k) s0 += g(G_QH + 7 + k) * v[k];
        s0 *= g(G_QH);
#pragma unroll
        for (int k = 0; k < 6; ++k) t[k] -= s0 * g(G_QH + 1 + k);
      }
    }
    // children's contributions: scheduled rounds of shuffles (DevModel::gather_*)
#pragma unroll
    for (int r = 0; r < (GR > 0 ? GR : 4); ++r) {
      if (GR > 0 || r < grounds) {
        const int src = int((gsrc >> (8 * r)) & 0xffu);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const T gk = __shfl_sync(mask, t[k], src, W);
          y[k] += gwy[r] * gk;
          if (ghas_t[r]) t[k] += gwt[r] * gk;
        }
      }
    }
  }

  // fp32 form of apply_hat on packed pairs (v = (v0,v1),(v2,v3),(v4,v5)):
  // FFMA2/FMUL2 do two lanes' worth of FP32 work per issue slot (B200: same
  // 4.4-cycle latency and 128 FMA/clk/SM pipe rate as FFMA).  Hp[3c + rp] =
  // (Hh[2rp][c], Hh[2rp+1][c]): Hh v_parent accumulates row pairs against the
  // broadcast v_parent[c] in the same order as the scalar form; Hh^T v is
  // formed per column as even/odd row partial sums plus one add.
  template <bool RARE, int GR>
  __device__ __forceinline__ void apply_hat_p(const float2 (&v)[3], float2 (&y)[3], const float2 (&Hp)[18]) const {
    float vp[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      vp[2 * k] = __shfl_sync(mask, v[k].x, par_src, W);
      vp[2 * k + 1] = __shfl_sync(mask, v[k].y, par_src, W);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) y[k] = v[k];
    if (RARE && any_diag) {
      if (diag_h) {
        const float vs[6] = {v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y};
        float ys[6];
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          float s = 0.f;
#pragma unroll
          for (int c = 0; c < 6; ++c) s += float(g(G_HD + sidx(r, c))) * vs[c];
          ys[r] = s;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) y[k] = make_float2(ys[2 * k], ys[2 * k + 1]);
      }
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) {
#pragma unroll
      for (int rp = 0; rp < 3; ++rp) y[rp] = __ffma2_rn(Hp[3 * c + rp], make_float2(vp[c], vp[c]), y[rp]);
    }
    float t[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      float2 acc = __fmul2_rn(Hp[3 * c], v[0]);
      acc = __ffma2_rn(Hp[3 * c + 1], v[1], acc);
      acc = __ffma2_rn(Hp[3 * c + 2], v[2], acc);
      t[c] = acc.x + acc.y;
    }
    if (RARE && any_quirk) {
      if (quirk) {
        const float vs[6] = {v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y};
        float s0 = 0.f;
#pragma unroll
        for (int k = 0; k < 6; ++k) s0 += float(g(G_QH + 7 + k)) * vs[k];
        s0 *= float(g(G_QH));
#pragma unroll
        for (int k = 0; k < 6; ++k) t[k] -= s0 * float(g(G_QH + 1 + k));
      }
    }
    float2 tp[3] = {make_float2(t[0], t[1]), make_float2(t[2], t[3]), make_float2(t[4], t[5])};
#pragma unroll
    for (int r = 0; r < (GR > 0 ? GR : 4); ++r) {
      if (GR > 0 || r < grounds) {
        const int src = int((gsrc >> (8 * r)) & 0xffu);
        float2 gp[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          gp[k].x = __shfl_sync(mask, tp[k].x, src, W);
          gp[k].y = __shfl_sync(mask, tp[k].y, src, W);
        }
        const float wy = float(gwy[r]), wt = float(gwt[r]);
#pragma unroll
        for (int k = 0; k < 3; ++k) y[k] = __ffma2_rn(gp[k], make_float2(wy, wy), y[k]);
        if (ghas_t[r]) {
#pragma unroll
          for (int k = 0; k < 3; ++k) tp[k] = __ffma2_rn(gp[k], make_float2(wt, wt), tp[k]);
        }
      }
    }
  }
};

__device__ __forceinline__ float dot6p(const float2 (&a)[3], const float2 (&b)[3]) {
  float2 p = __fmul2_rn(a[0], b[0]);
  p = __ffma2_rn(a[1], b[1], p);
  p = __ffma2_rn(a[2], b[2], p);
  return p.x + p.y;
}

// Cholesky factor Lc (lower, packed) of an SPD 6x6 block (krylov.cpp:27-41)
// with reciprocal diagonal rd and Mi = Lc^-1; identity when the block is not
// positive definite (the reference's identity fallback, krylov.cpp:76-80).
template <class T>
__device__ __forceinline__ bool factor6(const T (&H)[21], T (&Lc)[21], T (&rd)[6], T (&Mi)[21], bool dyn) {
  bool ok = dyn;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      T s = H[tri(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= Lc[tri(i, k)] * Lc[tri(j, k)];
      if (i == j) {
        ok = ok && (s > T(0));
        // lanes that end on the identity fallback (no body, static body, not
        // positive definite) take sqrt/reciprocal of 1 instead of 0 / negative /
        // NaN: same result, and no IEEE special-case slow-path call per lane
        const T sv = ok ? s : T(1);
        if constexpr (sizeof(T) == 4) {  // fp32: one MUFU.RSQ instead of IEEE sqrt + reciprocal
          rd[i] = rsqrtf(sv);
          Lc[tri(i, i)] = sv * rd[i];
        } else {
          const T d = sqrt(sv);
          Lc[tri(i, i)] = d;
          rd[i] = T(1) / d;
        }
      } else {
        Lc[tri(i, j)] = s * rd[j];
      }
    }
  }
  if (!ok) {
#pragma unroll
    for (int k = 0; k < 21; ++k) {
      Lc[k] = T(0);
      Mi[k] = T(0);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      Lc[tri(i, i)] = T(1);
      Mi[tri(i, i)] = T(1);
      rd[i] = T(1);
    }
    return false;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    Mi[tri(i, i)] = rd[i];
#pragma unroll
    for (int j = 0; j < i; ++j) {
      T s = T(0);
#pragma unroll
      for (int k = j; k < i; ++k) s += Lc[tri(i, k)] * Mi[tri(k, j)];
      Mi[tri(i, j)] = -s * rd[i];
    }
  }
  return true;
}

// alpha / beta of the PCR recurrences: fp32 uses reciprocal + multiply
// (two roundings; the f64 parity instrument keeps IEEE division).
// (rcp.approx.ftz + multiply: the value __fdividef gives for normal-range
// divisors, without its large-divisor range checks)
__device__ __forceinline__ float fdiv(float a, float b) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  return a * r;
}
__device__ __forceinline__ double fdiv(double a, double b) { return a / b; }

#ifndef STP_SCATTER_SUM
#define STP_SCATTER_SUM 1
#endif

// Four segment sums.  Reduce-scatter form: the first butterfly level trades
// two of the four values (each half keeps the pair it owns), the second one,
// the remaining levels carry one value; the four totals are then broadcast
// from lanes 0, W/4, W/2, 3W/4 of the segment.  10 shuffles + 6 adds + 6
// selects instead of 4 log2(W) shuffles + adds, and every lane ends with the
// same bits.
template <int W, class T>
__device__ __forceinline__ void seg_sum4(T& a, T& b, T& c, T& d, unsigned mask) {
  if constexpr (STP_SCATTER_SUM && W >= 4) {
    const int lane = threadIdx.x & (W - 1);
    const bool h1 = lane & (W / 2), h2 = lane & (W / 4);
    T k0 = h1 ? c : a, k1 = h1 ? d : b;
    const T s0 = h1 ? a : c, s1 = h1 ? b : d;
    k0 += __shfl_xor_sync(mask, s0, W / 2, W);
    k1 += __shfl_xor_sync(mask, s1, W / 2, W);
    T k = h2 ? k1 : k0;
    k += __shfl_xor_sync(mask, h2 ? k0 : k1, W / 4, W);
#pragma unroll
    for (int off = W / 8; off > 0; off >>= 1) k += __shfl_xor_sync(mask, k, off, W);
    // lane holds total index 2 h1 + h2: a at lane 0, b at W/4, c at W/2, d at 3W/4
    a = __shfl_sync(mask, k, 0, W);
    b = __shfl_sync(mask, k, W / 4, W);
    c = __shfl_sync(mask, k, W / 2, W);
    d = __shfl_sync(mask, k, 3 * W / 4, W);
  } else {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
      a += __shfl_xor_sync(mask, a, off, W);
      b += __shfl_xor_sync(mask, b, off, W);
      c += __shfl_xor_sync(mask, c, off, W);
      d += __shfl_xor_sync(mask, d, off, W);
    }
  }
}

template <int W, class T>
__device__ __forceinline__ void seg_sum3(T& a, T& b, T& c, unsigned mask) {
#pragma unroll
  for (int off = W / 2; off > 0; off >>= 1) {
    a += __shfl_xor_sync(mask, a, off, W);
    b += __shfl_xor_sync(mask, b, off, W);
    c += __shfl_xor_sync(mask, c, off, W);
  }
}

// Two float pairs summed over the segment (the packed PCR loop's one
// reduction per trip), in the reduce-scatter form of seg_sum4 when enabled.
template <int W>
__device__ __forceinline__ void seg_sum2x2(float2& q0, float2& q1, unsigned mask) {
  if constexpr (STP_SCATTER_SUM && W >= 4) {
    const int lane = threadIdx.x & (W - 1);
    const bool h1 = lane & (W / 2), h2 = lane & (W / 4);
    float2 keep = h1 ? q1 : q0;
    const float2 send = h1 ? q0 : q1;
    keep = __fadd2_rn(keep, make_float2(__shfl_xor_sync(mask, send.x, W / 2, W),
                                        __shfl_xor_sync(mask, send.y, W / 2, W)));
    float k = h2 ? keep.y : keep.x;
    k += __shfl_xor_sync(mask, h2 ? keep.x : keep.y, W / 4, W);
#pragma unroll
    for (int off = W / 8; off > 0; off >>= 1) k += __shfl_xor_sync(mask, k, off, W);
    // lane holds total 2 h1 + h2 of (q0.x, q0.y, q1.x, q1.y)
    q0 = make_float2(__shfl_sync(mask, k, 0, W), __shfl_sync(mask, k, W / 4, W));
    q1 = make_float2(__shfl_sync(mask, k, W / 2, W), __shfl_sync(mask, k, 3 * W / 4, W));
  } else {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
      q0 = __fadd2_rn(q0, make_float2(__shfl_xor_sync(mask, q0.x, off, W), __shfl_xor_sync(mask, q0.y, off, W)));
      q1 = __fadd2_rn(q1, make_float2(__shfl_xor_sync(mask, q1.x, off, W), __shfl_xor_sync(mask, q1.y, off, W)));
    }
  }
}

#ifndef STP_PACKED_PCR
#define STP_PACKED_PCR 1
#endif
constexpr bool kPackedPCR = STP_PACKED_PCR != 0;

#ifndef STP_ONE_REDUCTION
#define STP_ONE_REDUCTION 1
#endif

template <int W, class T>
__device__ __forceinline__ void seg_sum2(T& a, T& b, unsigned mask) {
#pragma unroll
  for (int off = W / 2; off > 0; off >>= 1) {
    a += __shfl_xor_sync(mask, a, off, W);
    b += __shfl_xor_sync(mask, b, off, W);
  }
}

// 4-warp blocks x 3 per SM (168 registers, 12 warps).  One-warp blocks x 12
// measured 0.6 % faster in the L2-flushed bench but 3 % slower with warm caches
// (Humanoid 4096: 0.1673 vs 0.1625 ms) and up to 10 % slower on terrain.
#ifndef STP_MINB
#define STP_MINB 3
#endif
#ifndef STP_TPB
#define STP_TPB 128
#endif
constexpr int kStepThreads = STP_TPB;  // threads per block (whole warps, one env segment each)

// Island mode (ISL): one CTA per contact-merged island, warp w = the island's
// w-th env in index order (the reference's slot order, solver.cpp:472-481).
// Envs stay warp-local; what couples them — inter-agent contact rows, the
// island-wide PCR reductions and exit tests, rollback — goes through shared
// memory and a named barrier over the island's warps.
template <class T>
__host__ __device__ constexpr int island_cap() {
  return sizeof(T) == 4 ? kIslandMax : kIslandMax / 2;
}
constexpr int kXch = kXchEntries;  // per-lane exchange entries (Mi is the largest)

// all warps of a big island arrive; lane 0 of each counts in and spins
static __device__ __noinline__ void big_island_barrier(int* bar_ctr, int target) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    atomicAdd(bar_ctr, 1);
    while (*reinterpret_cast<volatile int*>(bar_ctr) < target) __nanosleep(32);
    __threadfence();
  }
  __syncwarp();
}

template <class T, int W, int CPB, bool ISL = false, bool DBG = false>
__global__ void __launch_bounds__(ISL ? 32 * island_cap<T>() : kStepThreads, (sizeof(T) == 4 && !ISL ? STP_MINB : 1))
    k_env_step(const KArgs<T> a) {
  // programmatic dependent launch (sim_launch.h): when launched early behind
  // the inter-agent pre-step kernels (or K4), wait for them first; a grid
  // launched after this one (K4, the next step's pre-step kernels) may start
  // its own prologue on the SMs this grid frees
  pdl_wait();
  pdl_trigger();
  // env / island selection.  Island mode: big islands (isl_big_mode) are
  // consecutive CTAs of a cooperative launch; islands of <= cap envs are taken
  // round-robin by a persistent grid (isl_next), each CTA looping over them.
  int e = -1, isl_m = 1, isl_w = 0;
  const int* mem = nullptr;  // the island's member envs (unordered)
  int* bar_ctr = nullptr;    // big islands: global barrier counter
  T* big_area = nullptr;     // big islands: the island's global exchange area
  int isl_next = 0, n_isl = 0;
  int isl_base_w = 0;  // one-CTA islands: the island's first warp in the CTA (cap / 2 two-env islands share a CTA)
  int isl_bar_id = 1;  // its named barrier
  int n_pair = 0, n_pair_items = 0;
  if constexpr (ISL) {
    static_assert(W == 32, "island mode: one env per warp");
    constexpr int cap = island_cap<T>();
    if (a.isl_big_mode) {
      // this CTA's (big island, part): parts of an island are consecutive CTAs
      const int nbig = *a.big_count;
      int acc = 0, bi = -1, part = 0;
      for (int i = 0; i < nbig; ++i) {
        const int p = (a.big_size[i] + cap - 1) / cap;
        if (int(blockIdx.x) < acc + p) {
          bi = i;
          part = int(blockIdx.x) - acc;
          break;
        }
        acc += p;
      }
      if (bi < 0) return;
      isl_m = a.big_size[bi];
      mem = a.big_members + a.big_off[bi];
      isl_w = part * cap + int(threadIdx.x >> 5);
      if (isl_w >= isl_m) return;  // never arrives at the island barrier
      bar_ctr = a.big_bar + bi;
      big_area = a.big_xch + size_t(a.big_off[bi]) * kBigStride;
      // env = the member of rank isl_w (index order = the reference's slot order)
      const int ln = threadIdx.x & 31;
      int found = -1;
      for (int k = ln; k < isl_m; k += 32) {
        const int mk = mem[k];
        int rank = 0;
        for (int j = 0; j < isl_m; ++j) rank += mem[j] < mk;
        if (rank == isl_w) found = mk;
      }
      e = __reduce_max_sync(0xffffffffu, found);
    } else {
      n_isl = *a.isl_count;
      n_pair = *a.isl_npair;
      n_pair_items = (n_pair + int(blockDim.x >> 6) - 1) / int(blockDim.x >> 6);  // cap / 2 pairs per item
      isl_next = blockIdx.x;  // work item: a group of four two-env islands, or one other island
    }
  } else {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    e = a.e_begin + tid / W;
    if (e >= a.n) return;  // whole segments exit together
    if (a.merged && a.merged[e] == 1) return;  // stepped by the island launch
  }
  for (;;) {
    if constexpr (ISL) {
      if (!a.isl_big_mode) {  // the next work item of this CTA
        if (isl_next >= n_pair_items + (n_isl - n_pair)) return;
        const int cw = threadIdx.x >> 5;
        int island = -1;
        if (isl_next < n_pair_items) {  // warps 2j, 2j + 1: two-env island (cap / 2) item + j
          const int slot = int(blockDim.x >> 6) * isl_next + (cw >> 1);
          if (slot < n_pair) island = a.isl_order[slot];
          isl_base_w = cw & ~1;
          isl_bar_id = 1 + (cw >> 1);
          isl_w = cw & 1;
        } else {  // one island in the whole CTA
          island = a.isl_order[n_pair + isl_next - n_pair_items];
          isl_base_w = 0;
          isl_bar_id = 1;
          isl_w = cw;
        }
        mem = a.isl_members + (island >= 0 ? island : 0) * kIslandMax;
        isl_m = 0;
        if (island >= 0)
          for (int k = 0; k < kIslandMax; ++k) isl_m += mem[k] >= 0;
        e = -1;
        for (int k = 0; k < isl_m; ++k) {
          int rank = 0;
          for (int j = 0; j < isl_m; ++j) rank += mem[j] < mem[k];
          if (rank == isl_w) e = mem[k];
        }
      }
    }
    if (!ISL || a.isl_big_mode || isl_w < isl_m) {  // the step of env e
  const int lane = threadIdx.x & 31;
  const int b = lane % W;
  const int base = lane - b;
  const unsigned mask = W == 32 ? 0xffffffffu : (((1u << W) - 1u) << base);
  const DevModel<T>& M = *a.model;
  const DevCfg<T>& cf = a.cfg;
  const bool act = b < M.nb;
  const bool dyn = act && !M.is_static[b];
  const int par = act ? M.parent[b] : -1;
  const int jnt = act ? M.joint[b] : -1;
  const int par_src = par >= 0 ? par : b;
  const bool pdyn = par >= 0 && !M.is_static[par];
  const int J = M.nj;
  // contact slots per body: CPB in shared memory (+ overflow rows for terrain)
  constexpr int CT = CPB > 2 ? CPB + kSpillSlots : CPB;

  extern __shared__ unsigned char smem_raw[];
  Lane<T, W> L;
  L.sm = reinterpret_cast<T*>(smem_raw) + (threadIdx.x >> 5) * (smem_rows<CPB>() * 32);
  // island exchange area (ISL): per-lane entries, reduction partials, votes;
  // shared memory for one-CTA islands, a global area for big islands
  T* xch = reinterpret_cast<T*>(smem_raw) + (ISL ? island_cap<T>() : 0) * smem_rows<CPB>() * 32;
  T* red = xch + (ISL ? island_cap<T>() * 32 * kXch : 0);
  // one-CTA islands: two halves of 4 * cap partials (isl_sum / isl_sum4 alternate
  // between them, so the barrier that protected the reuse is not needed)
  int* vote = reinterpret_cast<int*>(red + 8 * island_cap<T>());
  if (ISL && big_area) {
    xch = big_area;
    red = xch + size_t(isl_m) * 32 * kXch;
    vote = reinterpret_cast<int*>(red + 4 * isl_m);
  } else if (ISL) {  // this island's slices (indexed by rank within the island)
    xch += isl_base_w * 32 * kXch;
    red += 4 * isl_base_w;
    vote += isl_base_w;
  }
  int bar_gen = 0;
  auto isl_bar = [&]() {
    if constexpr (ISL) {
      if (bar_ctr) {
        // all warps of a big island (several CTAs, co-resident by the
        // cooperative launch): generation-counted global barrier, out of
        // line (one copy instead of one per call site: the island kernel's
        // warps run alone on their SMs and stall on instruction fetch)
        big_island_barrier(bar_ctr, ++bar_gen * isl_m);
      } else {
        asm volatile("bar.sync %0, %1;\n" ::"r"(isl_bar_id), "r"(32 * isl_m) : "memory");
      }
    }
  };
  // segment sums / votes over the whole island (the warp forms without ISL)
  int red_par = 0;  // one-CTA islands: the half of `red` the next island sum uses
  // The half used by one sum is reused two sums later; the barrier of the sum
  // in between orders every warp's reads before any warp's next writes.
  auto red_buf = [&]() -> T* {
    if (bar_ctr) return red;  // big islands: one buffer, a trailing barrier
    T* rb = red + red_par * 4 * island_cap<T>();
    red_par ^= 1;
    return rb;
  };
  auto isl_sum = [&](T v) -> T {
    v = seg_sum<W>(v, mask);
    if constexpr (ISL) {
      T* rb = red_buf();
      if (lane == 0) rb[isl_w] = v;
      isl_bar();
      T s = T(0);
      for (int k = 0; k < isl_m; ++k) s += rb[k];
      if (bar_ctr) isl_bar();
      v = s;
    }
    return v;
  };
  auto isl_sum4 = [&](T& v0, T& v1, T& v2, T& v3) {
    seg_sum4<W>(v0, v1, v2, v3, mask);
    if constexpr (ISL) {
      T* rb = red_buf();
      if (lane == 0) {
        rb[4 * isl_w] = v0;
        rb[4 * isl_w + 1] = v1;
        rb[4 * isl_w + 2] = v2;
        rb[4 * isl_w + 3] = v3;
      }
      isl_bar();
      T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
      for (int k = 0; k < isl_m; ++k) {
        s0 += rb[4 * k];
        s1 += rb[4 * k + 1];
        s2 += rb[4 * k + 2];
        s3 += rb[4 * k + 3];
      }
      if (bar_ctr) isl_bar();
      v0 = s0;
      v1 = s1;
      v2 = s2;
      v3 = s3;
    }
  };
  auto isl_all = [&](bool p) -> bool {
    bool r = __all_sync(mask, p);
    if constexpr (ISL) {
      if (!bar_ctr) {
        // one-CTA island: the vote is the named barrier's own AND reduction
        // (one instruction instead of a shared-memory vote between two barriers)
        int v;
        asm volatile(
            "{\n\t.reg .pred pi, po;\n\tsetp.ne.b32 pi, %1, 0;\n\t"
            "bar.red.and.pred po, %2, %3, pi;\n\tselp.b32 %0, 1, 0, po;\n\t}\n"
            : "=r"(v)
            : "r"(int(r)), "r"(isl_bar_id), "r"(32 * isl_m)
            : "memory");
        return v != 0;
      }
      if (lane == 0) vote[isl_w] = r ? 1 : 0;
      isl_bar();
      r = true;
      for (int k = 0; k < isl_m; ++k) r = r && vote[k] != 0;
      isl_bar();
    }
    return r;
  };
  auto isl_any = [&](bool p) -> bool { return !isl_all(!p); };
  L.gs = a.scratch + size_t(e) * kScratchRows * W;
  L.mask = mask;
  L.lane = lane;
  L.base = base;
  L.b = b;
  L.par_src = par_src;
  L.maxc = M.max_children;
#pragma unroll
  for (int i = 0; i < 4; ++i) L.kid[i] = act ? M.child_list[i][b] : -1;
  L.has_off = dyn && pdyn && jnt >= 0;
  L.quirk = false;
  L.diag_h = false;
  L.any_quirk = false;
  L.any_diag = false;
  L.grounds = M.gather_rounds;
  L.gsrc = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    L.gsrc |= unsigned(M.gather_src[r][b] & 0xff) << (8 * r);
    L.gwy[r] = M.gather_wy[r][b];
    L.gwt[r] = M.gather_wt[r][b];
    L.ghas_t[r] = M.gather_has_t[r];
  }
  L.lim_s = T(0);
  L.lim_a = {0, 0, 0};

  // Task state, origin and the pre-step pose are (re)loaded from global
  // memory where needed instead of being kept live across the solve.
  auto load_counters = [&](int32_t (&c)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = a.counters ? a.counters[size_t(e) * 8 + k] : 0;
  };

  // ---- load body state (SoA, coalesced per field) ------------------------
  const size_t sbase = size_t(e) * kStateFields * W + b;
  v3<T> x{0, 0, 0}, v{0, 0, 0}, w{0, 0, 0};
  qt<T> q{1, 0, 0, 0};
  if (act) {
    x = {a.state[sbase + 0 * W], a.state[sbase + 1 * W], a.state[sbase + 2 * W]};
    q = {a.state[sbase + 3 * W], a.state[sbase + 4 * W], a.state[sbase + 5 * W], a.state[sbase + 6 * W]};
    v = {a.state[sbase + 7 * W], a.state[sbase + 8 * W], a.state[sbase + 9 * W]};
    w = {a.state[sbase + 10 * W], a.state[sbase + 11 * W], a.state[sbase + 12 * W]};
  }

  float act_u = 0.f;  // this lane's joint action (env mode)
  bool step_failed = false;
  bool overflow = false;
  int nc = 0;
  int newton_done = 0, krylov_total = 0;
  bool perturbed = false;
  int32_t cnt[8];
  double ox, oy;
  T tx, ty, ltau;
  unsigned feet_bits;

  bool do_reset = false;
  if (a.mode == 2) {
    load_counters(cnt);
    ox = a.origin[2 * e];
    oy = a.origin[2 * e + 1];
    tx = a.target ? a.target[2 * e] : T(0);
    ty = a.target ? a.target[2 * e + 1] : T(0);
    ltau = (jnt >= 0 && a.last_tau) ? a.last_tau[size_t(e) * J + jnt] : T(0);
    feet_bits = a.feet ? a.feet[e] : 0u;
    // reset only: performed at the shared reset site below
    do_reset = a.reset_mask == nullptr || a.reset_mask[e];
  } else {
    // ---------------- actuation (clamp_torques, solver.cpp:395-403) -------
    T tau = T(0);
    if (jnt >= 0) {
      if (a.mode == 1) {
        act_u = a.actions[size_t(e) * J + jnt];
        tau = T(act_u) * M.tmax[b];  // actions scaled by tau_max
      } else {
        tau = T(a.torques[size_t(e) * J + jnt]);
      }
      tau = min(max(tau, -M.tmax[b]), M.tmax[b]);
    }
    // external loads (Scene::external_force/torque, scene.hpp:45-46)
    v3<T> fext{0, 0, 0}, text{0, 0, 0};
    if (a.loads && act) {
      const size_t lb = size_t(e) * 6 * W + b;
      fext = {a.loads[lb + 0 * W], a.loads[lb + 1 * W], a.loads[lb + 2 * W]};
      text = {a.loads[lb + 3 * W], a.loads[lb + 4 * W], a.loads[lb + 5 * W]};
      for (int k = 0; k < 6; ++k) a.loads[lb + k * W] = T(0);  // clear_external_loads
    }
    // perturbation schedule (apply_perturbations)
    if (a.mode == 1 && a.task.perturb_max > 0 &&
        a.counters[size_t(e) * 8 + C_FRAME] == a.counters[size_t(e) * 8 + C_NEXTP]) {
      perturbed = true;
      if (b == M.root) {
        const uint64_t genv = uint64_t(a.env_offset + e);
        const uint64_t ps = stp_derive_seed(a.seed, STP_TAG_PERTURB,
                                            (genv << 32) | uint32_t(a.counters[size_t(e) * 8 + C_PERTDRAW]));
        const double f = a.task.force_lo + (a.task.force_hi - a.task.force_lo) * stp_uniform(ps, 1);
        const double phi = 2.0 * M_PI * stp_uniform(ps, 2);
        fext.x += T(f * cos(phi));
        fext.y += T(f * sin(phi));
      }
    }

    // ---------------- K1: contacts (detect_contacts, collide.cpp:270-299) -
    // slot k of this lane: rows R_CT + 11k: n(3) r(3) t1(3) d b; sep kept in d's row until rows are built
    auto add_contact = [&](v3<T> p, v3<T> n, T sep, int key = -1) {
      if (nc < CT) {
        const auto S = L.template slot<CPB>(nc);
        const v3<T> r = p - x;
        S[6] = T(key);
        S[0] = n.x;
        S[1] = n.y;
        S[2] = n.z;
        S[3] = r.x;
        S[4] = r.y;
        S[5] = r.z;
        S[10] = sep;
        ++nc;
      } else {
        overflow = true;
      }
    };
    if (dyn) {
      const T margin = cf.margin;
      const int shp = M.shape[b];
      const T rad = M.radius[b];
      // world_shape, collide.cpp:38-78
      const qt<T> lr{M.lrot[0][b], M.lrot[1][b], M.lrot[2][b], M.lrot[3][b]};
      const qt<T> rot = qmul(q, lr);
      const v3<T> pos = x + qrot(q, ldv(M.lpos, b));
      v3<T> p0 = pos, p1 = pos;
      T lo_z;
      T Rb[9];
      if (shp == STP_CAPSULE) {
        const v3<T> ax = qrot(rot, v3<T>{T(0), T(0), M.half_len[b]});
        p0 = pos - ax;
        p1 = pos + ax;
        lo_z = min(p0.z, p1.z) - rad;
      } else if (shp == STP_SPHERE) {
        lo_z = pos.z - rad;
      } else {
        rot_mat(rot, Rb);
        const T ez = fabs(Rb[6]) * M.hext[0][b] + fabs(Rb[7]) * M.hext[1][b] + fabs(Rb[8]) * M.hext[2][b];
        lo_z = pos.z - ez;
      }
      // collide_plane, collide.cpp:93-119 (gated by aabb_min.z < margin, :286)
      if (cf.plane && lo_z < margin) {
        const v3<T> up{0, 0, 1};
        if (shp == STP_SPHERE) {
          const T sep = p0.z - rad;
          if (sep < margin) add_contact(p0 - up * rad, up, sep);
        } else if (shp == STP_CAPSULE) {
          const T s0 = p0.z - rad;
          if (s0 < margin) add_contact(p0 - up * rad, up, s0, -2);
          const T s1 = p1.z - rad;
          if (s1 < margin) add_contact(p1 - up * rad, up, s1, -1);
        } else if constexpr (CPB > 2) {  // dynamic boxes: 8 corners (host picks the CPB = 4 + overflow instantiation)
          for (int cx = -1; cx <= 1; cx += 2)
            for (int cy = -1; cy <= 1; cy += 2)
              for (int cz = -1; cz <= 1; cz += 2) {
                const v3<T> l{T(cx) * M.hext[0][b], T(cy) * M.hext[1][b], T(cz) * M.hext[2][b]};
                const v3<T> corner{pos.x + Rb[0] * l.x + Rb[1] * l.y + Rb[2] * l.z,
                                   pos.y + Rb[3] * l.x + Rb[4] * l.y + Rb[5] * l.z,
                                   pos.z + Rb[6] * l.x + Rb[7] * l.y + Rb[8] * l.z};
                if (corner.z < margin) add_contact(corner, up, corner.z);
              }
        }
      }
      // static terrain boxes (collide.cpp:287-298), in box-index order
      // (terrain handles always run the CPB = 4 + overflow instantiation)
      if constexpr (CPB > 2) if (a.n_boxes > 0 && shp != STP_BOX) {
        const double ox = a.origin[2 * e], oy = a.origin[2 * e + 1];
        const v3<T> lo{min(p0.x, p1.x) - rad, min(p0.y, p1.y) - rad, min(p0.z, p1.z) - rad};
        const v3<T> hi{max(p0.x, p1.x) + rad, max(p0.y, p1.y) + rad, max(p0.z, p1.z) + rad};
        auto test_box = [&](int i) {
          const double* bx = a.boxes + 8 * i;
          const v3<T> c{T(bx[0] - ox), T(bx[1] - oy), T(bx[2])};  // relative to the env origin
          const v3<T> h{T(bx[3]), T(bx[4]), T(bx[5])};
          const T ex = h.x + h.y;
          if (hi.x + margin < c.x - ex || lo.x - margin > c.x + ex || hi.y + margin < c.y - ex ||
              lo.y - margin > c.y + ex || hi.z + margin < c.z - h.z || lo.z - margin > c.z + h.z)
            return;
          const T cs = T(bx[6]), sn = T(bx[7]);
          // point_obb, collide.cpp:140-173
          auto point_box = [&](v3<T> p, v3<T>& nrm, v3<T>& surf) -> T {
            const v3<T> d0 = p - c;
            const v3<T> loc{cs * d0.x + sn * d0.y, -sn * d0.x + cs * d0.y, d0.z};
            const v3<T> cl{min(max(loc.x, -h.x), h.x), min(max(loc.y, -h.y), h.y), min(max(loc.z, -h.z), h.z)};
            const v3<T> dl = loc - cl;
            const T out = vnorm(dl);
            if (out > T(1e-12)) {
              surf = {c.x + cs * cl.x - sn * cl.y, c.y + sn * cl.x + cs * cl.y, c.z + cl.z};
              nrm = {(cs * dl.x - sn * dl.y) / out, (sn * dl.x + cs * dl.y) / out, dl.z / out};
              return out;
            }
            T best = h.x - fabs(loc.x);
            int axis = 0;
            T sgn = loc.x >= T(0) ? T(1) : T(-1);
            if (h.y - fabs(loc.y) < best) {
              best = h.y - fabs(loc.y);
              axis = 1;
              sgn = loc.y >= T(0) ? T(1) : T(-1);
            }
            if (h.z - fabs(loc.z) < best) {
              best = h.z - fabs(loc.z);
              axis = 2;
              sgn = loc.z >= T(0) ? T(1) : T(-1);
            }
            v3<T> ln{0, 0, 0}, ls = loc;
            if (axis == 0) {
              ln.x = sgn;
              ls.x = sgn * h.x;
            } else if (axis == 1) {
              ln.y = sgn;
              ls.y = sgn * h.y;
            } else {
              ln.z = sgn;
              ls.z = sgn * h.z;
            }
            surf = {c.x + cs * ls.x - sn * ls.y, c.y + sn * ls.x + cs * ls.y, c.z + ls.z};
            nrm = {cs * ln.x - sn * ln.y, sn * ln.x + cs * ln.y, ln.z};
            return -best;
          };
          // one point_box call site per phase (code size: this runs inside the
          // step kernel, whose instruction working set is its bottleneck on
          // terrain): sphere = 1 query at p0 (collide_sphere_obb :175-181);
          // capsule (collide_capsule_obb :183-214) = 32-step ternary search on
          // t, then the mid point and the two end points in that order
          const v3<T> seg = p1 - p0;
          T tmid = T(0);
          if (shp != STP_SPHERE) {
            T lo_t = 0, hi_t = 1;
#pragma unroll 1
            for (int it = 0; it < 32; ++it) {
              const T m1 = lo_t + (hi_t - lo_t) / T(3), m2 = hi_t - (hi_t - lo_t) / T(3);
              T dq[2];
#pragma unroll 1
              for (int q = 0; q < 2; ++q) {
                v3<T> n1, s1;
                dq[q] = point_box(p0 + seg * (q == 0 ? m1 : m2), n1, s1);
              }
              if (dq[0] <= dq[1]) hi_t = m2;
              else lo_t = m1;
            }
            tmid = T(0.5) * (lo_t + hi_t);
          }
          bool mid_added = false;
          const int nq = shp == STP_SPHERE ? 1 : 3;
#pragma unroll 1
          for (int q = 0; q < nq; ++q) {
            const T tt = q == 0 ? tmid : T(q - 1);  // mid (sphere: p0), then t = 0, 1
            if (q > 0 && mid_added && fabs(tt - tmid) < T(0.05)) continue;
            v3<T> nrm, surf;
            const T d = point_box(q == 0 && shp == STP_SPHERE ? p0 : p0 + seg * tt, nrm, surf);
            if (d - rad < margin) {
              add_contact(surf, nrm, d - rad, 4 * i + q);
              if (q == 0) mid_added = true;
            }
          }
        };
        {
          // (stp_set_terrain builds the grid whenever there are boxes)
          // uniform-grid broadphase over the boxes' loose footprints; each box is
          // visited once (in the first shared cell) and the slots are re-sorted
          // by (box index, mid/end) afterwards: the reference's all-boxes loop
          // order (collide.cpp:287-298) is restored exactly.
          const double wx0 = ox + double(lo.x) - double(margin), wx1 = ox + double(hi.x) + double(margin);
          const double wy0 = oy + double(lo.y) - double(margin), wy1 = oy + double(hi.y) + double(margin);
          auto cell = [&](double w, double g0, int n) {
            const int c = int(floor((w - g0) * a.grid_inv));
            return c < 0 ? 0 : (c >= n ? n - 1 : c);
          };
          const int cx0 = cell(wx0, a.grid_x0, a.grid_nx), cx1 = cell(wx1, a.grid_x0, a.grid_nx);
          const int cy0 = cell(wy0, a.grid_y0, a.grid_ny), cy1 = cell(wy1, a.grid_y0, a.grid_ny);
          for (int cy = cy0; cy <= cy1; ++cy)
            for (int cx = cx0; cx <= cx1; ++cx) {
              const int c = cy * a.grid_nx + cx;
              for (int k = a.cell_start[c]; k < a.cell_start[c + 1]; ++k) {
                const int i = a.cell_list[k];
                const int4 bc = a.box_cells[i];
                if (cx != max(bc.x, cx0) || cy != max(bc.y, cy0)) continue;  // visited in an earlier cell
                test_box(i);
              }
            }
          // insertion sort of this lane's slots by key (plane contacts keep key < 0)
          for (int s1 = 1; s1 < nc; ++s1) {
            for (int s2 = s1; s2 > 0; --s2) {
              const auto A = L.template slot<CPB>(s2 - 1), B = L.template slot<CPB>(s2);
              if (!(A[6] > B[6])) break;
#pragma unroll
              for (int f = 0; f < 11; ++f) {
                const T tmp = A[f];
                A[f] = B[f];
                B[f] = tmp;
              }
            }
          }
        }
      }
    }
    const bool any_contact = __any_sync(mask, nc > 0);

    // ---------------- body dynamics (body_dynamics, solver.cpp:230-262) ---
    const qt<T> qp = from<W>(q, par_src, mask);
    v3<T> torque = text;
    {
      v3<T> jt{0, 0, 0};  // this joint's torque: + on the child, - on the parent
      if (jnt >= 0) {
        jt = qrot(qp, ldv(M.ax_p, b)) * tau;  // parent's axis (solver.cpp:240)
        torque = torque + jt;
      }
      T mine[3] = {jt.x, jt.y, jt.z}, kids[3];
      L.gather<3>(mine, kids);
      torque = torque - v3<T>{kids[0], kids[1], kids[2]};
    }
    sym3<T> Iw{0, 0, 0, 0, 0, 0}, Iinv{0, 0, 0, 0, 0, 0};
    const T inv_m = dyn ? M.inv_mass[b] : T(0);
    const T mass = dyn ? M.mass[b] : T(0);
    v3<T> vfree{0, 0, 0}, wfree{0, 0, 0};
    if (dyn) {
      T Rm[9];
      rot_mat(q, Rm);
      Iw = rdrt(Rm, M.inertia[0][b], M.inertia[1][b], M.inertia[2][b]);
      Iinv = rdrt(Rm, M.inv_inertia[0][b], M.inv_inertia[1][b], M.inv_inertia[2][b]);
      const v3<T> force = v3<T>{cf.gx, cf.gy, cf.gz} * mass + fext;
      vfree = v + force * (cf.dt * inv_m);
      // implicit_gyro, solver.cpp:216-226
      v3<T> wg = w;
      const v3<T> mom = smul(Iw, w) + torque * cf.dt;
      for (int it = 0; it < 2; ++it) {
        const v3<T> iw = smul(Iw, wg);
        const v3<T> f = iw + cross(wg, iw) * cf.dt - mom;
        const T I00 = Iw.xx, I01 = Iw.xy, I02 = Iw.xz, I11 = Iw.yy, I12 = Iw.yz, I22 = Iw.zz;
        T jm[9];  // skew(w) I - skew(I w)
        jm[0] = -wg.z * I01 + wg.y * I02;
        jm[1] = -wg.z * I11 + wg.y * I12 + iw.z;
        jm[2] = -wg.z * I12 + wg.y * I22 - iw.y;
        jm[3] = wg.z * I00 - wg.x * I02 - iw.z;
        jm[4] = wg.z * I01 - wg.x * I12;
        jm[5] = wg.z * I02 - wg.x * I22 + iw.x;
        jm[6] = -wg.y * I00 + wg.x * I01 + iw.y;
        jm[7] = -wg.y * I01 + wg.x * I11 - iw.x;
        jm[8] = -wg.y * I02 + wg.x * I12;
        const T A[9] = {I00 + jm[0] * cf.dt, I01 + jm[1] * cf.dt, I02 + jm[2] * cf.dt,
                        I01 + jm[3] * cf.dt, I11 + jm[4] * cf.dt, I12 + jm[5] * cf.dt,
                        I02 + jm[6] * cf.dt, I12 + jm[7] * cf.dt, I22 + jm[8] * cf.dt};
        // adjugate inverse (vec.hpp:107-120) applied to f
        const T cA = A[4] * A[8] - A[5] * A[7], cB = A[2] * A[7] - A[1] * A[8], cC = A[1] * A[5] - A[2] * A[4];
        const T cD = A[5] * A[6] - A[3] * A[8], cE = A[0] * A[8] - A[2] * A[6], cF = A[2] * A[3] - A[0] * A[5];
        const T cG = A[3] * A[7] - A[4] * A[6], cH = A[1] * A[6] - A[0] * A[7], cI = A[0] * A[4] - A[1] * A[3];
        const T det = A[0] * cA + A[1] * cD + A[2] * cG;
        const v3<T> step{(cA / det) * f.x + (cB / det) * f.y + (cC / det) * f.z,
                         (cD / det) * f.x + (cE / det) * f.y + (cF / det) * f.z,
                         (cG / det) * f.x + (cH / det) * f.y + (cI / det) * f.z};
        wg = wg - step;
      }
      wfree = vfinite(wg) ? wg : w;
    }

    // ---------------- joint rows (build_rows, solver.cpp:105-174) --------
    const T bdt = cf.beta / cf.dt;
    const bool has_joint = dyn && jnt >= 0;
    T Hown[21];  // constant part of this lane's diagonal block
    T rhs_own[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 21; ++k) Hown[k] = T(0);
    if (dyn) {
      Hown[tri(0, 0)] = mass;
      Hown[tri(1, 1)] = mass;
      Hown[tri(2, 2)] = mass;
      Hown[tri(3, 3)] = Iw.xx;
      Hown[tri(4, 3)] = Iw.xy;
      Hown[tri(4, 4)] = Iw.yy;
      Hown[tri(5, 3)] = Iw.xz;
      Hown[tri(5, 4)] = Iw.yz;
      Hown[tri(5, 5)] = Iw.zz;
      const v3<T> iwf = smul(Iw, wfree);
      rhs_own[0] = mass * vfree.x;
      rhs_own[1] = mass * vfree.y;
      rhs_own[2] = mass * vfree.z;
      rhs_own[3] = iwf.x;
      rhs_own[4] = iwf.y;
      rhs_own[5] = iwf.z;
    }
    {
      const v3<T> xp = from<W>(x, par_src, mask);
      const v3<T> wp = from<W>(w, par_src, mask);
      const T p_invm = from<W>(inv_m, par_src, mask);
      sym3<T> pI;
      pI.xx = from<W>(Iinv.xx, par_src, mask);
      pI.yy = from<W>(Iinv.yy, par_src, mask);
      pI.zz = from<W>(Iinv.zz, par_src, mask);
      pI.xy = from<W>(Iinv.xy, par_src, mask);
      pI.xz = from<W>(Iinv.xz, par_src, mask);
      pI.yz = from<W>(Iinv.yz, par_src, mask);
      T up[27];  // parent-side contributions (packed diag block + rhs)
#pragma unroll
      for (int k = 0; k < 27; ++k) up[k] = T(0);
      T lim[7] = {0, 0, 0, 0, 0, 0, 0};
      if (has_joint) {
        const v3<T> ra = qrot(qp, ldv(M.anc_p, b));
        const v3<T> rb = qrot(q, ldv(M.anc_c, b));
        const v3<T> cpos = (x + rb) - (xp + ra);
        const v3<T> aw = qrot(qp, ldv(M.ax_p, b));
        const v3<T> bw = qrot(q, ldv(M.ax_c, b));
        const v3<T> ref = fabs(aw.z) < T(0.9) ? v3<T>{0, 0, 1} : v3<T>{1, 0, 0};
        const v3<T> t1 = vunit(cross(aw, ref));
        const v3<T> t2 = cross(aw, t1);
        const v3<T> err = cross(aw, bw);
        T d5[5] = {0, 0, 0, 0, 0};  // row weights (0 = row skipped)
#pragma unroll
        for (int rr = 0; rr < 5; ++rr) {
          T ja[6], jb[6];
          T wsum = T(0);
          T bias;
          if (rr < 3) {
            const v3<T> ek{T(rr == 0), T(rr == 1), T(rr == 2)};
            const v3<T> ca = -cross(ra, ek), cb = cross(rb, ek);
            ja[0] = -ek.x; ja[1] = -ek.y; ja[2] = -ek.z; ja[3] = ca.x; ja[4] = ca.y; ja[5] = ca.z;
            jb[0] = ek.x; jb[1] = ek.y; jb[2] = ek.z; jb[3] = cb.x; jb[4] = cb.y; jb[5] = cb.z;
            if (pdyn) {
              wsum += p_invm * T(1);
              wsum += quad(pI, ca);
            }
            wsum += inv_m * T(1);
            wsum += quad(Iinv, cb);
            bias = -bdt * comp(cpos, rr);
          } else {
            const v3<T> t = rr == 3 ? t1 : t2;
            ja[0] = 0; ja[1] = 0; ja[2] = 0; ja[3] = -t.x; ja[4] = -t.y; ja[5] = -t.z;
            jb[0] = 0; jb[1] = 0; jb[2] = 0; jb[3] = t.x; jb[4] = t.y; jb[5] = t.z;
            if (pdyn) wsum += quad(pI, -t);
            wsum += quad(Iinv, t);
            bias = -bdt * dot(t, err);
          }
          const T d = cf.kj * (wsum > T(1e-12) ? T(1) / wsum : T(0));  // effective_mass, :69-80
          if (!(d > T(0))) continue;  // assemble skips reg <= 0 (solver.cpp:331)
          d5[rr] = d;
          sym_add(Hown, jb, d);
          const T db = d * bias;
#pragma unroll
          for (int r = 0; r < 6; ++r) rhs_own[r] += jb[r] * db;
          if (pdyn) {
#pragma unroll
            for (int r = 0; r < 6; ++r) {
              const T dj = d * ja[r];
#pragma unroll
              for (int c = 0; c <= r; ++c) up[tri(r, c)] += dj * ja[c];
              up[21 + r] += ja[r] * db;
            }
          }
          if (rr == 0 && M.quirk[b]) {  // aliasing quirk: H(p,c) misses row 0
            L.quirk = true;
            L.at(R_QRK + 0) = d;
            L.at(R_QRK + 1) = ja[3];
            L.at(R_QRK + 2) = ja[4];
            L.at(R_QRK + 3) = ja[5];
            L.at(R_QRK + 4) = jb[3];
            L.at(R_QRK + 5) = jb[4];
            L.at(R_QRK + 6) = jb[5];
          }
        }
        // H(c,p) = sum_r d_r jb_r ja_r^T written once in closed form: the
        // structural zeros of the anchor rows (+-e_r on the linear part) and the
        // axis rows (angular only) are skipped, every non-zero entry is the same
        // fma chain in row order as the row-by-row accumulation.
        if (pdyn) {
          v3<T> ca[3], cb[3];
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const v3<T> ek{T(r == 0), T(r == 1), T(r == 2)};
            ca[r] = -cross(ra, ek);
            cb[r] = cross(rb, ek);
          }
#pragma unroll
          for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              L.at(R_HOFF + i * 6 + j) = i == j ? -d5[i] : T(0);
              L.at(R_HOFF + i * 6 + 3 + j) = d5[i] * comp(ca[i], j);
              L.at(R_HOFF + (3 + i) * 6 + j) = -(d5[j] * comp(cb[j], i));
              T acc = T(0);
#pragma unroll
              for (int r = 0; r < 3; ++r) acc += (d5[r] * comp(cb[r], i)) * comp(ca[r], j);
              acc += (d5[3] * comp(t1, i)) * -comp(t1, j);
              acc += (d5[4] * comp(t2, i)) * -comp(t2, j);
              L.at(R_HOFF + (3 + i) * 6 + 3 + j) = acc;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < 36; ++k) L.at(R_HOFF + k) = T(0);
        }
        // speculative limits (solver.cpp:144-173): angular rows along the child axis
        const qt<T> rest{M.rest[0][b], M.rest[1][b], M.rest[2][b], M.rest[3][b]};
        const v3<T> axc = ldv(M.ax_c, b);
        const T angle = hinge_angle(qp, q, rest, axc);
        const v3<T> axw = qrot(q, axc);
        const T rate = dot(axw, w - wp);
        const T lo_gap = angle - M.lim_lo[b];
        const T hi_gap = M.lim_hi[b] - angle;
        const T thr = max(cf.lim_act, T(1.5) * fabs(rate) * cf.dt);
        T wl = T(0);
        if (pdyn) wl += quad(pI, axw);
        wl += quad(Iinv, axw);
        const T meff = wl > T(1e-12) ? T(1) / wl : T(0);
        lim[0] = axw.x;
        lim[1] = axw.y;
        lim[2] = axw.z;
        if (lo_gap < thr) {
          lim[3] = cf.kl * meff;
          lim[5] = uni_bias(lo_gap, cf.beta, cf.dt);
        }
        if (hi_gap < thr) {
          lim[4] = cf.kl * meff;
          lim[6] = uni_bias(hi_gap, cf.beta, cf.dt);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 36; ++k) L.at(R_HOFF + k) = T(0);
      }
#pragma unroll
      for (int k = 0; k < 7; ++k) L.at(R_LIM + k) = lim[k];
      // parent gathers its children's contributions, 9 values at a time
#pragma unroll
      for (int chunk = 0; chunk < 3; ++chunk) {
        T mine[9], got[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) mine[k] = up[9 * chunk + k];
        L.gather<9>(mine, got);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          const int idx = 9 * chunk + k;
          if (idx < 21) Hown[idx] += got[k];
          else rhs_own[idx - 21] += got[k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 21; ++k) L.at(R_HEQ + k) = Hown[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) L.at(R_HEQ + 21 + k) = rhs_own[k];
    // contact rows (solver.cpp:176-210): normal weight + tangent basis
    auto contact_row = [&](const typename Lane<T, W>::Slot& S) {
      const v3<T> n{S[0], S[1], S[2]};
      const v3<T> rr{S[3], S[4], S[5]};
      const T sep = S[10];
      const v3<T> rn = cross(rr, n);
      T wsum = inv_m * dot(n, n);
      wsum += quad(Iinv, rn);
      const v3<T> ref = fabs(n.z) < T(0.9) ? v3<T>{0, 0, 1} : v3<T>{1, 0, 0};
      const v3<T> t1 = vunit(cross(n, ref));
      S[6] = t1.x;
      S[7] = t1.y;
      S[8] = t1.z;
      S[9] = cf.kc * (wsum > T(1e-12) ? T(1) / wsum : T(0));
      S[10] = uni_bias(sep, cf.beta, cf.dt);
    };
    if constexpr (CT > CPB) {  // terrain: one call site (instruction working set)
#pragma unroll 1
      for (int k = 0; k < nc; ++k) contact_row(L.template slot<CPB>(k));
    } else {
#pragma unroll
      for (int k = 0; k < CPB; ++k) {
        if (k < nc) contact_row(L.template slot<CPB>(k));
      }
    }
    // inter-agent contact rows (island mode; collide.cpp:251-266, rows
    // solver.cpp:176-210): slots in the reference's contact order, lever arms,
    // tangent basis, bias and the normal row's weight kc / (J M^-1 J^T) summed
    // over body_a then body_b as effective_mass does (:69-80) — computed the
    // same way on both sides so both agree on every activity decision.
    int xc = 0;
    if constexpr (ISL) {
      const int gme = e * M.nb + b;
      if (act) xc = min(a.xcount[gme], kXSlots);
      int ord[kXSlots] = {0, 1, 2, 3};
      for (int s1 = 1; s1 < xc; ++s1)
        for (int s2 = s1; s2 > 0 && a.xslots[size_t(gme) * kXSlots + ord[s2 - 1]].key >
                                        a.xslots[size_t(gme) * kXSlots + ord[s2]].key;
             --s2) {
          const int t = ord[s2];
          ord[s2] = ord[s2 - 1];
          ord[s2 - 1] = t;
        }
      T* my = xch + (isl_w * 32 + lane) * kXch;
      my[0] = inv_m;
      my[1] = Iinv.xx;
      my[2] = Iinv.yy;
      my[3] = Iinv.zz;
      my[4] = Iinv.xy;
      my[5] = Iinv.xz;
      my[6] = Iinv.yz;
      isl_bar();
      for (int s2 = 0; s2 < xc; ++s2) {
        const XSlot& X = a.xslots[size_t(gme) * kXSlots + ord[s2]];
        const int pe = X.partner / M.nb, pb = X.partner % M.nb;
        int pw = 0;
        for (int k = 0; k < isl_m; ++k) pw += mem[k] < pe;
        const T* pp = xch + (pw * 32 + pb) * kXch;
        const T pinv = pp[0];
        const sym3<T> pI{pp[1], pp[2], pp[3], pp[4], pp[5], pp[6]};
        const int G = G_XS + kXSlotRows * s2;
        const v3<T> n{T(X.normal[0]), T(X.normal[1]), T(X.normal[2])};
        const v3<T> ro{T(X.r_own[0]), T(X.r_own[1]), T(X.r_own[2])};
        const v3<T> rp{T(X.r_part[0]), T(X.r_part[1]), T(X.r_part[2])};
        const v3<T> ref = fabs(n.z) < T(0.9) ? v3<T>{0, 0, 1} : v3<T>{1, 0, 0};
        const v3<T> t1 = vunit(cross(n, ref));
        const bool own_a = X.role > 0;
        const T ia = own_a ? inv_m : pinv, ib = own_a ? pinv : inv_m;
        const sym3<T>& Ia = own_a ? Iinv : pI;
        const sym3<T>& Ib = own_a ? pI : Iinv;
        const v3<T> ra = own_a ? ro : rp, rb = own_a ? rp : ro;
        T wsum = ia * dot(n, n);
        wsum += quad(Ia, cross(ra, n));
        wsum += ib * dot(n, n);
        wsum += quad(Ib, cross(rb, n));  // jb = -(n, rb x n): the quadratic forms are equal
        L.g(G + 0) = T(pw);
        L.g(G + 1) = T(pb);
        L.g(G + 2) = T(X.role);
        L.g(G + 3) = ro.x;
        L.g(G + 4) = ro.y;
        L.g(G + 5) = ro.z;
        L.g(G + 6) = rp.x;
        L.g(G + 7) = rp.y;
        L.g(G + 8) = rp.z;
        L.g(G + 9) = n.x;
        L.g(G + 10) = n.y;
        L.g(G + 11) = n.z;
        L.g(G + 12) = t1.x;
        L.g(G + 13) = t1.y;
        L.g(G + 14) = t1.z;
        L.g(G + 15) = uni_bias(T(X.sep), cf.beta, cf.dt);
        L.g(G + 16) = cf.kc * (wsum > T(1e-12) ? T(1) / wsum : T(0));
        L.g(G + 55) = T(X.partner);
      }
      isl_bar();  // exchange area free again
    }
    // the constant off-diagonal block must be finite (krylov.cpp:113)
    bool off_fin = true;
    if (L.has_off) {
      T z = T(0);
#pragma unroll
      for (int k = 0; k < 36; ++k) z = nf_acc(z, L.at(R_HOFF + k));
      off_fin = isfinite(z);
    }
    const bool off_ok = isl_all(off_fin);

    // ---------------- Newton loop (solver.cpp:540-548) ---------------------
    T u[6] = {v.x, v.y, v.z, w.x, w.y, w.z};  // warm start from current velocities
    // segment-uniform decisions are taken through votes throughout: the
    // compiler then sees uniform control flow and drops the convergence
    // checks it would otherwise put in front of every shuffle of the solve
    const bool need_solve = isl_any(J > 0 || any_contact || xc > 0);
    if (!need_solve) {  // free-body fast path, solver.cpp:517-523
      u[0] = vfree.x; u[1] = vfree.y; u[2] = vfree.z;
      u[3] = wfree.x; u[4] = wfree.y; u[5] = wfree.z;
    } else {
      for (int it = 0; it < cf.newton; ++it) {
        T H[21], rhs[6];
#pragma unroll
        for (int k = 0; k < 21; ++k) H[k] = L.at(R_HEQ + k);
#pragma unroll
        for (int k = 0; k < 6; ++k) rhs[k] = L.at(R_HEQ + 21 + k);
        // unilateral activity + friction weights at the iterate (:304-328)
        const T wpa[3] = {__shfl_sync(mask, u[3], par_src, W), __shfl_sync(mask, u[4], par_src, W),
                          __shfl_sync(mask, u[5], par_src, W)};
        T lim_s = T(0);
        T pl[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (has_joint) {
          const v3<T> axw{L.at(R_LIM), L.at(R_LIM + 1), L.at(R_LIM + 2)};
          const T wc_a = axw.x * u[3] + axw.y * u[4] + axw.z * u[5];
          const T wp_a = pdyn ? axw.x * wpa[0] + axw.y * wpa[1] + axw.z * wpa[2] : T(0);
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const T d = L.at(R_LIM + 3 + side);
            const T bias = L.at(R_LIM + 5 + side);
            const T sg = side == 0 ? T(1) : T(-1);  // lo: jb = +axw; hi: jb = -axw
            const T pred = d * (bias - sg * (wc_a - wp_a));
            if (d > T(0) && pred > T(0)) {
              lim_s -= d;
              const T jb[6] = {0, 0, 0, sg * axw.x, sg * axw.y, sg * axw.z};
              sym_add(H, jb, d);
              const T db = d * bias;
              rhs[3] += jb[3] * db;
              rhs[4] += jb[4] * db;
              rhs[5] += jb[5] * db;
              if (pdyn) {
                pl[0] += d * axw.x * axw.x;
                pl[1] += d * axw.y * axw.x;
                pl[2] += d * axw.y * axw.y;
                pl[3] += d * axw.z * axw.x;
                pl[4] += d * axw.z * axw.y;
                pl[5] += d * axw.z * axw.z;
                pl[6] -= sg * axw.x * db;
                pl[7] -= sg * axw.y * db;
                pl[8] -= sg * axw.z * db;
              }
            }
          }
          L.lim_a = axw;
        }
        L.lim_s = lim_s;
        {
          T got[9];
          L.gather<9>(pl, got);
          H[tri(3, 3)] += got[0];
          H[tri(4, 3)] += got[1];
          H[tri(4, 4)] += got[2];
          H[tri(5, 3)] += got[3];
          H[tri(5, 4)] += got[4];
          H[tri(5, 5)] += got[5];
          rhs[3] += got[6];
          rhs[4] += got[7];
          rhs[5] += got[8];
        }
        // contacts: normal + smoothed Coulomb friction (:311-327)
        auto contact_newton = [&](const typename Lane<T, W>::Slot& S) {
          const v3<T> n{S[0], S[1], S[2]};
          const v3<T> rr{S[3], S[4], S[5]};
          const T cd = S[9], cb = S[10];
          const v3<T> rn = cross(rr, n);
          const T jn[6] = {n.x, n.y, n.z, rn.x, rn.y, rn.z};
          const T pred = cd * (cb - dot6(jn, u));
          if (pred > T(0)) {
            const v3<T> ta{S[6], S[7], S[8]};
            const v3<T> tb = cross(n, ta);
            const v3<T> rta = cross(rr, ta), rtb = cross(rr, tb);
            const T j1[6] = {ta.x, ta.y, ta.z, rta.x, rta.y, rta.z};
            const T j2[6] = {tb.x, tb.y, tb.z, rtb.x, rtb.y, rtb.z};
            const T vt1 = dot6(j1, u), vt2 = dot6(j2, u);
            const T fw = fric_weight(pred, sqrt(vt1 * vt1 + vt2 * vt2), cf.epsf);
            if (cd > T(0)) {
              sym_add(H, jn, cd);
              const T db = cd * cb;
#pragma unroll
              for (int r = 0; r < 6; ++r) rhs[r] += jn[r] * db;
            }
            if (fw > T(0)) {
              sym_add(H, j1, fw);
              sym_add(H, j2, fw);
            }
          }
        };
        if constexpr (CT > CPB) {  // terrain: one call site (instruction working set)
#pragma unroll 1
          for (int k = 0; k < nc; ++k) contact_newton(L.template slot<CPB>(k));
        } else {
#pragma unroll
          for (int k = 0; k < CPB; ++k) {
            if (k < nc) contact_newton(L.template slot<CPB>(k));
          }
        }
        if constexpr (ISL) {
          // inter-agent rows at the iterate: partners' velocities through the
          // exchange area; rates in body_a, body_b order (assemble :304-327)
          T* my = xch + (isl_w * 32 + lane) * kXch;
#pragma unroll
          for (int k = 0; k < 6; ++k) my[k] = u[k];
          isl_bar();
          for (int s2 = 0; s2 < xc; ++s2) {
            const int G = G_XS + kXSlotRows * s2;
            const T* up = xch + (int(L.g(G)) * 32 + int(L.g(G + 1))) * kXch;
            const T role = L.g(G + 2);
            const v3<T> ro{L.g(G + 3), L.g(G + 4), L.g(G + 5)}, rp{L.g(G + 6), L.g(G + 7), L.g(G + 8)};
            const v3<T> n{L.g(G + 9), L.g(G + 10), L.g(G + 11)}, t1{L.g(G + 12), L.g(G + 13), L.g(G + 14)};
            const v3<T> t2 = cross(n, t1);
            const T bias = L.g(G + 15), dn = L.g(G + 16);
            auto rate = [&](const v3<T>& d) {  // J_a u_a + J_b u_b of the row along d
              const v3<T> co = cross(ro, d) * role, cp = cross(rp, d) * (-role);
              const v3<T> lo = d * role, lp = d * (-role);
              const T jo[6] = {lo.x, lo.y, lo.z, co.x, co.y, co.z};
              const T jp[6] = {lp.x, lp.y, lp.z, cp.x, cp.y, cp.z};
              T upv[6];
#pragma unroll
              for (int k = 0; k < 6; ++k) upv[k] = up[k];
              return role > T(0) ? dot6(jo, u) + dot6(jp, upv) : dot6(jp, upv) + dot6(jo, u);
            };
            const T pred = dn * (bias - rate(n));
            T rn = T(0), rf = T(0);
            if (pred > T(0)) {
              const T vt1 = rate(t1), vt2 = rate(t2);
              rf = fric_weight(pred, sqrt(vt1 * vt1 + vt2 * vt2), cf.epsf);
              rn = dn;
            }
            auto jown = [&](const v3<T>& d, T (&j)[6]) {
              const v3<T> c = cross(ro, d) * role;
              j[0] = d.x * role;
              j[1] = d.y * role;
              j[2] = d.z * role;
              j[3] = c.x;
              j[4] = c.y;
              j[5] = c.z;
            };
            if (rn > T(0)) {
              T jn[6];
              jown(n, jn);
              sym_add(H, jn, rn);
              const T db = rn * bias;
#pragma unroll
              for (int r = 0; r < 6; ++r) rhs[r] += jn[r] * db;
            }
            if (rf > T(0)) {
              T j1[6], j2[6];
              jown(t1, j1);
              jown(t2, j2);
              sym_add(H, j1, rf);
              sym_add(H, j2, rf);
            } else {
              rf = T(0);
            }
            L.g(G + 17) = rn;
            L.g(G + 18) = rf;
          }
          isl_bar();
        }

        // ---------------- PCR (solve_krylov_inplace, krylov.cpp:106-174) --
        // Split block-Jacobi form.  With L_b L_b^T = H_bb (krylov.cpp:27-41),
        // plain CR on Ahat = L^-1 H L^-T, xhat = L^T x, bhat = L^-1 b yields
        // the reference's left-preconditioned CR iterates exactly (in exact
        // arithmetic): z = M^-1 r = L^-T rhat, z.Az = rhat.Ahat rhat and
        // Ap.M^-1 Ap = |Ahat phat|^2.  Ahat has identity diagonal blocks, so
        // an iteration needs no diagonal product and no preconditioner solve.
        if constexpr (DBG) {
          if (it == 0 && e == a.dbg_env) {  // assemble_system hook (solver.hpp:41-44)
            T* d = a.dbg + b * kDbgStride;
#pragma unroll
            for (int k = 0; k < 21; ++k) d[k] = H[k];
#pragma unroll
            for (int k = 0; k < 6; ++k) d[21 + k] = rhs[k];
#pragma unroll
            for (int k = 0; k < 6; ++k)
#pragma unroll
              for (int c = 0; c < 6; ++c)
                d[27 + k * 6 + c] = !L.has_off ? T(0)
                                                : L.at(R_HOFF + k * 6 + c) +
                                                      (k >= 3 && c >= 3 ? L.lim_s * comp(L.lim_a, k - 3) *
                                                                              comp(L.lim_a, c - 3)
                                                                        : T(0));
#pragma unroll
            for (int k = 0; k < 7; ++k) d[63 + k] = L.quirk ? L.at(R_QRK + k) : T(0);
          }
        }
        T nz = T(0);
#pragma unroll
        for (int k = 0; k < 21; ++k) nz = nf_acc(nz, H[k]);
#pragma unroll
        for (int k = 0; k < 6; ++k) nz = nf_acc(nz, rhs[k]);
        const bool fin = isfinite(nz);
        ++newton_done;
        if (!off_ok || !isl_all(fin)) {  // reference throws (krylov.cpp:113-114)
          step_failed = true;
          break;
        }
        const T bb = isl_sum(dot6(rhs, rhs));
        if (isl_all(bb == T(0))) {
#pragma unroll
          for (int k = 0; k < 6; ++k) u[k] = T(0);
          continue;
        }
        // Order keeps the register peak low: Lc, rhs, u and H die once bhat,
        // xhat are formed, before the parent's Mi arrives for the Hh build.
        T bh[6], xh[6];
        T lbw;
        {
          T Mi[21];
          {
            T Lc[21], rd[6];
            const bool ok = factor6(H, Lc, rd, Mi, dyn);
            {
              // sigma_min(L)^2 >= 1 / ||L^-1||_F^2: per-lane weight of the cheap
              // lower bound sum_b lbw_b |rhat_b|^2 <= ||r||^2 (see the PCR loop)
              T f = T(0);
#pragma unroll
              for (int k = 0; k < 21; ++k) f += Mi[k] * Mi[k];
              lbw = dyn ? T(1) / f : T(0);
            }
#pragma unroll
            for (int k = 0; k < 21; ++k) L.g(G_LC + k) = Lc[k];
            L.diag_h = dyn && !ok;
            L.any_diag = __any_sync(mask, L.diag_h);
            L.any_quirk = __any_sync(mask, L.quirk);
#pragma unroll
            for (int k = 0; k < 6; ++k) L.at(R_SCAT + k) = rd[k];
            if (L.diag_h) {
#pragma unroll
              for (int k = 0; k < 21; ++k) L.g(G_HD + k) = H[k];
            }
#pragma unroll
            for (int i = 0; i < 6; ++i) {
              T sb = T(0), sx = T(0);
#pragma unroll
              for (int k = 0; k <= i; ++k) sb += Mi[tri(i, k)] * rhs[k];
#pragma unroll
              for (int k = i; k < 6; ++k) sx += Lc[tri(k, i)] * u[k];
              bh[i] = sb;
              xh[i] = sx;
            }
          }
          T Mp[21];
#pragma unroll
          for (int k = 0; k < 21; ++k) Mp[k] = __shfl_sync(mask, Mi[k], par_src, W);
          // Hh = Mi ((H(c,p) + limit term) Mp^T): each row k of H(c,p) is read
          // once, turned into row k of Q = H Mp^T, and scattered into the rows
          // i >= k of Hh (Mi lower triangular)
#pragma unroll
          for (int k = 0; k < 36; ++k) L.Hh[k] = T(0);
          if (L.has_off) {
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              T h[6];
#pragma unroll
              for (int c = 0; c < 6; ++c) {
                h[c] = L.at(R_HOFF + k * 6 + c);
                if (k >= 3 && c >= 3) h[c] += L.lim_s * comp(L.lim_a, k - 3) * comp(L.lim_a, c - 3);
              }
              T qk[6];
#pragma unroll
              for (int j = 0; j < 6; ++j) {
                T sum = T(0);
#pragma unroll
                for (int c = 0; c <= j; ++c) sum += h[c] * Mp[tri(j, c)];
                qk[j] = sum;
              }
#pragma unroll
              for (int i = k; i < 6; ++i) {
                const T m = Mi[tri(i, k)];
#pragma unroll
                for (int j = 0; j < 6; ++j) L.Hh[i * 6 + j] += m * qk[j];
              }
            }
          }
          if (L.quirk) {  // transformed aliasing term: d0 (Mp ja0)(Mi jb0)^T
            const T ja0[6] = {T(-1), 0, 0, L.at(R_QRK + 1), L.at(R_QRK + 2), L.at(R_QRK + 3)};
            const T jb0[6] = {T(1), 0, 0, L.at(R_QRK + 4), L.at(R_QRK + 5), L.at(R_QRK + 6)};
            L.g(G_QH) = L.at(R_QRK);
#pragma unroll
            for (int i = 0; i < 6; ++i) {
              T qa = T(0), qc = T(0);
#pragma unroll
              for (int k = 0; k <= i; ++k) {
                qa += Mp[tri(i, k)] * ja0[k];
                qc += Mi[tri(i, k)] * jb0[k];
              }
              L.g(G_QH + 1 + i) = qa;
              L.g(G_QH + 7 + i) = qc;
            }
          }
          if constexpr (ISL) {
            // transformed coupling blocks of the inter-agent rows:
            // Ahat(own, partner) = Mi_own H(own, partner) Mi_partner^T
            //                    = sum_rows w (Mi_own j_own)(Mi_partner j_partner)^T
            T* my = xch + (isl_w * 32 + lane) * kXch;
#pragma unroll
            for (int k = 0; k < 21; ++k) my[k] = Mi[k];
            isl_bar();
            for (int s2 = 0; s2 < xc; ++s2) {
              const int G = G_XS + kXSlotRows * s2;
              const T* mp = xch + (int(L.g(G)) * 32 + int(L.g(G + 1))) * kXch;
              const T role = L.g(G + 2);
              const v3<T> ro{L.g(G + 3), L.g(G + 4), L.g(G + 5)}, rp{L.g(G + 6), L.g(G + 7), L.g(G + 8)};
              const v3<T> n{L.g(G + 9), L.g(G + 10), L.g(G + 11)}, t1{L.g(G + 12), L.g(G + 13), L.g(G + 14)};
              const v3<T> t2 = cross(n, t1);
              const T wrow[3] = {L.g(G + 17), L.g(G + 18), L.g(G + 18)};
              const v3<T> dir[3] = {n, t1, t2};
              T hx[36];
#pragma unroll
              for (int k = 0; k < 36; ++k) hx[k] = T(0);
#pragma unroll
              for (int r = 0; r < 3; ++r) {
                if (!(wrow[r] > T(0))) continue;
                const v3<T> d = dir[r];
                const v3<T> co = cross(ro, d) * role, cp = cross(rp, d) * (-role);
                const T jo[6] = {d.x * role, d.y * role, d.z * role, co.x, co.y, co.z};
                const T jp[6] = {-d.x * role, -d.y * role, -d.z * role, cp.x, cp.y, cp.z};
                T al[6], be[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                  T sa = T(0), sb = T(0);
#pragma unroll
                  for (int k = 0; k <= i; ++k) {
                    sa += Mi[tri(i, k)] * jo[k];
                    sb += mp[tri(i, k)] * jp[k];
                  }
                  al[i] = wrow[r] * sa;
                  be[i] = sb;
                }
#pragma unroll
                for (int i = 0; i < 6; ++i)
#pragma unroll
                  for (int j = 0; j < 6; ++j) hx[i * 6 + j] += al[i] * be[j];
              }
              if constexpr (sizeof(T) == 4) {  // row pairs (2 rp, 2 rp + 1) as float2 rows rp * 6 + c
#pragma unroll
                for (int rp = 0; rp < 3; ++rp)
#pragma unroll
                  for (int c = 0; c < 6; ++c)
                    L.g2(G + 19, rp * 6 + c) = make_float2(hx[(2 * rp) * 6 + c], hx[(2 * rp + 1) * 6 + c]);
              } else {
#pragma unroll
                for (int k = 0; k < 36; ++k) L.g(G + 19 + k) = hx[k];
              }
            }
            isl_bar();
          }
        }
        // Exit test of the reference, ||r|| > tol ||b|| (krylov.cpp:141, :154),
        // compared squared.  ||r|| = |L rhat| costs 27 FMA per lane, so each
        // iteration first reduces the rigorous lower bound
        // sum_b |rhat_b|^2 / ||L_b^-1||_F^2 <= ||r||^2; only when that bound
        // does not already exceed tol^2 ||b||^2 (by a rounding margin) is the
        // exact norm formed.  The exit decisions are the reference's.
        const T tol2 = cf.tol * cf.tol * bb;
        const T tol2_safe = tol2 * T(1.0001);
        auto res_exact = [&](const T (&rh)[6]) {  // |L rhat|^2, L from the scratch rows
          T s0 = T(0);
#pragma unroll
          for (int i = 0; i < 6; ++i) {
            T ri = T(0);
#pragma unroll
            for (int k = 0; k <= i; ++k) ri += L.g(G_LC + tri(i, k)) * rh[k];
            s0 += ri * ri;
          }
          return isl_sum(s0);
        };
        // The loop is instantiated three times so the common case runs without
        // the rare-term branches and with a compile-time gather schedule.  Exit
        // decisions are segment-uniform by construction (reduced values) and
        // are taken through votes so the compiler sees uniform control flow.
        auto pcr = [&](auto rare_c, auto gr_c) -> int {
          constexpr bool RARE = decltype(rare_c)::value;
          constexpr int GR = decltype(gr_c)::value;
          // y = Ahat v: the env's own blocks, plus in island mode the
          // inter-agent coupling blocks against the partners' v (exchange area)
          // island mode: += the inter-agent coupling blocks against the partners' v
          // One-CTA islands alternate between two 6-entry halves of the
          // exchange slots, so the barrier that protected their reuse is not
          // needed (the island sum after every product orders it)
          int xpar = 0;
          auto couple = [&](const T (&v)[6], T (&y)[6]) {
            if constexpr (ISL) {
              const int h = bar_ctr ? 0 : 6 * xpar;
              xpar ^= 1;
              T* my = xch + (isl_w * 32 + lane) * kXch + h;
#pragma unroll
              for (int k = 0; k < 6; ++k) my[k] = v[k];
              isl_bar();
              for (int s2 = 0; s2 < xc; ++s2) {
                const int G = G_XS + kXSlotRows * s2;
                const T* vp = xch + (int(L.g(G)) * 32 + int(L.g(G + 1))) * kXch + h;
                if constexpr (sizeof(T) == 4) {  // packed row pairs: same products and order per row
                  float2 acc[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                  for (int c = 0; c < 6; ++c)
#pragma unroll
                    for (int rp = 0; rp < 3; ++rp)
                      acc[rp] = __ffma2_rn(L.g2(G + 19, rp * 6 + c), make_float2(vp[c], vp[c]), acc[rp]);
#pragma unroll
                  for (int rp = 0; rp < 3; ++rp) {
                    y[2 * rp] += acc[rp].x;
                    y[2 * rp + 1] += acc[rp].y;
                  }
                } else {
#pragma unroll
                  for (int r = 0; r < 6; ++r) {
                    T acc = T(0);
#pragma unroll
                    for (int c = 0; c < 6; ++c) acc += L.g(G + 19 + r * 6 + c) * vp[c];
                    y[r] += acc;
                  }
                }
              }
              if (bar_ctr) isl_bar();
            }
          };
          auto apply_x = [&](const T (&v)[6], T (&y)[6]) {
            L.template apply_hat<RARE, GR>(v, y);
            couple(v, y);
          };
          if constexpr (sizeof(T) == 4 && kPackedPCR) {
            // fp32: the loop on packed pairs (see Lane::apply_hat_p); island
            // mode adds the coupling blocks and takes its sums / votes over the
            // island (apply_p, sum3 / sum4, all_of)
            float2 Hp[18];
#pragma unroll
            for (int c = 0; c < 6; ++c) {
#pragma unroll
              for (int rp = 0; rp < 3; ++rp) Hp[3 * c + rp] = make_float2(L.Hh[(2 * rp) * 6 + c], L.Hh[(2 * rp + 1) * 6 + c]);
            }
            auto apply_p = [&](const float2 (&v)[3], float2 (&y)[3]) {
              L.template apply_hat_p<RARE, GR>(v, y, Hp);
              if constexpr (ISL) {
                const T vs[6] = {v[0].x, v[0].y, v[1].x, v[1].y, v[2].x, v[2].y};
                T ys[6] = {y[0].x, y[0].y, y[1].x, y[1].y, y[2].x, y[2].y};
                couple(vs, ys);
#pragma unroll
                for (int k = 0; k < 3; ++k) y[k] = make_float2(ys[2 * k], ys[2 * k + 1]);
              }
            };
            auto all_of = [&](bool p) -> bool {
              if constexpr (ISL) return isl_all(p);
              else return __all_sync(mask, p);
            };
            float2 x2[3], rh[3], ar[3], ph[3], ap[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) x2[k] = make_float2(xh[2 * k], xh[2 * k + 1]);
            apply_p(x2, ar);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              rh[k] = dyn ? make_float2(bh[2 * k] - ar[k].x, bh[2 * k + 1] - ar[k].y) : make_float2(0.f, 0.f);
            }
            apply_p(rh, ar);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              ph[k] = rh[k];
              ap[k] = ar[k];
            }
            auto res_exact_p = [&]() {
              const T r6[6] = {rh[0].x, rh[0].y, rh[1].x, rh[1].y, rh[2].x, rh[2].y};
              return res_exact(r6);
            };
            T zaz = dot6p(rh, ar), lb = lbw * dot6p(rh, rh), denom = dot6p(ar, ar);
            if constexpr (ISL) {
              T dummy = T(0);
              isl_sum4(zaz, lb, denom, dummy);
            } else {
              seg_sum3<W>(zaz, lb, denom, mask);
            }
            int kk = 0;
            // Exit tests of krylov.cpp: ||r|| <= tol ||b|| (:141, :154) and the
            // breakdown test (:144) of the next trip are decided together at
            // the end of a trip (both just leave the loop); all operands are
            // segment-uniform, so every test is one vote.
            auto go_on = [&](float lbv, float zv, float dv) {
              bool above = lbv > tol2_safe;
              if (!all_of(above)) above = res_exact_p() > tol2;  // near convergence only
              return all_of(above && dv > 0.f && zv > 0.f);
            };
            if (kk < cf.kmax && go_on(lb, zaz, denom)) {
              for (;;) {
                const float alpha = fdiv(zaz, denom);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                  x2[k] = __ffma2_rn(ph[k], make_float2(alpha, alpha), x2[k]);
                  rh[k] = __ffma2_rn(ap[k], make_float2(-alpha, -alpha), rh[k]);
                }
                if (++kk >= cf.kmax) break;  // exit certain: the rest cannot change xhat
                apply_p(rh, ar);
                // one reduction per trip: (lb, zn) and (aa, ax) as two pairs
                float2 q0 = make_float2(lbw * dot6p(rh, rh), dot6p(rh, ar));
                float2 q1 = make_float2(dot6p(ar, ar), dot6p(ar, ap));
                if constexpr (ISL) isl_sum4(q0.x, q0.y, q1.x, q1.y);
                else seg_sum2x2<W>(q0, q1, mask);
                const float zn = q0.y, aa = q1.x, ax = q1.y;
                const float beta = fdiv(zn, zaz);
                denom = aa + beta * (2.f * ax + beta * denom);
                if (!go_on(q0.x, zn, denom)) break;
                zaz = zn;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                  ph[k] = __ffma2_rn(ph[k], make_float2(beta, beta), rh[k]);
                  ap[k] = __ffma2_rn(ap[k], make_float2(beta, beta), ar[k]);
                }
              }
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              xh[2 * k] = x2[k].x;
              xh[2 * k + 1] = x2[k].y;
            }
            return kk;
          } else {
          T rh[6], ar[6], ph[6], ap[6];
          apply_x(xh, ar);
#pragma unroll
          for (int k = 0; k < 6; ++k) rh[k] = dyn ? bh[k] - ar[k] : T(0);
          apply_x(rh, ar);
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            ph[k] = rh[k];
            ap[k] = ar[k];
          }
          T zaz = dot6(rh, ar), lb = lbw * dot6(rh, rh);
          int kk = 0;
#if STP_ONE_REDUCTION
          // One reduction per trip: |Ahat p|^2 of the next trip follows from
          // |Ahat r|^2, Ahat r . Ahat p and |Ahat p|^2 of this one
          // (Ahat p' = Ahat r + beta Ahat p); ap itself is still updated
          // explicitly, only its norm is formed by the expansion.
          T denom = dot6(ar, ar);
          if constexpr (ISL) {
            T dummy = T(0);
            isl_sum4(zaz, lb, denom, dummy);
          } else {
            seg_sum3<W>(zaz, lb, denom, mask);
          }
          bool above = lb > tol2_safe || res_exact(rh) > tol2;
          while (isl_all(kk < cf.kmax && above)) {
            if (!isl_all(denom > T(0) && zaz > T(0))) break;  // breakdown (krylov.cpp:144)
            const T alpha = fdiv(zaz, denom);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              xh[k] += alpha * ph[k];
              rh[k] -= alpha * ap[k];
            }
            ++kk;
            // at the iteration cap the exit is certain: the product, the norms
            // and the exit test of this point cannot change xhat
            if (kk >= cf.kmax) break;
            apply_x(rh, ar);
            T zn = dot6(rh, ar), aa = dot6(ar, ar), ax = dot6(ar, ap);
            lb = lbw * dot6(rh, rh);
            isl_sum4(lb, zn, aa, ax);
            above = lb > tol2_safe || res_exact(rh) > tol2;
            if (!isl_all(above)) break;
            const T beta = fdiv(zn, zaz);
            zaz = zn;
            denom = aa + beta * (T(2) * ax + beta * denom);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              ph[k] = rh[k] + beta * ph[k];
              ap[k] = ar[k] + beta * ap[k];
            }
          }
#else
          seg_sum2<W>(zaz, lb, mask);
          bool above = lb > tol2_safe || res_exact(rh) > tol2;
          while (__all_sync(mask, kk < cf.kmax && above)) {
            const T denom = seg_sum<W>(dot6(ap, ap), mask);
            if (!__all_sync(mask, denom > T(0) && zaz > T(0))) break;  // breakdown (krylov.cpp:144)
            const T alpha = fdiv(zaz, denom);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              xh[k] += alpha * ph[k];
              rh[k] -= alpha * ap[k];
            }
            ++kk;
            // at the iteration cap the exit is certain: the product, the norms
            // and the exit test of this point cannot change xhat
            if (kk >= cf.kmax) break;
            L.template apply_hat<RARE, GR>(rh, ar);
            T zn = dot6(rh, ar);
            lb = lbw * dot6(rh, rh);
            seg_sum2<W>(lb, zn, mask);
            above = lb > tol2_safe || res_exact(rh) > tol2;
            if (!__all_sync(mask, above)) break;
            const T beta = fdiv(zn, zaz);
            zaz = zn;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              ph[k] = rh[k] + beta * ph[k];
              ap[k] = ar[k] + beta * ap[k];
            }
          }
#endif
          return kk;
          }
        };
        int kk;
        if (ISL || L.any_diag || L.any_quirk) kk = pcr(std::true_type{}, std::integral_constant<int, 0>{});
        else if (__all_sync(mask, L.grounds == 2)) kk = pcr(std::false_type{}, std::integral_constant<int, 2>{});
        else kk = pcr(std::false_type{}, std::integral_constant<int, 0>{});
        // back to velocities: solve L^T u = xhat (reciprocal diagonal parked in R_SCAT)
#pragma unroll
        for (int i = 5; i >= 0; --i) {
          T sum = xh[i];
#pragma unroll
          for (int k = i + 1; k < 6; ++k) sum -= L.g(G_LC + tri(k, i)) * u[k];
          u[i] = sum * L.at(R_SCAT + i);
        }
        krylov_total += kk;
        if constexpr (DBG) {
          if (e == a.dbg_env && b == 0 && it < kDbgNewton) a.dbg[32 * kDbgStride + it] = T(kk);
        }
        T uz = T(0);
#pragma unroll
        for (int k = 0; k < 6; ++k) uz = nf_acc(uz, u[k]);
        const bool ufin = isfinite(uz);
        if (!isl_all(ufin)) {  // never hand back a poisoned iterate (:168-172)
#pragma unroll
          for (int k = 0; k < 6; ++k) u[k] = T(0);
        }
      }
    }

    // pre-step pose, origin and task state back from global memory
    if (act) {
      x = {a.state[sbase + 0 * W], a.state[sbase + 1 * W], a.state[sbase + 2 * W]};
      q = {a.state[sbase + 3 * W], a.state[sbase + 4 * W], a.state[sbase + 5 * W], a.state[sbase + 6 * W]};
      v = {a.state[sbase + 7 * W], a.state[sbase + 8 * W], a.state[sbase + 9 * W]};
      w = {a.state[sbase + 10 * W], a.state[sbase + 11 * W], a.state[sbase + 12 * W]};
    }
    load_counters(cnt);
    ox = a.origin[2 * e];
    oy = a.origin[2 * e + 1];
    tx = a.target ? a.target[2 * e] : T(0);
    ty = a.target ? a.target[2 * e + 1] : T(0);
    ltau = (jnt >= 0 && a.last_tau) ? a.last_tau[size_t(e) * J + jnt] : T(0);
    feet_bits = a.feet ? a.feet[e] : 0u;

    // ---------------- impulse report (report_impulses, :365-391) ----------
    if (a.record) {
      int off = nc;
#pragma unroll
      for (int s2 = 1; s2 < W; s2 <<= 1) {
        const int o = __shfl_up_sync(mask, off, s2, W);
        if (b >= s2) off += o;
      }
      off -= nc;  // exclusive prefix: contact list order = body order
      const int total = __shfl_sync(mask, off + nc, W - 1, W);
      if (b == 0) a.c_count[e] = total;
#pragma unroll 1
      for (int k = 0; k < nc; ++k) {
        if (off + k < a.cap) {
          const auto S = L.template slot<CPB>(k);
          const v3<T> n{S[0], S[1], S[2]};
          const v3<T> rr{S[3], S[4], S[5]};
          const T cd = S[9], cb = S[10];
          const v3<T> rn = cross(rr, n);
          const T jn[6] = {n.x, n.y, n.z, rn.x, rn.y, rn.z};
          const T pn = max(T(0), cd * (cb - dot6(jn, u)));
          v3<T> pt{0, 0, 0};
          if (pn > T(0)) {
            const v3<T> ta{S[6], S[7], S[8]};
            const v3<T> tb = cross(n, ta);
            const v3<T> rta = cross(rr, ta), rtb = cross(rr, tb);
            const T j1[6] = {ta.x, ta.y, ta.z, rta.x, rta.y, rta.z};
            const T j2[6] = {tb.x, tb.y, tb.z, rtb.x, rtb.y, rtb.z};
            const T vt1 = dot6(j1, u), vt2 = dot6(j2, u);
            const T fw = fric_weight(pn, sqrt(vt1 * vt1 + vt2 * vt2), cf.epsf);
            pt = ta * (-fw * vt1) + tb * (-fw * vt2);
          }
          const size_t slot = size_t(e) * a.cap + off + k;
          a.c_body[slot] = b;  // body_b = static (high bits 0, see below)
          double* cdp = a.c_data + slot * kCData;
          const v3<T> pw = x + rr;
          // separation: recovered from the bias row (unilateral_bias is invertible)
          const T sep = cb > T(0) ? -cb * cf.dt / cf.beta : -cb * cf.dt;
          cdp[0] = ox + double(pw.x);
          cdp[1] = oy + double(pw.y);
          cdp[2] = double(pw.z);
          cdp[3] = double(n.x);
          cdp[4] = double(n.y);
          cdp[5] = double(n.z);
          cdp[6] = double(sep);
          cdp[7] = double(pn);
          cdp[8] = double(pt.x);
          cdp[9] = double(pt.y);
          cdp[10] = double(pt.z);
        }
      }
          if constexpr (ISL) {
        // inter-agent contacts follow the env's static ones, in (a, b) order,
        // listed with body_a's env; body_b = partner's global index, encoded
        // in c_body above the low 8 bits (+1, 0 = static)
        T* my = xch + (isl_w * 32 + lane) * kXch;
#pragma unroll
        for (int k = 0; k < 6; ++k) my[k] = u[k];
        isl_bar();
        int na = 0;
        for (int s2 = 0; s2 < xc; ++s2) na += L.g(G_XS + kXSlotRows * s2 + 2) > T(0);
        int offx = na;
#pragma unroll
        for (int s2 = 1; s2 < W; s2 <<= 1) {
          const int o = __shfl_up_sync(mask, offx, s2, W);
          if (b >= s2) offx += o;
        }
        offx -= na;
        const int totx = __shfl_sync(mask, offx + na, W - 1, W);
        int q = 0;
        for (int s2 = 0; s2 < xc; ++s2) {
          const int G = G_XS + kXSlotRows * s2;
          if (!(L.g(G + 2) > T(0))) continue;
          const int idx = total + offx + q++;
          if (idx >= a.cap) continue;
          const T* up = xch + (int(L.g(G)) * 32 + int(L.g(G + 1))) * kXch;
          const v3<T> ro{L.g(G + 3), L.g(G + 4), L.g(G + 5)}, rp{L.g(G + 6), L.g(G + 7), L.g(G + 8)};
          const v3<T> n{L.g(G + 9), L.g(G + 10), L.g(G + 11)}, t1{L.g(G + 12), L.g(G + 13), L.g(G + 14)};
          const v3<T> t2 = cross(n, t1);
          const T cb = L.g(G + 15), dn = L.g(G + 16);
          auto rate = [&](const v3<T>& d) {  // body_a (this lane) then body_b
            const v3<T> ca = cross(ro, d), cp = cross(rp, d);
            const T ja[6] = {d.x, d.y, d.z, ca.x, ca.y, ca.z};
            const T jb[6] = {-d.x, -d.y, -d.z, -cp.x, -cp.y, -cp.z};
            T upv[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) upv[k] = up[k];
            return dot6(ja, u) + dot6(jb, upv);
          };
          const T pn = max(T(0), dn * (cb - rate(n)));
          v3<T> pt{0, 0, 0};
          if (pn > T(0)) {
            const T vt1 = rate(t1), vt2 = rate(t2);
            const T fw = fric_weight(pn, sqrt(vt1 * vt1 + vt2 * vt2), cf.epsf);
            pt = t1 * (-fw * vt1) + t2 * (-fw * vt2);
          }
          const size_t slot = size_t(e) * a.cap + idx;
          a.c_body[slot] = b | ((int(L.g(G + 55)) + 1) << 8);
          double* cdp = a.c_data + slot * kCData;
          const v3<T> pw = x + ro;
          const T sep = cb > T(0) ? -cb * cf.dt / cf.beta : -cb * cf.dt;
          cdp[0] = ox + double(pw.x);
          cdp[1] = oy + double(pw.y);
          cdp[2] = double(pw.z);
          cdp[3] = double(n.x);
          cdp[4] = double(n.y);
          cdp[5] = double(n.z);
          cdp[6] = double(sep);
          cdp[7] = double(pn);
          cdp[8] = double(pt.x);
          cdp[9] = double(pt.y);
          cdp[10] = double(pt.z);
        }
        if (b == 0) a.c_count[e] = total + totx;
        isl_bar();
      }
}

    // ---------------- integrate + rollback (:562-569, :580-593) -----------
    v3<T> xn = x, vn = v, wn = w;
    qt<T> qn = q;
    if (dyn) {
      vn = {u[0], u[1], u[2]};
      wn = {u[3], u[4], u[5]};
      xn = x + vn * cf.dt;
      qn = qunit(qmul(qexp(wn * cf.dt), q));
    }
    const bool fin_state = vfinite(xn) && qfinite(qn) && vfinite(vn) && vfinite(wn);
    step_failed = step_failed || !isl_all(fin_state);  // the whole island rolls back (:580-593)
    if (!step_failed) {
      x = xn;
      q = qn;
      v = vn;
      w = wn;
    }
  }

  // ---------------- K3: task epilogue (env_step) ---------
  bool reuse_angles = false, reuse_head = false;
  T yaw_r = T(0), head_r = T(0), ang_r = T(0);
  constexpr bool kF32 = std::is_same<T, float>::value;
  T sy_r = T(0), cy_r = T(1), sh_r = T(0), ch_r = T(1);  // fp32: yaw / heading unit vectors
  if (a.mode == 1) {
    const T tx_r = tx, ty_r = ty;
    const int R = M.root;
    const T prev_rx = a.state[size_t(e) * kStateFields * W + 0 * W + R];
    const T prev_ry = a.state[size_t(e) * kStateFields * W + 1 * W + R];
    const v3<T> xr = from<W>(x, R, mask);
    const qt<T> qr = from<W>(q, R, mask);
    // feet-ground flags: foot has >= 1 static contact this step
    const unsigned fb = __ballot_sync(mask, act && nc > 0 && ((M.feet_mask >> b) & 1)) >> base;
    T rew = T(0);
    const qt<T> qpn = from<W>(q, par_src, mask);
    // angles the observation can reuse when the env is not reset (same inputs)
    if (!step_failed) {
      // compute_reward
      const T ox_ = tx - prev_rx, oy_ = ty - prev_ry;
      const T od0 = sqrt(ox_ * ox_ + oy_ * oy_);
      T S = T(0);
      if (od0 > T(0)) S = ((xr.x - prev_rx) * ox_ + (xr.y - prev_ry) * oy_) / od0 / cf.dt;
      T cth;
      if constexpr (kF32) {  // cos(heading - yaw) from the two unit vectors, no angles
        unit_dir(T(2) * (qr.w * qr.z + qr.x * qr.y), T(1) - T(2) * (qr.y * qr.y + qr.z * qr.z), &sy_r, &cy_r);
        unit_dir(ty - xr.y, tx - xr.x, &sh_r, &ch_r);
        cth = ch_r * cy_r + sh_r * sy_r;
      } else {
        const T yaw = atan2(T(2) * (qr.w * qr.z + qr.x * qr.y), T(1) - T(2) * (qr.y * qr.y + qr.z * qr.z));
        yaw_r = yaw;
        head_r = atan2(ty - xr.y, tx - xr.x);
        cth = cos_(head_r - yaw);
      }
      const T rhead = cth > T(0.8) ? T(1) : cth / T(0.8);
      const T cvert = T(1) - T(2) * (qr.x * qr.x + qr.y * qr.y);
      const T rstand = cvert > T(0.93) ? T(1) : T(0);
      T tc = T(0), uc = T(0), nl = T(0);
      if (jnt >= 0) {
        const T uu = T(act_u);
        tc = fabs(min(max(uu, T(-1)), T(1)));
        uc = uu * uu;
        const T ang = hinge_angle(qpn, q, qt<T>{M.rest[0][b], M.rest[1][b], M.rest[2][b], M.rest[3][b]},
                                  ldv(M.ax_c, b));
        ang_r = ang;
        nl = (ang - M.lim_lo[b] < cf.lim_act || M.lim_hi[b] - ang < cf.lim_act) ? T(1) : T(0);
      }
      seg_sum2<W>(tc, uc, mask);
      nl = seg_sum<W>(nl, mask);
      const T nfeet = T(__popc(fb));
      rew = M.alive_bonus + S + T(0.5) * rhead + T(0.05) * rstand - T(4) * tc - T(0.5) * uc - T(0.2) * nl - nfeet;
    }
    // termination
    const int frame_before = cnt[C_FRAME];
    cnt[C_FRAME] += 1;
    const bool low = xr.z < M.fall_height;
    cnt[C_FALL] = low ? cnt[C_FALL] + 1 : 0;
    const bool fell = a.task.fall_grace > 0 ? cnt[C_FALL] >= a.task.fall_grace : low;
    const bool dn = step_failed || fell || cnt[C_FRAME] >= a.task.episode_cap;
    const uint64_t genv = uint64_t(a.env_offset + e);
    if (perturbed) {
      cnt[C_PERTDRAW] += 1;
      const uint64_t ps = stp_derive_seed(a.seed, STP_TAG_PERTURB, (genv << 32) | uint32_t(cnt[C_PERTDRAW]));
      const int span = a.task.perturb_max - a.task.perturb_min + 1;
      int k = int(floor(stp_uniform(ps, 0) * span));
      if (k >= span) k = span - 1;
      cnt[C_NEXTP] = frame_before + a.task.perturb_min + k;
    }
    // flagrun targets (update_flagrun_targets)
    if (a.task.target_refresh > 0) {
      cnt[C_FLAG] += 1;
      const T dx = tx - xr.x, dy = ty - xr.y;
      if (cnt[C_FLAG] >= a.task.target_refresh || sqrt(dx * dx + dy * dy) < T(a.task.target_tolerance)) {
        const uint64_t fs = stp_derive_seed(a.seed, STP_TAG_FLAG, (genv << 32) | uint32_t(cnt[C_FLAGDRAW]));
        cnt[C_FLAGDRAW] += 1;
        const double rad = a.task.target_radius * sqrt(stp_uniform(fs, 0));
        const double phi = 2.0 * M_PI * stp_uniform(fs, 1);
        tx = T(double(xr.x) + rad * cos(phi));
        ty = T(double(xr.y) + rad * sin(phi));
        cnt[C_FLAG] = 0;
      }
    }
    ltau = jnt >= 0 ? min(max(T(act_u), T(-1)), T(1)) : T(0);
    feet_bits = fb;
    do_reset = dn && a.task.auto_reset;
    reuse_angles = !step_failed && !do_reset;
    reuse_head = reuse_angles && tx == tx_r && ty == ty_r;
    if (b == 0) {
      if (a.reward) a.reward[e] = float(rew);
      if (a.done) a.done[e] = dn ? 1 : 0;
    }
  }
  if (do_reset) {  // single inlined reset site (SPEC.md:261-269 / auto-reset)
    reset_env<T, W>(a, M, e, b, mask, act, x, q, v, w, cnt, tx, ty, ox, oy);
    ltau = T(0);
    feet_bits = 0;
  }
  if (a.mode >= 1) {
    if (jnt >= 0 && a.last_tau) a.last_tau[size_t(e) * J + jnt] = ltau;
    if (b == 0 && a.feet) a.feet[e] = feet_bits;
    // observation (Table 2)
    if (a.obs) {
      const int R = M.root;
      float* o = a.obs + size_t(e) * a.obs_dim;
      const v3<T> xr2 = from<W>(x, R, mask);
      const qt<T> qr2 = from<W>(q, R, mask);
      const v3<T> vr2 = from<W>(v, R, mask);
      const v3<T> wr2 = from<W>(w, R, mask);
      T yaw = T(0), sy, cy;
      if constexpr (kF32) {
        sy = sy_r;
        cy = cy_r;
        if (!reuse_angles)
          unit_dir(T(2) * (qr2.w * qr2.z + qr2.x * qr2.y), T(1) - T(2) * (qr2.y * qr2.y + qr2.z * qr2.z), &sy, &cy);
      } else {
        yaw = reuse_angles ? yaw_r
                           : atan2(T(2) * (qr2.w * qr2.z + qr2.x * qr2.y),
                                   T(1) - T(2) * (qr2.y * qr2.y + qr2.z * qr2.z));
        sincos_(yaw, &sy, &cy);
      }
      if (b == 0) {
        o[0] = float(xr2.z);
        o[1] = float(atan2(T(2) * (qr2.w * qr2.x + qr2.y * qr2.z), T(1) - T(2) * (qr2.x * qr2.x + qr2.y * qr2.y)));
        T sp = T(2) * (qr2.w * qr2.y - qr2.z * qr2.x);
        sp = min(max(sp, T(-1)), T(1));
        o[2] = float(asin(sp));
        o[3] = float(cy * vr2.x + sy * vr2.y);
        o[4] = float(-sy * vr2.x + cy * vr2.y);
        o[5] = float(vr2.z);
        o[6] = float(cy * wr2.x + sy * wr2.y);
        o[7] = float(-sy * wr2.x + cy * wr2.y);
        o[8] = float(wr2.z);
        T sh, ch;
        if constexpr (kF32) {  // sin / cos of (heading - yaw) by the angle-difference identities
          T sh0 = sh_r, ch0 = ch_r;
          if (!reuse_head) unit_dir(ty - xr2.y, tx - xr2.x, &sh0, &ch0);
          sh = sh0 * cy - ch0 * sy;
          ch = ch0 * cy + sh0 * sy;
        } else {
          sincos_((reuse_head ? head_r : atan2(ty - xr2.y, tx - xr2.x)) - yaw, &sh, &ch);
        }
        o[9] = float(sh);
        o[10] = float(ch);
        for (int f = 0; f < M.n_feet; ++f) o[11 + 3 * J + f] = ((feet_bits >> M.feet[f]) & 1) ? 1.f : 0.f;
      }
      const qt<T> qpo = from<W>(q, par_src, mask);
      const v3<T> wpo = from<W>(w, par_src, mask);
      if (jnt >= 0) {
        const v3<T> axc = ldv(M.ax_c, b);
        const T ang = reuse_angles
                          ? ang_r
                          : hinge_angle(qpo, q, qt<T>{M.rest[0][b], M.rest[1][b], M.rest[2][b], M.rest[3][b]}, axc);
        const T rate = dot(qrot(q, axc), w - wpo);  // joint_velocity, solver.cpp:413-417
        o[11 + jnt] = float(ang);
        o[11 + J + jnt] = float(rate);
        o[11 + 2 * J + jnt] = float(ltau);
      }
      if (a.task.height_map) {
        const double rx = ox + double(xr2.x), ry = oy + double(xr2.y);
        for (int k = b; k < 165; k += W) {
          const int i = k / 11, jj = k % 11;
          const double fx = geo_offset(i - 7), fy = geo_offset(jj - 5);
          const double px = rx + double(cy) * fx - double(sy) * fy;
          const double py = ry + double(sy) * fx + double(cy) * fy;
          o[11 + 3 * J + M.n_feet + k] = float(terrain_height_grid(a, px, py) - double(xr2.z));
        }
      }
    }
  }

  // ---------------- re-centre the env origin on the root (fp32 range) -----
  {
    const T rx = from<W>(x.x, M.root, mask), ry = from<W>(x.y, M.root, mask);
    const T sx = fabs(rx) >= T(1) ? T(rint(rx)) : T(0);
    const T sy = fabs(ry) >= T(1) ? T(rint(ry)) : T(0);
    if (sx != T(0) || sy != T(0)) {
      x.x -= sx;
      x.y -= sy;
      tx -= sx;
      ty -= sy;
      ox += double(sx);
      oy += double(sy);
    }
  }

  // ---------------- store ---------------------------------------------------
  if (act) {
    a.state[sbase + 0 * W] = x.x;
    a.state[sbase + 1 * W] = x.y;
    a.state[sbase + 2 * W] = x.z;
    a.state[sbase + 3 * W] = q.w;
    a.state[sbase + 4 * W] = q.x;
    a.state[sbase + 5 * W] = q.y;
    a.state[sbase + 6 * W] = q.z;
    a.state[sbase + 7 * W] = v.x;
    a.state[sbase + 8 * W] = v.y;
    a.state[sbase + 9 * W] = v.z;
    a.state[sbase + 10 * W] = w.x;
    a.state[sbase + 11 * W] = w.y;
    a.state[sbase + 12 * W] = w.z;
  }
  if (b == 0) {
    a.origin[2 * e] = ox;
    a.origin[2 * e + 1] = oy;
    if (a.target) {
      a.target[2 * e] = tx;
      a.target[2 * e + 1] = ty;
    }
    if (a.counters)
      for (int k = 0; k < 8; ++k) a.counters[size_t(e) * 8 + k] = cnt[k];
    if (a.mode != 2) {
      if (a.newton_out) a.newton_out[e] = newton_done;
      if (a.krylov_out) a.krylov_out[e] = krylov_total;
      if (a.failed_out) a.failed_out[e] = step_failed ? 1 : 0;
    }
  }
  if (a.mode != 2 && a.overflow_out) {
    bool ov = __any_sync(mask, overflow);
    // flagged in the island preparation (reported, never silent): island
    // steps when cross contacts were dropped; an env whose island did not
    // fit the island launches (merged 2, stepped alone) or when candidate
    // env pairs were dropped (bit 8)
    if constexpr (ISL) ov = ov || *a.isl_err != 0;
    else if (a.merged) ov = ov || a.merged[e] == 2 || (*a.isl_err & 8) != 0;
    if (b == 0) a.overflow_out[e] = ov ? 1 : 0;
  }
    }
    if constexpr (!ISL) return;
    if (a.isl_big_mode) return;
    __syncthreads();  // exchange area and named barrier free for the next island
    isl_next += gridDim.x;
  }
}

template <class T, int W, int CPB, bool DBG = false>
static cudaError_t launch_one(const KArgs<T>& a, cudaStream_t s, bool pdl = true) {
  constexpr int threads = kStepThreads;
  const size_t smem = size_t(threads / 32) * smem_rows<CPB>() * 32 * sizeof(T);
  static bool configured[64] = {};
  if (first_on_device(configured)) {
    cudaError_t err = cudaFuncSetAttribute(k_env_step<T, W, CPB, false, DBG>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (err != cudaSuccess) return err;
  }
  const long long total = (long long)(a.n - a.e_begin) * W;
  const int blocks = int((total + threads - 1) / threads);
  if (!pdl) {
    k_env_step<T, W, CPB, false, DBG><<<blocks, threads, smem, s>>>(a);
    return cudaGetLastError();
  }
  return launch_pdl(k_env_step<T, W, CPB, false, DBG>, dim3(blocks), dim3(threads), smem, s, a);
}

template <class T, int CPB>
int big_island_ctas();

template <class T, int W, int CPB>
static cudaError_t launch_island(const KArgs<T>& a, cudaStream_t s, const volatile int* count_hint) {
  constexpr int cap = island_cap<T>();
  const size_t smem = size_t(cap) * smem_rows<CPB>() * 32 * sizeof(T) + size_t(cap) * 32 * kXch * sizeof(T) +
                      size_t(8 * cap) * sizeof(T) + size_t(cap) * sizeof(int);
  static bool configured[64] = {};
  if (first_on_device(configured)) {
    cudaError_t err = cudaFuncSetAttribute(k_env_step<T, W, CPB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(smem));
    if (err != cudaSuccess) return err;
  }
  // a persistent grid (islands are taken round-robin): at most n / 2 islands,
  // at most one CTA per SM
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // An island CTA holds an SM's whole register file (8 warps x 254
  // registers), so a CTA without an island still keeps the main launch off its
  // SM until it exits: with the previous step's island count as a hint the
  // grid is 2x that + 8 (the round-robin loop covers any count)
  const int half = (a.n - a.e_begin) / 2 > 0 ? (a.n - a.e_begin) / 2 : 1;
  int grid = half < sms ? half : sms;
  if (count_hint) {
    const int h = 2 * *count_hint + 8;
    if (h < grid) grid = h;
  }
  k_env_step<T, W, CPB, true><<<grid, 32 * cap, smem, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (count_hint)  // this step's count for the next step's grid (async, pinned)
    e = cudaMemcpyAsync(const_cast<int*>(count_hint), a.isl_count, sizeof(int), cudaMemcpyDeviceToHost, s);
  return e;
}

// islands with more envs than one CTA holds: consecutive CTAs per island, all
// co-resident (cooperative launch) so the island's global barrier cannot wait
// on an unscheduled CTA; CTAs without a part exit at once.  Launched on the
// caller's stream after the main launch: a cooperative grid on the
// high-priority side stream would hold back the main launch's remaining blocks
// until the whole grid fits (~22 us per step even with no big island)
template <class T, int W, int CPB>
static cudaError_t launch_island_big(const KArgs<T>& a, cudaStream_t s) {
  if (!a.big_count) return cudaSuccess;
  constexpr int cap = island_cap<T>();
  const size_t smem = size_t(cap) * smem_rows<CPB>() * 32 * sizeof(T) + size_t(cap) * 32 * kXch * sizeof(T) +
                      size_t(8 * cap) * sizeof(T) + size_t(cap) * sizeof(int);
  KArgs<T> b = a;
  b.isl_big_mode = 1;
  void* args[] = {&b};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_env_step<T, W, CPB, true>),
                                     dim3(big_island_ctas<T, CPB>()), dim3(32 * cap), args, smem, s);
}

// co-resident CTAs of the island launch on this device: the part budget of
// the big islands (k_islands flags islands beyond it)
template <class T, int CPB>
int big_island_ctas() {
  static int per_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 1;
  if (!per_dev[dev]) {
    constexpr int cap = island_cap<T>();
    const size_t smem = size_t(cap) * smem_rows<CPB>() * 32 * sizeof(T) + size_t(cap) * 32 * kXch * sizeof(T) +
                        size_t(8 * cap) * sizeof(T) + size_t(cap) * sizeof(int);
    cudaFuncSetAttribute(k_env_step<T, 32, CPB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_env_step<T, 32, CPB, true>, 32 * cap, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    per_dev[dev] = per_sm * sms > 0 ? per_sm * sms : 1;
  }
  return per_dev[dev];
}

template <class T>
int island_launch_budget(int cpb) {
  // STP_ISLAND_BUDGET (tests only) lowers the budget to exercise the
  // over-budget path (islands stepped env by env and flagged)
  static const char* env = getenv("STP_ISLAND_BUDGET");
  const int lim = cpb <= 2 ? big_island_ctas<T, 2>() : big_island_ctas<T, 4>();
  return env ? std::min(lim, atoi(env)) : lim;
}

template <class T>
cudaError_t launch_env_step(const KArgs<T>& a, int lanes, int cpb, cudaStream_t s, const IslandStreams* isl) {
  if (a.dbg) {  // assemble_system hook: its own instantiations (no cost on the hot path)
    if (a.merged) return cudaErrorInvalidValue;
    if (lanes == 32) return cpb <= 2 ? launch_one<T, 32, 2, true>(a, s) : launch_one<T, 32, 4, true>(a, s);
    if (lanes == 16) return cpb <= 2 ? launch_one<T, 16, 2, true>(a, s) : launch_one<T, 16, 4, true>(a, s);
    return cpb <= 2 ? launch_one<T, 8, 2, true>(a, s) : launch_one<T, 8, 4, true>(a, s);
  }
  if (a.merged) {  // inter-agent collisions: the merged islands and the independent envs
    if (lanes != 32) return cudaErrorInvalidValue;
    // The island launches touch only merged envs and the main launch skips
    // them, so they run concurrently: islands first on the side stream (an
    // island CTA is one latency-bound chain of a few warps), the main launch
    // on `s` filling the rest of the machine, then `s` joins the side stream.
    cudaStream_t is = isl && isl->side ? isl->side : s;
    cudaError_t e = cudaSuccess;
    if (is != s) {
      e = cudaEventRecord(isl->fork, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(is, isl->fork, 0);
      if (e != cudaSuccess) return e;
    }
    const volatile int* hint = isl ? isl->h_count : nullptr;
    e = cpb <= 2 ? launch_island<T, 32, 2>(a, is, hint) : launch_island<T, 32, 4>(a, is, hint);
    if (e != cudaSuccess) return e;
    // with islands last step, a plain launch: an early (PDL) main launch would
    // take every SM before the island CTAs, which need a whole SM's register
    // file each, are released by the fork; launched together, the side
    // stream's priority places them first.  Without islands, PDL.
    const bool pdl = is == s || (hint && *hint == 0);
    e = cpb <= 2 ? launch_one<T, 32, 2>(a, s, pdl) : launch_one<T, 32, 4>(a, s, pdl);
    if (e != cudaSuccess) return e;
    e = cpb <= 2 ? launch_island_big<T, 32, 2>(a, s) : launch_island_big<T, 32, 4>(a, s);
    if (e != cudaSuccess || is == s) return e;
    e = cudaEventRecord(isl->join, is);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, isl->join, 0);
    return e;
  }
  if (lanes == 32) {
    if (cpb <= 2) return launch_one<T, 32, 2>(a, s);
    return launch_one<T, 32, 4>(a, s);
  }
  if (lanes == 16) {
    if (cpb <= 2) return launch_one<T, 16, 2>(a, s);
    return launch_one<T, 16, 4>(a, s);
  }
  if (cpb <= 2) return launch_one<T, 8, 2>(a, s);
  return launch_one<T, 8, 4>(a, s);
}

}  // namespace stp
