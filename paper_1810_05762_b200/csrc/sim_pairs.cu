// Inter-agent contact detection: the dynamic-pair part of
// detect_contacts (collide.cpp:300-343) for every env of a sim, on the GPU.
//
// The reference bins margin-expanded body AABBs into a hash grid and then
// keeps the pairs (a < b) of different agents whose AABBs overlap within the
// margin (aabb_overlap, :80-84), sorted by (a, b), one segment-segment contact
// each (closest_segment_segment :219-249, collide_dynamic_pair :251-266).  The
// grid is only a broadphase: any overlapping pair shares a cell, so the pair
// set is exactly "different agents, overlapping AABBs".  Here:
//   K_a  one warp per env: world shapes of its bodies in double (env origin +
//        local pose, world_shape :38-78), the env's AABB, and the env filed in
//        a hashed 2-D grid by its AABB centre;
//   K_b  per env: the grid cells within reach -> env pairs whose AABBs
//        overlap within the margin;
//   K_c  one warp per candidate env pair: all body pairs, the reference's AABB
//        test and narrow phase.
// The detection entry sorts the contacts by (a, b) (cub) for its output; the
// step path writes them into per-body slots (sorted there) and forms islands.
// Body indices are global within the sim: env * B + body.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "sim_device.cuh"
#include "sim_launch.h"

namespace stp {
namespace {

struct WShape {  // world shape of one body (double), collide.cpp:27-36
  double p0[3], p1[3], lo[3], hi[3];
  double x[3];  // body position (row lever arms, solver.cpp:180-181)
  double r;
  int ok;  // dynamic sphere / capsule (boxes never pair, :255)
};

__device__ __forceinline__ bool box_overlap(const double* a, const double* b, double m) {
  // a, b: lo[3], hi[3]; the reference's aabb_overlap with margin m
  return a[0] <= b[3] + m && b[0] <= a[3] + m && a[1] <= b[4] + m && b[1] <= a[4] + m && a[2] <= b[5] + m &&
         b[2] <= a[5] + m;
}

// Broadphase over envs on a hashed 2-D grid (cell kCell m): one warp per env
// forms its bodies' world shapes (lane = body) and the env AABB by warp
// min / max, and files the env under the cell of its AABB centre; the query
// visits the cells within reach (from the largest env extent of the step) and
// keeps the pairs whose env AABBs overlap within the margin.  Envs that do
// not fit their bin go to an overflow list every query also scans, so the
// candidate set is always complete.
constexpr double kCell = 3.0;
constexpr int kBinCap = 8;

__device__ __forceinline__ int cell_of(double v) { return int(floor(v / kCell)); }
__device__ __forceinline__ unsigned cell_hash(int cx, int cy, unsigned hmask) {
  return (unsigned(cx) * 73856093u ^ unsigned(cy) * 19349663u) & hmask;
}

template <class T>
__device__ __forceinline__ void shapes_of_env(const DevModel<T>* __restrict__ Mp, const T* __restrict__ state,
                                              const double* __restrict__ origin, int e, int b, int W,
                                              WShape* __restrict__ ws, WShape* sw, double* __restrict__ env_box,
                                              int2* __restrict__ env_cell, int* __restrict__ bin_count,
                                              int* __restrict__ bins, unsigned hmask, int* __restrict__ ovf,
                                              int* __restrict__ n_ovf, int& ext_bits, int* __restrict__ xcount) {
  const DevModel<T>& M = *Mp;
  const int B = M.nb;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  if (b < B) {
    WShape s{};
    if (xcount) xcount[size_t(e) * B + b] = 0;  // this step's cross-contact slots (step path)
    const size_t sb = size_t(e) * kStateFields * W + b;
    auto st = [&](int f) { return state[sb + size_t(f) * W]; };
    // rotations in the handle's precision (world_shape, collide.cpp:38-78),
    // the env origin added in double
    const v3<T> xr{st(0), st(1), st(2)};
    const qt<T> q{st(3), st(4), st(5), st(6)};
    const qt<T> lr{M.lrot[0][b], M.lrot[1][b], M.lrot[2][b], M.lrot[3][b]};
    const v3<T> lp{M.lpos[0][b], M.lpos[1][b], M.lpos[2][b]};
    const qt<T> rot = qmul(q, lr);
    const v3<T> off = qrot(q, lp);
    v3<T> ax{T(0), T(0), T(0)};
    if (M.shape[b] == STP_CAPSULE) ax = qrot(rot, v3<T>{T(0), T(0), M.half_len[b]});
    const double ox = origin[2 * e], oy = origin[2 * e + 1];
    const v3<double> x{ox + double(xr.x), oy + double(xr.y), double(xr.z)};
    const v3<double> pos{x.x + double(off.x), x.y + double(off.y), x.z + double(off.z)};
    const double r = double(M.radius[b]);
    const v3<double> p0{pos.x - double(ax.x), pos.y - double(ax.y), pos.z - double(ax.z)};
    const v3<double> p1{pos.x + double(ax.x), pos.y + double(ax.y), pos.z + double(ax.z)};
    s.ok = !M.is_static[b] && M.shape[b] != STP_BOX;
    s.r = r;
    s.x[0] = x.x;
    s.x[1] = x.y;
    s.x[2] = x.z;
    const double a0[3] = {p0.x, p0.y, p0.z}, a1[3] = {p1.x, p1.y, p1.z};
    for (int k = 0; k < 3; ++k) {
      s.p0[k] = a0[k];
      s.p1[k] = a1[k];
      s.lo[k] = fmin(a0[k], a1[k]) - r;
      s.hi[k] = fmax(a0[k], a1[k]) + r;
      if (s.ok) {
        lo[k] = s.lo[k];
        hi[k] = s.hi[k];
      }
    }
    sw[b] = s;
  }
  __syncwarp();
  {
    static_assert(sizeof(WShape) % 8 == 0, "WShape words");
    constexpr int kWords = int(sizeof(WShape) / 8);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(sw);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(ws + size_t(e) * B);
    for (int i = b; i < B * kWords; i += 32) dst[i] = src[i];
  }
  for (int off = 16; off > 0; off >>= 1)
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], off));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], off));
    }
  if (b == 0) {
    for (int k = 0; k < 3; ++k) {
      env_box[6 * e + k] = lo[k];
      env_box[6 * e + 3 + k] = hi[k];
    }
    if (!(lo[0] <= hi[0])) {  // no dynamic sphere / capsule: never pairs
      env_cell[e] = make_int2(INT_MIN, INT_MIN);
      return;
    }
    const int cx = cell_of(0.5 * (lo[0] + hi[0])), cy = cell_of(0.5 * (lo[1] + hi[1]));
    env_cell[e] = make_int2(cx, cy);
    ext_bits = __float_as_int(__double2float_ru(fmax(hi[0] - lo[0], hi[1] - lo[1])));
    const unsigned h = cell_hash(cx, cy, hmask);
    const int slot = atomicAdd(&bin_count[h], 1);
    if (slot < kBinCap) bins[h * kBinCap + slot] = e;
    else ovf[atomicAdd(n_ovf, 1)] = e;
  }
}

// one launch zeroing the step's counters and the hash-bin counts (was four
// cudaMemsetAsync operations, each a separate ~2-3 us item on the stream)
__global__ void k_pairs_reset(int* __restrict__ bin_count, int nbins, int* __restrict__ gcnt,
                              int* __restrict__ counters, int* __restrict__ icnt) {
  pdl_wait();  // programmatic dependent launch (sim_launch.h)
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nbins) bin_count[i] = 0;
  if (i < 2) {
    gcnt[i] = 0;
    counters[i] = 0;
  }
  if (icnt && i < 5) icnt[i] = 0;
}

template <class T>
__global__ void k_shapes_warp(const DevModel<T>* __restrict__ Mp, const T* __restrict__ state,
                              const double* __restrict__ origin, int n, int W, WShape* __restrict__ ws,
                              double* __restrict__ env_box, int2* __restrict__ env_cell, int* __restrict__ bin_count,
                              int* __restrict__ bins, unsigned hmask, int* __restrict__ ovf, int* __restrict__ n_ovf,
                              int* __restrict__ max_ext_bits, int* __restrict__ xcount) {
  pdl_wait();  // programmatic dependent launch (sim_launch.h)
  pdl_trigger();
  // the warp's shapes are staged in shared memory and written out as
  // coalesced 8-byte words (one 136-byte struct per lane would scatter)
  __shared__ WShape stage[4][32];  // launched with 128 threads
  __shared__ int blk_ext[4];  // the block's largest env extent -> one atomicMax per block
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, b = threadIdx.x & 31;
  if (b == 0) blk_ext[threadIdx.x >> 5] = 0;
  if (e < n) shapes_of_env(Mp, state, origin, e, b, W, ws, stage[threadIdx.x >> 5], env_box, env_cell, bin_count,
                           bins, hmask, ovf, n_ovf, blk_ext[threadIdx.x >> 5], xcount);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int m = max(max(blk_ext[0], blk_ext[1]), max(blk_ext[2], blk_ext[3]));
    if (m > 0) atomicMax(max_ext_bits, m);  // positive floats order as ints
  }
}

__global__ void k_env_query(int n, const double* __restrict__ env_box, const int2* __restrict__ env_cell,
                            const int* __restrict__ bin_count, const int* __restrict__ bins, unsigned hmask,
                            const int* __restrict__ ovf, const int* __restrict__ n_ovf,
                            const int* __restrict__ max_ext_bits, double margin, int2* __restrict__ pairs, int cap,
                            int* __restrict__ n_pairs) {
  pdl_wait();  // programmatic dependent launch (sim_launch.h)
  pdl_trigger();
  // one warp per env; lanes over (cell, bin slot) candidates
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= n) return;
  const int2 ci = env_cell[i];
  if (ci.x == INT_MIN) return;
  const double* bi = env_box + 6 * i;
  // centres of overlapping envs differ by <= (ext_i + ext_max) / 2 + margin
  const double ext_i = fmax(bi[3] - bi[0], bi[4] - bi[1]);
  const double reach = 0.5 * (ext_i + double(__int_as_float(*max_ext_bits))) + margin;
  const int rc = int(floor(reach / kCell)) + 1;  // |x_i - x_j| <= R  =>  |cell_i - cell_j| <= floor(R / C) + 1
  const int side = 2 * rc + 1;
  auto test = [&](int j) {
    if (j <= i) return;
    if (box_overlap(bi, env_box + 6 * j, margin)) {
      const int slot = atomicAdd(n_pairs, 1);
      if (slot < cap) pairs[slot] = make_int2(i, j);
    }
  };
  // kU candidates per lane per pass, their dependent loads (bin count -> bin
  // entry -> cell -> box) issued side by side
  constexpr int kU = 4;
  const int total = side * side * kBinCap;
  for (int u0 = lane; u0 < total; u0 += 32 * kU) {
    int cx[kU], cy[kU], j[kU];
    unsigned h[kU];
    int cnt[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int u = u0 + 32 * q;
      const int c = u / kBinCap;
      cx[q] = ci.x + c % side - rc;
      cy[q] = ci.y + c / side - rc;
      h[q] = cell_hash(cx[q], cy[q], hmask);
      cnt[q] = u < total ? bin_count[h[q]] : 0;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int k = (u0 + 32 * q) % kBinCap;
      j[q] = k < min(cnt[q], kBinCap) ? bins[h[q] * kBinCap + k] : -1;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      if (j[q] < 0) continue;
      const int2 cj = env_cell[j[q]];
      if (cj.x == cx[q] && cj.y == cy[q]) test(j[q]);  // hash collisions: each env once, in its own cell
    }
  }
  const int no = *n_ovf;
  for (int k = lane; k < no; k += 32) test(ovf[k]);
}

// closest points between segments p1q1 and p2q2 (Ericson; collide.cpp:219-249)
__device__ void seg_seg(const double* p1, const double* q1, const double* p2, const double* q2, double* c1,
                        double* c2) {
  double d1[3], d2[3], r[3];
  for (int k = 0; k < 3; ++k) {
    d1[k] = q1[k] - p1[k];
    d2[k] = q2[k] - p2[k];
    r[k] = p1[k] - p2[k];
  }
  auto dot3 = [](const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
  auto clamp01 = [](double v) { return fmin(fmax(v, 0.0), 1.0); };
  const double a = dot3(d1, d1), e = dot3(d2, d2), f = dot3(d2, r);
  const double eps = 1e-12;
  double s = 0.0, t = 0.0;
  if (a <= eps && e <= eps) {
    // two points
  } else if (a <= eps) {
    t = clamp01(f / e);
  } else {
    const double c = dot3(d1, r);
    if (e <= eps) {
      s = clamp01(-c / a);
    } else {
      const double b = dot3(d1, d2);
      const double den = a * e - b * b;
      if (den > eps) s = clamp01((b * f - c * e) / den);
      t = (b * s + f) / e;
      if (t < 0.0) {
        t = 0.0;
        s = clamp01(-c / a);
      } else if (t > 1.0) {
        t = 1.0;
        s = clamp01((b - c) / a);
      }
    }
  }
  for (int k = 0; k < 3; ++k) {
    c1[k] = p1[k] + d1[k] * s;
    c2[k] = p2[k] + d2[k] * t;
  }
}

struct PairContact {
  unsigned long long key;  // a * NB + b
  double point[3], normal[3], sep;
};

// one warp per candidate env pair (A < B): every body pair, aabb test, narrow phase
// a warp's candidate bodies of env pair pr: those whose AABB overlaps the
// other env's AABB within the margin (exact pruning of the B x B body pairs,
// see k_narrow_slots); bit b of the first / second mask: body b of pr.x / pr.y
__device__ __forceinline__ void candidate_bodies(const int2 pr, int B, const WShape* __restrict__ ws,
                                                 const double* __restrict__ env_box, double margin, int lane,
                                                 unsigned& ma, unsigned& mb) {
  bool ta = false, tb = false;
  if (lane < B) {
    const WShape& A = ws[size_t(pr.x) * B + lane];
    const WShape& Bs = ws[size_t(pr.y) * B + lane];
    const double la[6] = {A.lo[0], A.lo[1], A.lo[2], A.hi[0], A.hi[1], A.hi[2]};
    const double lb[6] = {Bs.lo[0], Bs.lo[1], Bs.lo[2], Bs.hi[0], Bs.hi[1], Bs.hi[2]};
    ta = A.ok && box_overlap(la, env_box + 6 * size_t(pr.y), margin);
    tb = Bs.ok && box_overlap(lb, env_box + 6 * size_t(pr.x), margin);
  }
  ma = __ballot_sync(0xffffffffu, ta);
  mb = __ballot_sync(0xffffffffu, tb);
}

__global__ void k_narrow(const int2* __restrict__ pairs, const int* __restrict__ n_pairs_p, int pair_cap, int B,
                         long long NB, const WShape* __restrict__ ws, const double* __restrict__ env_box,
                         double margin, PairContact* __restrict__ out, int cap, int* __restrict__ n_out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int np = min(*n_pairs_p, pair_cap);
  if (warp >= np) return;
  const int2 pr = pairs[warp];
  unsigned ma, mb;
  candidate_bodies(pr, B, ws, env_box, margin, lane, ma, mb);
  const int na = __popc(ma), nb = __popc(mb);
  for (int u = lane; u < na * nb; u += 32) {
    const int ba = __fns(ma, 0, u / nb + 1), bb = __fns(mb, 0, u % nb + 1);
    const WShape& A = ws[size_t(pr.x) * B + ba];
    const WShape& Bs = ws[size_t(pr.y) * B + bb];
    const double la[6] = {A.lo[0], A.lo[1], A.lo[2], A.hi[0], A.hi[1], A.hi[2]};
    const double lb[6] = {Bs.lo[0], Bs.lo[1], Bs.lo[2], Bs.hi[0], Bs.hi[1], Bs.hi[2]};
    if (!box_overlap(la, lb, margin)) continue;
    double ca[3], cb[3];
    seg_seg(A.p0, A.p1, Bs.p0, Bs.p1, ca, cb);
    const double dl[3] = {ca[0] - cb[0], ca[1] - cb[1], ca[2] - cb[2]};
    const double dist = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
    double nrm[3] = {0.0, 0.0, 1.0};
    if (dist > 1e-9) {
      for (int k = 0; k < 3; ++k) nrm[k] = dl[k] / dist;
    }
    const double sep = dist - A.r - Bs.r;
    if (!(sep < margin)) continue;
    PairContact c;
    const long long ga = (long long)pr.x * B + ba, gb = (long long)pr.y * B + bb;
    c.key = (unsigned long long)(ga * NB + gb);
    const double off = Bs.r + 0.5 * (dist - A.r - Bs.r);
    for (int k = 0; k < 3; ++k) {
      c.point[k] = cb[k] + nrm[k] * off;
      c.normal[k] = nrm[k];
    }
    c.sep = sep;
    const int slot = atomicAdd(n_out, 1);
    if (slot < cap) out[slot] = c;
  }
}

// Step path: the same narrow phase, written straight into each body's cross
// contact slots (both sides) plus the env edge of every contact; persistent
// warps loop over the device-counted candidate pairs (no host round trip).
__global__ void k_narrow_slots(const int2* __restrict__ pairs, const int* __restrict__ n_pairs_p, int pair_cap,
                               int B, long long NB, const WShape* __restrict__ ws, const double* __restrict__ env_box,
                               double margin,
                               XSlot* __restrict__ xslots, int* __restrict__ xcount, int2* __restrict__ edges,
                               int edge_cap, int* __restrict__ n_edges, int* __restrict__ err) {
  pdl_wait();  // programmatic dependent launch (sim_launch.h)
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int np = min(*n_pairs_p, pair_cap);
  if (blockIdx.x == 0 && threadIdx.x == 0 && *n_pairs_p > pair_cap) atomicOr(err, 8);  // candidates dropped
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < np; w += nwarps) {
    const int2 pr = pairs[w];
    // exact pruning: a body pair can only overlap (AABBs within the margin) if
    // each body's AABB overlaps the other env's AABB (the union of its bodies'),
    // so only those bodies of either env are paired (crowded HFH: a few bodies
    // near the other agent instead of all B x B)
    unsigned ma, mb;
    candidate_bodies(pr, B, ws, env_box, margin, lane, ma, mb);
    const int na = __popc(ma), nb = __popc(mb);
    for (int u = lane; u < na * nb; u += 32) {
      const int ba = __fns(ma, 0, u / nb + 1), bb = __fns(mb, 0, u % nb + 1);
      const WShape& A = ws[size_t(pr.x) * B + ba];
      const WShape& Bs = ws[size_t(pr.y) * B + bb];
      const double la[6] = {A.lo[0], A.lo[1], A.lo[2], A.hi[0], A.hi[1], A.hi[2]};
      const double lb[6] = {Bs.lo[0], Bs.lo[1], Bs.lo[2], Bs.hi[0], Bs.hi[1], Bs.hi[2]};
      if (!box_overlap(la, lb, margin)) continue;
      double ca[3], cb[3];
      seg_seg(A.p0, A.p1, Bs.p0, Bs.p1, ca, cb);
      const double dl[3] = {ca[0] - cb[0], ca[1] - cb[1], ca[2] - cb[2]};
      const double dist = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
      double nrm[3] = {0.0, 0.0, 1.0};
      if (dist > 1e-9) {
        for (int k = 0; k < 3; ++k) nrm[k] = dl[k] / dist;
      }
      const double sep = dist - A.r - Bs.r;
      if (!(sep < margin)) continue;
      const long long ga = (long long)pr.x * B + ba, gb = (long long)pr.y * B + bb;
      const double off = Bs.r + 0.5 * (dist - A.r - Bs.r);
      double pt[3], xa[3], xb[3];
      for (int k = 0; k < 3; ++k) {
        pt[k] = cb[k] + nrm[k] * off;
        xa[k] = A.x[k];
        xb[k] = Bs.x[k];
      }
      for (int side = 0; side < 2; ++side) {
        const long long me = side == 0 ? ga : gb;
        const int slot = atomicAdd(&xcount[me], 1);
        if (slot >= kXSlots) {
          atomicOr(err, 1);
          continue;
        }
        XSlot x;
        x.key = ga * NB + gb;
        x.partner = int(side == 0 ? gb : ga);
        x.role = side == 0 ? 1 : -1;
        for (int k = 0; k < 3; ++k) {
          x.r_own[k] = pt[k] - (side == 0 ? xa[k] : xb[k]);
          x.r_part[k] = pt[k] - (side == 0 ? xb[k] : xa[k]);
          x.normal[k] = nrm[k];
        }
        x.sep = sep;
        xslots[me * kXSlots + slot] = x;
      }
      const int ei = atomicAdd(n_edges, 1);
      if (ei < edge_cap) edges[ei] = pr;
      else atomicOr(err, 4);
    }
  }
}

// Islands of envs (solver.cpp:458-482 restricted to what couples envs): label
// propagation over the contact edges, then island lists.  One CTA.
// Contact-merged islands by label propagation in one CTA.  Labels live in
// shared memory when the env count fits (`slab`), else in `label`; only edge
// endpoints ever change label (every label value is an endpoint's index), so
// the propagation and pointer-jumping passes run over the edges alone.
__global__ void k_islands(int n, const int2* __restrict__ edges, const int* __restrict__ n_edges_p, int edge_cap,
                          int* __restrict__ label, uint8_t* __restrict__ merged, int* __restrict__ isl_of,
                          int* __restrict__ isl_size, int* __restrict__ isl_fill, int* __restrict__ isl_big,
                          int* __restrict__ isl_members, int* __restrict__ isl_count, int* __restrict__ err,
                          int labels_in_smem, int cap, int max_parts, int* __restrict__ big_count,
                          int* __restrict__ big_off, int* __restrict__ big_size, int* __restrict__ big_fill,
                          int* __restrict__ big_members, int* __restrict__ big_bar, int* __restrict__ isl_order,
                          int* __restrict__ npair, int* __restrict__ nrest) {
  pdl_wait();  // programmatic dependent launch (sim_launch.h)
  pdl_trigger();
  extern __shared__ int slab[];
  __shared__ int changed, any_big;
  int* L = labels_in_smem ? slab : label;
  const int ne = min(*n_edges_p, edge_cap);
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    L[e] = e;
    merged[e] = 0;
  }
  if (threadIdx.x == 0) {
    any_big = 0;
    *big_count = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    merged[edges[i].x] = 1;
    merged[edges[i].y] = 1;
  }
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < ne; i += blockDim.x) {
      const int a = edges[i].x, b = edges[i].y;
      const int la = L[a], lb = L[b];
      if (la != lb) {
        const int m = min(la, lb);
        atomicMin(&L[a], m);
        atomicMin(&L[b], m);
        atomicMin(&L[max(la, lb)], m);
        changed = 1;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * ne; i += blockDim.x) {  // pointer jumping
      const int e = (i & 1) ? edges[i >> 1].y : edges[i >> 1].x;
      const int l = L[e], ll = L[l];
      if (ll < l) {
        atomicMin(&L[e], ll);
        changed = 1;
      }
    }
    __syncthreads();
    if (!changed) break;
  }
  // one record per island (root = its smallest env), then the sizes
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    if (merged[e] && L[e] == e) {
      const int i = atomicAdd(isl_count, 1);
      isl_of[e] = i;
      isl_size[i] = 0;
      isl_fill[i] = 0;
      isl_big[i] = -1;
      for (int k = 0; k < kIslandMax; ++k) isl_members[i * kIslandMax + k] = -1;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    if (merged[e]) atomicAdd(&isl_size[isl_of[L[e]]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    if (merged[e] && L[e] == e && isl_size[isl_of[e]] > cap) any_big = 1;
  __syncthreads();
  if (any_big && threadIdx.x == 0) {
    // islands larger than one CTA: records in root order (deterministic), as
    // long as their CTA parts fit the co-resident budget of the launch;
    // beyond it an island is stepped env by env and flagged (merged = 2)
    int nb = 0, off = 0, parts = 0;
    for (int e = 0; e < n; ++e) {
      if (!merged[e] || L[e] != e) continue;
      const int i = isl_of[e], m = isl_size[i];
      if (m <= cap) continue;
      const int p = (m + cap - 1) / cap;
      if (nb < kBigIslands && parts + p <= max_parts) {
        big_off[nb] = off;
        big_size[nb] = m;
        big_fill[nb] = 0;
        big_bar[nb] = 0;
        isl_big[i] = nb++;
        off += m;
        parts += p;
      } else {
        isl_big[i] = -2;
        atomicOr(err, 2);
      }
    }
    *big_count = nb;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    if (!merged[e]) continue;
    const int i = isl_of[L[e]];
    const int bi = isl_big[i];
    if (bi >= 0) {
      big_members[big_off[bi] + atomicAdd(&big_fill[bi], 1)] = e;
    } else if (bi == -2) {
      merged[e] = 2;
    } else {
      isl_members[i * kIslandMax + atomicAdd(&isl_fill[i], 1)] = e;
    }
  }
  // island order for the one-CTA launch: two-env islands first (four share
  // an island CTA), then the rest (big islands there have no members here)
  __syncthreads();
  const int nisl = *isl_count;
  for (int i = threadIdx.x; i < nisl; i += blockDim.x)
    if (isl_size[i] == 2 && isl_big[i] == -1) isl_order[atomicAdd(npair, 1)] = i;
  __syncthreads();
  const int np = *npair;
  for (int i = threadIdx.x; i < nisl; i += blockDim.x)
    if (!(isl_size[i] == 2 && isl_big[i] == -1)) isl_order[np + atomicAdd(nrest, 1)] = i;
}

__global__ void k_keys(const PairContact* __restrict__ c, const int* __restrict__ n_p, int cap,
                       unsigned long long* __restrict__ keys, int* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = min(*n_p, cap);
  if (i >= n) return;
  keys[i] = c[i].key;
  idx[i] = i;
}

}  // namespace

// Device scratch of the detection, owned by the sim handle (grown on demand).
struct PairScratch {
  size_t n_cap = 0, pair_cap = 0, c_cap = 0, tmp_bytes = 0;
  WShape* ws = nullptr;
  double* env_box = nullptr;
  int2* pairs = nullptr;
  int* counters = nullptr;  // [0] env pairs, [1] contacts
  PairContact* cont = nullptr;
  unsigned long long *ckey = nullptr, *sckey = nullptr;
  int *cidx = nullptr, *scidx = nullptr;
  void* tmp = nullptr;
  // hashed env grid
  unsigned hmask = 0;
  int2* env_cell = nullptr;
  int *bin_count = nullptr, *bins = nullptr, *ovf = nullptr, *gcnt = nullptr;  // gcnt: [0] overflow, [1] max extent
  // step path (prepare_islands)
  size_t isl_n = 0;
  XSlot* xslots = nullptr;
  int* xcount = nullptr;
  int2* edges = nullptr;
  int* icnt = nullptr;  // [0] edges, [1] islands, [2] error bits, [3] two-env islands, [4] the rest placed
  int *label = nullptr, *isl_of = nullptr, *isl_size = nullptr, *isl_members = nullptr;
  int *isl_fill = nullptr, *isl_big = nullptr, *isl_order = nullptr;
  uint8_t* merged = nullptr;
  // big islands: [0] count, then off / size / fill / barrier [kBigIslands] each
  int* big = nullptr;
  int* big_members = nullptr;
  void* big_xch = nullptr;  // [n][kBigStride] doubles (either precision fits)
};

void pair_scratch_free(PairScratch* p) {
  if (!p) return;
  for (void* q : {(void*)p->ws, (void*)p->env_box, (void*)p->pairs, (void*)p->counters, (void*)p->cont, (void*)p->ckey, (void*)p->sckey,
                  (void*)p->cidx, (void*)p->scidx, p->tmp, (void*)p->xslots, (void*)p->xcount, (void*)p->edges,
                  (void*)p->icnt, (void*)p->label, (void*)p->isl_of, (void*)p->isl_size, (void*)p->isl_members,
                  (void*)p->merged, (void*)p->env_cell, (void*)p->bin_count, (void*)p->bins, (void*)p->ovf,
                  (void*)p->gcnt, (void*)p->isl_fill, (void*)p->isl_big, (void*)p->isl_order, (void*)p->big,
                  (void*)p->big_members, p->big_xch})
    if (q) cudaFree(q);
  delete p;
}

// candidate env pairs (i < j, env AABBs overlapping within the margin) of the
// current state into P->pairs / P->counters[0]; world shapes into P->ws
template <class T>
static cudaError_t broadphase(PairScratch* P, const DevModel<T>* model, const T* state, const double* origin, int n,
                              int W, double margin, cudaStream_t st, int* xcount = nullptr, int* icnt = nullptr) {
  const int nbins = int(P->hmask + 1);
  cudaError_t e = launch_pdl(k_pairs_reset, dim3((nbins + 255) / 256), dim3(256), 0, st, P->bin_count, nbins, P->gcnt,
                             P->counters, icnt);
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_shapes_warp<T>, dim3((n * 32 + 127) / 128), dim3(128), 0, st, model, state, origin, n, W, P->ws,
                 P->env_box, P->env_cell, P->bin_count, P->bins, P->hmask, P->ovf, P->gcnt, P->gcnt + 1, xcount);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_env_query, dim3((n * 32 + 127) / 128), dim3(128), 0, st, n, (const double*)P->env_box,
                    (const int2*)P->env_cell, (const int*)P->bin_count, (const int*)P->bins, P->hmask,
                    (const int*)P->ovf, (const int*)P->gcnt, (const int*)(P->gcnt + 1), margin, P->pairs,
                    int(P->pair_cap), P->counters);
}

template <class T>
cudaError_t detect_pairs(PairScratch*& P, const DevModel<T>* model, int B, const T* state, const double* origin,
                         int n, int W, double margin, int cap_out, int* count, int32_t* body_a, int32_t* body_b,
                         double* point, double* normal, double* separation, bool* overflow, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
#define STP_CK(x)            \
  do {                       \
    e = (x);                 \
    if (e != cudaSuccess) return e; \
  } while (0)
  if (!P) P = new PairScratch();
  const size_t pair_cap = size_t(n) * 32 + 64, c_cap = size_t(n) * B * 4 + 64;
  if (P->n_cap < size_t(n) || P->pair_cap < pair_cap || P->c_cap < c_cap) {
    PairScratch* old = P;
    P = new PairScratch();
    pair_scratch_free(old);
    P->n_cap = n;
    P->pair_cap = pair_cap;
    P->c_cap = c_cap;
    STP_CK(cudaMalloc(&P->ws, sizeof(WShape) * size_t(n) * B));
    STP_CK(cudaMalloc(&P->env_box, sizeof(double) * 6 * n));
    STP_CK(cudaMalloc(&P->pairs, sizeof(int2) * pair_cap));
    STP_CK(cudaMalloc(&P->counters, sizeof(int) * 2));
    STP_CK(cudaMalloc(&P->cont, sizeof(PairContact) * c_cap));
    STP_CK(cudaMalloc(&P->ckey, sizeof(unsigned long long) * c_cap));
    STP_CK(cudaMalloc(&P->sckey, sizeof(unsigned long long) * c_cap));
    STP_CK(cudaMalloc(&P->cidx, sizeof(int) * c_cap));
    STP_CK(cudaMalloc(&P->scidx, sizeof(int) * c_cap));
    size_t t2 = 0;
    STP_CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, P->ckey, P->sckey, P->cidx, P->scidx, int(c_cap)));
    P->tmp_bytes = t2;
    STP_CK(cudaMalloc(&P->tmp, P->tmp_bytes));
    unsigned H = 1024;
    while (H < 2u * unsigned(n)) H <<= 1;
    P->hmask = H - 1;
    STP_CK(cudaMalloc(&P->env_cell, sizeof(int2) * n));
    STP_CK(cudaMalloc(&P->bin_count, sizeof(int) * H));
    STP_CK(cudaMalloc(&P->bins, sizeof(int) * H * kBinCap));
    STP_CK(cudaMalloc(&P->ovf, sizeof(int) * n));
    STP_CK(cudaMalloc(&P->gcnt, sizeof(int) * 2));
  }
  STP_CK(broadphase<T>(P, model, state, origin, n, W, margin, st));
  int h_cnt[2] = {0, 0};
  STP_CK(cudaMemcpyAsync(h_cnt, P->counters, sizeof(int), cudaMemcpyDeviceToHost, st));
  STP_CK(cudaStreamSynchronize(st));
  const int np = h_cnt[0] < int(pair_cap) ? h_cnt[0] : int(pair_cap);
  *overflow = h_cnt[0] > int(pair_cap);
  if (np > 0) {
    k_narrow<<<(np * 32 + 127) / 128, 128, 0, st>>>(P->pairs, P->counters, int(pair_cap), B, (long long)n * B, P->ws,
                                                    (const double*)P->env_box, margin, P->cont, int(c_cap),
                                                    P->counters + 1);
    STP_CK(cudaGetLastError());
  }
  STP_CK(cudaMemcpyAsync(h_cnt + 1, P->counters + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  STP_CK(cudaStreamSynchronize(st));
  const int nc = h_cnt[1] < int(c_cap) ? h_cnt[1] : int(c_cap);
  *overflow = *overflow || h_cnt[1] > int(c_cap);
  *count = nc;
  if (nc == 0) return cudaSuccess;
  k_keys<<<(nc + 127) / 128, 128, 0, st>>>(P->cont, P->counters + 1, int(c_cap), P->ckey, P->cidx);
  STP_CK(cudaGetLastError());
  size_t tb = P->tmp_bytes;
  STP_CK(cub::DeviceRadixSort::SortPairs(P->tmp, tb, P->ckey, P->sckey, P->cidx, P->scidx, nc, 0, 64, st));
  // gather to the host in key order
  std::vector<PairContact> hc(nc);
  std::vector<int> order(nc);
  STP_CK(cudaMemcpyAsync(hc.data(), P->cont, sizeof(PairContact) * nc, cudaMemcpyDeviceToHost, st));
  STP_CK(cudaMemcpyAsync(order.data(), P->scidx, sizeof(int) * nc, cudaMemcpyDeviceToHost, st));
  STP_CK(cudaStreamSynchronize(st));
  const unsigned long long NB = (unsigned long long)n * B;
  for (int i = 0; i < nc && i < cap_out; ++i) {
    const PairContact& c = hc[order[i]];
    if (body_a) body_a[i] = int32_t(c.key / NB);
    if (body_b) body_b[i] = int32_t(c.key % NB);
    for (int k = 0; k < 3; ++k) {
      if (point) point[3 * i + k] = c.point[k];
      if (normal) normal[3 * i + k] = c.normal[k];
    }
    if (separation) separation[i] = c.sep;
  }
  return cudaSuccess;
#undef STP_CK
}

// Device-only preparation of the step's inter-agent coupling: cross contact
// slots per body, env islands and the merged flags (no host round trip).
template <class T>
cudaError_t prepare_islands(PairScratch*& P, const DevModel<T>* model, int B, const T* state, const double* origin,
                            int n, int W, double margin, int cap, int max_parts, IslandView* view,
                            cudaStream_t st) {
  cudaError_t e = cudaSuccess;
#define STP_CK(x)                   \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) return e; \
  } while (0)
  if (!P) P = new PairScratch();
  const size_t pair_cap = size_t(n) * 32 + 64;
  if (P->n_cap < size_t(n) || P->pair_cap < pair_cap) {
    // (re)build the detection scratch through the detection entry's allocator
    int cnt = 0;
    bool ov = false;
    STP_CK(detect_pairs<T>(P, model, B, state, origin, n, W, margin, 0, &cnt, nullptr, nullptr, nullptr, nullptr,
                           nullptr, &ov, st));
  }
  if (P->isl_n < size_t(n)) {
    for (void* q : {(void*)P->xslots, (void*)P->xcount, (void*)P->edges, (void*)P->icnt, (void*)P->label,
                    (void*)P->isl_of, (void*)P->isl_size, (void*)P->isl_members, (void*)P->merged,
                    (void*)P->isl_fill, (void*)P->isl_big, (void*)P->isl_order, (void*)P->big, (void*)P->big_members,
                    P->big_xch})
      if (q) cudaFree(q);
    P->isl_n = n;
    STP_CK(cudaMalloc(&P->xslots, sizeof(XSlot) * size_t(n) * B * kXSlots));
    STP_CK(cudaMalloc(&P->xcount, sizeof(int) * size_t(n) * B));
    STP_CK(cudaMalloc(&P->edges, sizeof(int2) * size_t(n) * B * kXSlots));
    STP_CK(cudaMalloc(&P->icnt, sizeof(int) * 5));
    STP_CK(cudaMalloc(&P->label, sizeof(int) * n));
    STP_CK(cudaMalloc(&P->isl_of, sizeof(int) * n));
    STP_CK(cudaMalloc(&P->isl_size, sizeof(int) * (n / 2 + 1)));
    STP_CK(cudaMalloc(&P->isl_members, sizeof(int) * (n / 2 + 1) * kIslandMax));
    STP_CK(cudaMalloc(&P->merged, n));
    STP_CK(cudaMalloc(&P->isl_fill, sizeof(int) * (n / 2 + 1)));
    STP_CK(cudaMalloc(&P->isl_big, sizeof(int) * (n / 2 + 1)));
    STP_CK(cudaMalloc(&P->isl_order, sizeof(int) * (n / 2 + 1)));
    STP_CK(cudaMalloc(&P->big, sizeof(int) * (1 + 4 * kBigIslands)));
    STP_CK(cudaMalloc(&P->big_members, sizeof(int) * n));
    STP_CK(cudaMalloc(&P->big_xch, sizeof(double) * kBigStride * size_t(n)));
  }
  const int edge_cap = n * B * kXSlots;
  STP_CK(broadphase<T>(P, model, state, origin, n, W, margin, st, P->xcount, P->icnt));
  STP_CK(launch_pdl(k_narrow_slots, dim3(148 * 2), dim3(256), 0, st, P->pairs, P->counters, int(P->pair_cap), B,
                    (long long)n * B, P->ws, (const double*)P->env_box, margin, P->xslots, P->xcount, P->edges,
                    edge_cap, P->icnt, P->icnt + 2));
  // labels in shared memory up to 48K envs (192 KB), else in global scratch
  const size_t lab_bytes = size_t(n) * sizeof(int);
  const bool lab_smem = lab_bytes <= 192 * 1024;
  static bool lab_attr[64] = {};  // per device
  if (lab_smem && lab_bytes > 48 * 1024 && first_on_device(lab_attr))
    STP_CK(cudaFuncSetAttribute(k_islands, cudaFuncAttributeMaxDynamicSharedMemorySize, int(192 * 1024)));
  int* bg = P->big;
  STP_CK(launch_pdl(k_islands, dim3(1), dim3(1024), lab_smem ? lab_bytes : 0, st, n, P->edges, P->icnt, edge_cap,
                    P->label, P->merged, P->isl_of, P->isl_size, P->isl_fill, P->isl_big, P->isl_members,
                    P->icnt + 1, P->icnt + 2, int(lab_smem), cap, max_parts, bg, bg + 1, bg + 1 + kBigIslands,
                    bg + 1 + 2 * kBigIslands, P->big_members, bg + 1 + 3 * kBigIslands, P->isl_order, P->icnt + 3,
                    P->icnt + 4));
  view->merged = P->merged;
  view->isl_members = P->isl_members;
  view->isl_count = P->icnt + 1;
  view->isl_order = P->isl_order;
  view->isl_npair = P->icnt + 3;
  view->err = P->icnt + 2;
  view->xslots = P->xslots;
  view->xcount = P->xcount;
  view->big_count = bg;
  view->big_off = bg + 1;
  view->big_size = bg + 1 + kBigIslands;
  view->big_members = P->big_members;
  view->big_bar = bg + 1 + 3 * kBigIslands;
  view->big_xch = P->big_xch;
  return cudaSuccess;
#undef STP_CK
}

template cudaError_t prepare_islands<float>(PairScratch*&, const DevModel<float>*, int, const float*, const double*,
                                            int, int, double, int, int, IslandView*, cudaStream_t);
template cudaError_t prepare_islands<double>(PairScratch*&, const DevModel<double>*, int, const double*,
                                             const double*, int, int, double, int, int, IslandView*, cudaStream_t);

template cudaError_t detect_pairs<float>(PairScratch*&, const DevModel<float>*, int, const float*, const double*, int,
                                         int, double, int, int*, int32_t*, int32_t*, double*, double*, double*, bool*,
                                         cudaStream_t);
template cudaError_t detect_pairs<double>(PairScratch*&, const DevModel<double>*, int, const double*, const double*,
                                          int, int, double, int, int*, int32_t*, int32_t*, double*, double*, double*,
                                          bool*, cudaStream_t);

}  // namespace stp
