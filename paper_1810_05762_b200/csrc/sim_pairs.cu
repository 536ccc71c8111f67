// Inter-agent contact detection: the dynamic-pair part of
// detect_contacts (collide.cpp:300-343) for every env of a sim, on the GPU.
//
// The reference bins margin-expanded body AABBs into a hash grid and then
// keeps the pairs (a < b) of different agents whose AABBs overlap within the
// margin (aabb_overlap, :80-84), sorted by (a, b), one segment-segment contact
// each (closest_segment_segment :219-249, collide_dynamic_pair :251-266).  The
// grid is only a broadphase: any overlapping pair shares a cell, so the pair
// set is exactly "different agents, overlapping AABBs".  Here:
//   K_a  per env: world shapes of its bodies in double (env origin + local
//        pose, world_shape :38-78) and the env's AABB (union);
//   sort envs by AABB x-min (cub radix sort), then
//   K_b  sweep: each env scans the envs after it in x order while their x-min
//        is within reach and keeps the pairs whose env AABBs overlap;
//   K_c  one warp per candidate env pair: all body pairs, the reference's AABB
//        test and narrow phase, emitted with key (a, b);
//   sort contacts by key (cub) -> the reference's order.
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
  double r;
  int ok;  // dynamic sphere / capsule (boxes never pair, :255)
};

template <class T>
__global__ void k_world_shapes(const DevModel<T>* __restrict__ Mp, const T* __restrict__ state,
                               const double* __restrict__ origin, int n, int W, double margin, WShape* __restrict__ ws,
                               double* __restrict__ env_box, float* __restrict__ key, int* __restrict__ idx) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const DevModel<T>& M = *Mp;
  const int B = M.nb;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int b = 0; b < B; ++b) {
    WShape s{};
    const size_t sb = size_t(e) * kStateFields * W + b;
    auto st = [&](int f) { return double(state[sb + size_t(f) * W]); };
    const v3<double> x{st(0) + origin[2 * e], st(1) + origin[2 * e + 1], st(2)};
    const qt<double> q{st(3), st(4), st(5), st(6)};
    const qt<double> lr{double(M.lrot[0][b]), double(M.lrot[1][b]), double(M.lrot[2][b]), double(M.lrot[3][b])};
    const v3<double> lp{double(M.lpos[0][b]), double(M.lpos[1][b]), double(M.lpos[2][b])};
    const qt<double> rot = qmul(q, lr);
    const v3<double> pos = x + qrot(q, lp);
    const double r = double(M.radius[b]);
    v3<double> p0 = pos, p1 = pos;
    if (M.shape[b] == STP_CAPSULE) {
      const v3<double> ax = qrot(rot, v3<double>{0.0, 0.0, double(M.half_len[b])});
      p0 = pos - ax;
      p1 = pos + ax;
    }
    s.ok = !M.is_static[b] && M.shape[b] != STP_BOX;
    s.r = r;
    const double a0[3] = {p0.x, p0.y, p0.z}, a1[3] = {p1.x, p1.y, p1.z};
    for (int k = 0; k < 3; ++k) {
      s.p0[k] = a0[k];
      s.p1[k] = a1[k];
      s.lo[k] = fmin(a0[k], a1[k]) - r;
      s.hi[k] = fmax(a0[k], a1[k]) + r;
      if (s.ok) {
        lo[k] = fmin(lo[k], s.lo[k]);
        hi[k] = fmax(hi[k], s.hi[k]);
      }
    }
    ws[size_t(e) * B + b] = s;
  }
  for (int k = 0; k < 3; ++k) {
    env_box[6 * e + k] = lo[k];
    env_box[6 * e + 3 + k] = hi[k];
  }
  // sort key: x-min rounded down to float (a conservative lower bound)
  float kx = __double2float_rd(lo[0] - margin);
  if (!(lo[0] <= hi[0])) kx = INFINITY;  // no dynamic sphere/capsule body
  key[e] = kx;
  idx[e] = e;
}

__device__ __forceinline__ bool box_overlap(const double* a, const double* b, double m) {
  // a, b: lo[3], hi[3]; the reference's aabb_overlap with margin m
  return a[0] <= b[3] + m && b[0] <= a[3] + m && a[1] <= b[4] + m && b[1] <= a[4] + m && a[2] <= b[5] + m &&
         b[2] <= a[5] + m;
}

__global__ void k_env_pairs(int n, const float* __restrict__ skey, const int* __restrict__ sidx,
                            const double* __restrict__ env_box, double margin, int2* __restrict__ pairs, int cap,
                            int* __restrict__ n_pairs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int i = sidx[p];
  const double* bi = env_box + 6 * i;
  if (!(bi[0] <= bi[3])) return;
  const double reach = bi[3] + 2.0 * margin;  // x-min of a partner is <= hi.x + margin (key carries -margin)
  for (int q = p + 1; q < n; ++q) {
    if (double(skey[q]) > reach) break;
    const int j = sidx[q];
    if (box_overlap(bi, env_box + 6 * j, margin)) {
      const int slot = atomicAdd(n_pairs, 1);
      if (slot < cap) pairs[slot] = make_int2(min(i, j), max(i, j));
    }
  }
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
__global__ void k_narrow(const int2* __restrict__ pairs, const int* __restrict__ n_pairs_p, int pair_cap, int B,
                         long long NB, const WShape* __restrict__ ws, double margin, PairContact* __restrict__ out,
                         int cap, int* __restrict__ n_out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int np = min(*n_pairs_p, pair_cap);
  if (warp >= np) return;
  const int2 pr = pairs[warp];
  for (int u = lane; u < B * B; u += 32) {
    const int ba = u / B, bb = u % B;
    const WShape& A = ws[size_t(pr.x) * B + ba];
    const WShape& Bs = ws[size_t(pr.y) * B + bb];
    if (!A.ok || !Bs.ok) continue;
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
  float *key = nullptr, *skey = nullptr;
  int *idx = nullptr, *sidx = nullptr;
  int2* pairs = nullptr;
  int* counters = nullptr;  // [0] env pairs, [1] contacts
  PairContact* cont = nullptr;
  unsigned long long *ckey = nullptr, *sckey = nullptr;
  int *cidx = nullptr, *scidx = nullptr;
  void* tmp = nullptr;
};

void pair_scratch_free(PairScratch* p) {
  if (!p) return;
  for (void* q : {(void*)p->ws, (void*)p->env_box, (void*)p->key, (void*)p->skey, (void*)p->idx, (void*)p->sidx,
                  (void*)p->pairs, (void*)p->counters, (void*)p->cont, (void*)p->ckey, (void*)p->sckey,
                  (void*)p->cidx, (void*)p->scidx, p->tmp})
    if (q) cudaFree(q);
  delete p;
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
    STP_CK(cudaMalloc(&P->key, sizeof(float) * n));
    STP_CK(cudaMalloc(&P->skey, sizeof(float) * n));
    STP_CK(cudaMalloc(&P->idx, sizeof(int) * n));
    STP_CK(cudaMalloc(&P->sidx, sizeof(int) * n));
    STP_CK(cudaMalloc(&P->pairs, sizeof(int2) * pair_cap));
    STP_CK(cudaMalloc(&P->counters, sizeof(int) * 2));
    STP_CK(cudaMalloc(&P->cont, sizeof(PairContact) * c_cap));
    STP_CK(cudaMalloc(&P->ckey, sizeof(unsigned long long) * c_cap));
    STP_CK(cudaMalloc(&P->sckey, sizeof(unsigned long long) * c_cap));
    STP_CK(cudaMalloc(&P->cidx, sizeof(int) * c_cap));
    STP_CK(cudaMalloc(&P->scidx, sizeof(int) * c_cap));
    size_t t1 = 0, t2 = 0;
    STP_CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, P->key, P->skey, P->idx, P->sidx, n));
    STP_CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, P->ckey, P->sckey, P->cidx, P->scidx, int(c_cap)));
    P->tmp_bytes = t1 > t2 ? t1 : t2;
    STP_CK(cudaMalloc(&P->tmp, P->tmp_bytes));
  }
  STP_CK(cudaMemsetAsync(P->counters, 0, sizeof(int) * 2, st));
  k_world_shapes<T><<<(n + 127) / 128, 128, 0, st>>>(model, state, origin, n, W, margin, P->ws, P->env_box, P->key,
                                                     P->idx);
  STP_CK(cudaGetLastError());
  size_t tb = P->tmp_bytes;
  STP_CK(cub::DeviceRadixSort::SortPairs(P->tmp, tb, P->key, P->skey, P->idx, P->sidx, n, 0, 32, st));
  k_env_pairs<<<(n + 127) / 128, 128, 0, st>>>(n, P->skey, P->sidx, P->env_box, margin, P->pairs, int(pair_cap),
                                               P->counters);
  STP_CK(cudaGetLastError());
  int h_cnt[2] = {0, 0};
  STP_CK(cudaMemcpyAsync(h_cnt, P->counters, sizeof(int), cudaMemcpyDeviceToHost, st));
  STP_CK(cudaStreamSynchronize(st));
  const int np = h_cnt[0] < int(pair_cap) ? h_cnt[0] : int(pair_cap);
  *overflow = h_cnt[0] > int(pair_cap);
  if (np > 0) {
    k_narrow<<<(np * 32 + 127) / 128, 128, 0, st>>>(P->pairs, P->counters, int(pair_cap), B, (long long)n * B, P->ws,
                                                    margin, P->cont, int(c_cap), P->counters + 1);
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
  tb = P->tmp_bytes;
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

template cudaError_t detect_pairs<float>(PairScratch*&, const DevModel<float>*, int, const float*, const double*, int,
                                         int, double, int, int*, int32_t*, int32_t*, double*, double*, double*, bool*,
                                         cudaStream_t);
template cudaError_t detect_pairs<double>(PairScratch*&, const DevModel<double>*, int, const double*, const double*,
                                          int, int, double, int, int*, int32_t*, int32_t*, double*, double*, double*,
                                          bool*, cudaStream_t);

}  // namespace stp
