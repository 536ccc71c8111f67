// The fused B200 environment-step kernel.
//
// One warp segment of W lanes = one environment; lane b = body b.  A single
// launch performs, per env:
//   K1  speculative contacts vs plane / terrain boxes     (collide.cpp:270-299)
//   K2  actuation, body dynamics, constraint rows, 4 x (assembly + PCR),
//       impulse report, integration, rollback             (solver.cpp:395-597,
//                                                          krylov.cpp:106-174)
//   K3  task epilogue: reward, termination, flagrun, perturbation schedule,
//       auto-reset via hinge FK, observation
// so the body state is read from HBM once and written once per step.
//
// The system matrix is never materialised in HBM (see sim_step.cuh for the
// per-lane block layout and the split block-Jacobi PCR).  Dot products are
// segment reductions over warp shuffles.
#pragma once

#include <type_traits>

#include "sim_device.cuh"
#include "stp_rng.h"

namespace stp {

constexpr int kCData = 11;  // recorded contact: point3 normal3 sep pn pt3 (double)

// One inter-agent contact seen from one of its bodies (collide.cpp:251-266,
// rows solver.cpp:176-210): the reference's row Jacobians are
// j_own = role * (n, r_own x n), j_partner = -role * (n, r_partner x n)
// (role +1: this body is body_a, -1: body_b), likewise for the tangents.
struct XSlot {
  long long key;  // a * (n * B) + b: the contact's place in the reference's (a, b) order
  int partner;    // global body index (env * B + body) of the other body
  int role;       // +1 body_a, -1 body_b
  double r_own[3], r_part[3];  // contact point minus each body's position (pre-step)
  double normal[3];            // from body_b to body_a
  double sep;
};
constexpr int kXSlots = 4;      // cross contacts per body
constexpr int kIslandMax = 8;   // envs per merged island of the one-CTA launch (one warp each)
constexpr int kBigIslands = 64; // islands larger than that per step (multi-CTA launch)

template <class T>
struct KArgs {
  const DevModel<T>* model;
  DevCfg<T> cfg;
  DevTask task;
  int n;        // envs [e_begin, n) are stepped by this launch
  int e_begin;  // first env (host-buffer pipelining launches env chunks)
  int mode;  // 0 = physics::step, 1 = env_step, 2 = reset
  uint64_t seed;
  long long env_offset;
  T* state;        // [n][16][W]
  double* origin;  // [n][2]
  T* loads;        // [n][6][W] or null
  const float* torques;  // mode 0: [n][J] (N*m)
  const float* actions;  // mode 1: [n][J] (normalised)
  float* obs;
  float* reward;
  uint8_t* done;
  int obs_dim;
  int32_t* counters;  // [n][8]
  T* target;          // [n][2], relative to origin
  T* last_tau;        // [n][J]
  uint32_t* feet;     // [n] feet-contact bits of the last env step
  const uint8_t* reset_mask;
  int32_t* newton_out;
  int32_t* krylov_out;
  uint8_t* failed_out;
  uint8_t* overflow_out;
  int record;
  int cap;
  int32_t* c_count;   // [n]
  int32_t* c_body;    // [n][cap]
  double* c_data;     // [n][cap][11]
  int n_boxes;
  const double* boxes;  // [nbox][8]: cx cy cz hx hy hz cos(yaw) sin(yaw)
  T* scratch;           // [n][34][W] rarely used per-lane rows (sim_step.cuh G_*)
  // uniform grid over the boxes' loose xy footprints (stp_set_terrain)
  int grid_nx, grid_ny;
  double grid_x0, grid_y0, grid_inv;
  const int* cell_start;  // [nx*ny + 1]
  const int* cell_list;   // box indices, ascending within a cell
  const int4* box_cells;  // per box: first/last cell (x0, y0, x1, y1)
  // inter-agent contacts (Scene::inter_agent_collisions): envs
  // linked by one are stepped together by the island launch (sim_pairs.cu)
  const uint8_t* merged;      // [n] 1: env belongs to a contact-merged island
  const int* isl_members;     // [n / 2][kIslandMax] member envs (unordered; -1 unused)
  const int* isl_count;       // number of merged islands
  const int* isl_order;       // island indices: the two-env islands first ([0, *isl_npair)), then the rest
  const int* isl_npair;       // number of two-env islands (packed four per island CTA)
  const XSlot* xslots;        // [n * B][kXSlots] cross contacts of each body
  const int* xcount;          // [n * B]
  const int* isl_err;         // preparation overflow bits (see IslandView)
  // islands larger than one CTA's warps (multi-CTA launch, sim_pairs.cu
  // k_islands): CTA c of the launch takes part p of big island i; the
  // island's warps exchange through a global area and a global barrier
  int isl_big_mode;           // 0: one CTA per island (isl_members), 1: big islands
  const int* big_count;       // number of big islands this step
  const int* big_off;         // [kBigIslands] first member in big_members
  const int* big_size;        // [kBigIslands] member count
  const int* big_members;     // member envs (unordered within an island)
  int* big_bar;               // [kBigIslands] barrier arrival counters (zeroed per step)
  T* big_xch;                 // [sum of sizes][kBigStride] exchange / reduction area
  // assemble_system hook (stp_debug_first_system): env dbg_env writes its first
  // Newton linearisation per lane [kDbgStride] and its Krylov count per Newton
  T* dbg;
  int dbg_env;
};
// per lane: H_bb (21, packed), rhs (6), H(child, parent) (36, row-major incl.
// the active limit term), aliasing quirk d0, ja angular (3), jb angular (3);
// then kDbgNewton Krylov counts at 32 * kDbgStride
constexpr int kDbgStride = 21 + 6 + 36 + 7;
constexpr int kDbgNewton = 64;
// per-env entries of the big islands' global exchange area: 32 lanes x kXch,
// 4 reduction partials, 1 vote
constexpr int kXchEntries = 21;
constexpr int kBigStride = 32 * kXchEntries + 5;

enum { C_FRAME = 0, C_FLAG = 1, C_FALL = 2, C_NEXTP = 3, C_EPISODE = 4, C_FLAGDRAW = 5, C_PERTDRAW = 6 };
constexpr int kGridCols = 64;

template <int W, class T>
__device__ __forceinline__ T seg_sum(T v, unsigned mask) {
#pragma unroll
  for (int off = W / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off, W);
  return v;
}
template <int W, class T>
__device__ __forceinline__ T from(T v, int src, unsigned mask) {
  return __shfl_sync(mask, v, src, W);
}
template <int W, class T>
__device__ __forceinline__ v3<T> from(v3<T> v, int src, unsigned mask) {
  return {__shfl_sync(mask, v.x, src, W), __shfl_sync(mask, v.y, src, W), __shfl_sync(mask, v.z, src, W)};
}
template <int W, class T>
__device__ __forceinline__ qt<T> from(qt<T> v, int src, unsigned mask) {
  return {__shfl_sync(mask, v.w, src, W), __shfl_sync(mask, v.x, src, W), __shfl_sync(mask, v.y, src, W),
          __shfl_sync(mask, v.z, src, W)};
}

// packed symmetric 6x6 rank-1 update H += d j j^T (assemble, solver.cpp:337-338)
template <class T>
__device__ __forceinline__ void sym_add(T (&H)[21], const T (&j)[6], T d) {
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    const T dj = d * j[r];
#pragma unroll
    for (int c = 0; c <= r; ++c) H[tri(r, c)] += dj * j[c];
  }
}

// 6-term dot product as a depth-4 tree (shorter dependency chain than the
// reference's left-to-right sum; same value up to rounding)
template <class T>
__device__ __forceinline__ T dot6(const T (&a)[6], const T (&b)[6]) {
  return ((a[0] * b[0] + a[1] * b[1]) + (a[2] * b[2] + a[3] * b[3])) + (a[4] * b[4] + a[5] * b[5]);
}

// unilateral_bias, solver.cpp:84-87
template <class T>
__device__ __forceinline__ T uni_bias(T gap, T beta, T dt) {
  return gap < T(0) ? -(beta / dt) * gap : -gap / dt;
}

// friction_weight, solver.cpp:267-270
template <class T>
__device__ __forceinline__ T fric_weight(T pn, T vt, T eps) {
  const T s = vt / eps;
  return pn / (eps * sqrt(T(1) + s * s));  // mu = 1 (collide.cpp:25)
}

// Body inertia quadratic form a^T Iinv a + inv_m |l|^2 for one side of a row.
template <class T>
__device__ __forceinline__ T quad(const sym3<T>& Iinv, v3<T> a) {
  return dot(a, smul(Iinv, a));
}

// joint_angle, solver.cpp:405-411
template <class T>
__device__ __forceinline__ T hinge_angle(qt<T> qp, qt<T> qc, qt<T> rest, v3<T> axc) {
  const qt<T> rel = qmul(qconj(qp), qc);
  qt<T> d = qmul(qconj(rest), rel);
  if (d.w < T(0)) d = qt<T>{-d.w, -d.x, -d.y, -d.z};
  const T proj = d.x * axc.x + d.y * axc.y + d.z * axc.z;
  return T(2) * atan2(proj, d.w);
}

template <class T>
__device__ __forceinline__ v3<T> ldv(const T (&a)[3][32], int b) {
  return {a[0][b], a[1][b], a[2][b]};
}

// ---------------------------------------------------------------------------
// Environment reset via hinge forward kinematics (the FK
// convention reproduces joint_angle, solver.cpp:405-411, at the drawn angle).
// All lanes of the segment call it; depth levels are resolved in order.
// ---------------------------------------------------------------------------
template <class T, int W>
__device__ void reset_env(const KArgs<T>& a, const DevModel<T>& M, int e, int b, unsigned mask, bool act,
                          v3<T>& x, qt<T>& q, v3<T>& v, v3<T>& w, int32_t (&cnt)[8], T& tx, T& ty, double& ox,
                          double& oy) {
  const uint64_t genv = uint64_t(a.env_offset + e);
  const uint64_t s = stp_derive_seed(a.seed, STP_TAG_RESET, (genv << 32) | uint32_t(cnt[C_EPISODE]));
  cnt[C_EPISODE] += 1;
  const double amp = a.task.reset_noise;
  const int J = M.nj;
  auto noise = [&](uint32_t k) { return amp * (2.0 * stp_uniform(s, k) - 1.0); };
  ox = double(genv % kGridCols) * a.task.spacing;
  oy = double(genv / kGridCols) * a.task.spacing;
  const int r = M.root;
  if (b == r) {
    x = {T(double(M.rest_state[0][b]) + noise(0)), T(double(M.rest_state[1][b]) + noise(1)),
         T(double(M.rest_state[2][b]) + noise(2))};
    const v3<T> rv{T(noise(3)), T(noise(4)), T(noise(5))};
    const qt<T> rq{M.rest_state[3][b], M.rest_state[4][b], M.rest_state[5][b], M.rest_state[6][b]};
    q = qunit(qmul(qexp(rv), rq));
    v = {T(noise(6 + J)), T(noise(7 + J)), T(noise(8 + J))};
    w = {T(noise(9 + J)), T(noise(10 + J)), T(noise(11 + J))};
  } else if (act) {
    // static bodies keep their rest pose; dynamic ones are set by FK below
    x = {M.rest_state[0][b], M.rest_state[1][b], M.rest_state[2][b]};
    q = {M.rest_state[3][b], M.rest_state[4][b], M.rest_state[5][b], M.rest_state[6][b]};
    v = {0, 0, 0};
    w = {0, 0, 0};
  }
  const int jn = act ? M.joint[b] : -1;
  const int par = act && M.parent[b] >= 0 ? M.parent[b] : b;
  const int my_depth = act ? M.depth[b] : -1;
  for (int d = 1; d <= M.max_depth; ++d) {
    const v3<T> xp = from<W>(x, par, mask);
    const qt<T> qp = from<W>(q, par, mask);
    const v3<T> vp = from<W>(v, par, mask);
    const v3<T> wp = from<W>(w, par, mask);
    if (my_depth == d && jn >= 0 && !M.is_static[b]) {
      const T th = T(noise(6 + jn));
      const T thd = T(noise(12 + J + jn));
      const v3<T> axc = ldv(M.ax_c, b);
      const qt<T> rest{M.rest[0][b], M.rest[1][b], M.rest[2][b], M.rest[3][b]};
      // Quat::from_axis_angle, vec.hpp:130-135
      T sh, ch;
      sincos_(T(0.5) * th, &sh, &ch);
      const v3<T> au = vunit(axc);
      const qt<T> aa{ch, au.x * sh, au.y * sh, au.z * sh};
      q = qmul(qmul(qp, rest), aa);
      const v3<T> anchor = xp + qrot(qp, ldv(M.anc_p, b));
      x = anchor - qrot(q, ldv(M.anc_c, b));
      w = wp + qrot(q, axc) * thd;
      v = vp + cross(wp, anchor - xp) - cross(w, anchor - x);
    }
  }
  cnt[C_FRAME] = 0;
  cnt[C_FLAG] = 0;
  cnt[C_FALL] = 0;
  const v3<T> xr = from<W>(x, r, mask);
  if (a.task.target_refresh > 0) {
    const uint64_t fs = stp_derive_seed(a.seed, STP_TAG_FLAG, (genv << 32) | uint32_t(cnt[C_FLAGDRAW]));
    cnt[C_FLAGDRAW] += 1;
    const double rad = a.task.target_radius * sqrt(stp_uniform(fs, 0));
    const double phi = 2.0 * M_PI * stp_uniform(fs, 1);
    tx = T(double(xr.x) + rad * cos(phi));
    ty = T(double(xr.y) + rad * sin(phi));
  } else {
    tx = xr.x + T(1000);
    ty = xr.y;
  }
  if (a.task.perturb_max > 0 && a.task.perturb_max >= a.task.perturb_min) {
    const uint64_t ps = stp_derive_seed(a.seed, STP_TAG_PERTURB, (genv << 32) | uint32_t(cnt[C_PERTDRAW]));
    const int span = a.task.perturb_max - a.task.perturb_min + 1;
    int k = int(floor(stp_uniform(ps, 0) * span));
    if (k >= span) k = span - 1;
    cnt[C_NEXTP] = a.task.perturb_min + k;
  } else {
    cnt[C_NEXTP] = -1;
  }
}

// terrain_height over the box list, relative to the env origin
// (collide.cpp:348-359); boxes in double world coordinates.
__device__ __forceinline__ double terrain_height_dev(const double* boxes, int n, double x, double y) {
  double h = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* bx = boxes + 8 * i;
    const double dx = x - bx[0], dy = y - bx[1];
    const double lx = bx[6] * dx + bx[7] * dy;
    const double ly = -bx[7] * dx + bx[6] * dy;
    if (fabs(lx) <= bx[3] && fabs(ly) <= bx[4]) h = fmax(h, bx[2] + bx[5]);
  }
  return h;
}

// terrain_height through the grid: the box footprints covering (x, y)
// are all registered in the cell containing it.
template <class T>
__device__ __forceinline__ double terrain_height_grid(const KArgs<T>& a, double x, double y) {
  if (a.grid_nx <= 0) return terrain_height_dev(a.boxes, a.n_boxes, x, y);
  const int cx = int(floor((x - a.grid_x0) * a.grid_inv)), cy = int(floor((y - a.grid_y0) * a.grid_inv));
  if (cx < 0 || cy < 0 || cx >= a.grid_nx || cy >= a.grid_ny) return 0.0;
  const int c = cy * a.grid_nx + cx;
  double h = 0.0;
  for (int k = a.cell_start[c]; k < a.cell_start[c + 1]; ++k) {
    const double* bx = a.boxes + 8 * a.cell_list[k];
    const double dx = x - bx[0], dy = y - bx[1];
    const double lx = bx[6] * dx + bx[7] * dy;
    const double ly = -bx[7] * dx + bx[6] * dy;
    if (fabs(lx) <= bx[3] && fabs(ly) <= bx[4]) h = fmax(h, bx[2] + bx[5]);
  }
  return h;
}

// geometric height-map offsets (ratio 1.3 from 0.2 m)
// 0.2 (1.3^a - 1) / 0.3 for a = 0..7, evaluated once on the host with libm
// (the oracle's std::pow) and written as exact binary literals: no per-sample
// double pow in the kernel.
__device__ __forceinline__ double geo_offset(int k) {
  const int a = k < 0 ? -k : k;
  double d;
  switch (a) {
    case 0: d = 0x0p+0; break;
    case 1: d = 0x1.999999999999bp-3; break;
    case 2: d = 0x1.d70a3d70a3d73p-2; break;
    case 3: d = 0x1.989374bc6a7f1p-1; break;
    case 4: d = 0x1.3cc63f141205ep+0; break;
    case 5: d = 0x1.cf01b866e43adp+0; break;
    case 6: d = 0x1.468deb0fadf31p+1; break;
    default: d = 0x1.c21ee4c795559p+1; break;
  }
  return k < 0 ? -d : d;
}

}  // namespace stp
