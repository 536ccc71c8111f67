// Device-side data structures and small-vector math of the B200 stepper.
//
// Layout decisions (DESIGN.md §"HBM layout"):
//  * one environment = one segment of W lanes of a warp (W = 32 for the
//    22-body Humanoid, 16 for the 9-body Ant, 8 for tiny test scenes);
//    lane b of the segment owns body b;
//  * body state is SoA per env: state[((e * 16) + field) * W + lane] so a
//    segment reads each field with one coalesced transaction;
//  * positions are stored relative to a per-env origin (double xy) that is
//    re-centred on the root every step, so fp32 keeps ~1e-7 m resolution
//    anywhere in a 200 m env grid (the reference is double everywhere).
#pragma once

#include <stdint.h>

#include "stampede_sim.h"

namespace stp {

constexpr int kStateFields = 16;  // 13 used: x3 q4 v3 w3 (+3 pad)
constexpr int kTaskCounters = 8;

// Per-body / per-joint model constants, indexed by body lane.  The joint
// fields describe the hinge whose child is that body (tree: at most one).
template <class T>
struct DevModel {
  int nb, nj, root, feet_mask, n_feet;
  int feet[STP_MAX_FEET];
  int shape[32], is_static[32], parent[32], joint[32], child_mask[32], depth[32], quirk[32];
  int max_depth;
  int child_list[4][32];  // up to 4 child bodies per body (-1 = none)
  int max_children;
  // shuffle schedule of the child -> parent sum in the PCR matvec (host-built,
  // sim_host.cu gather_schedule): per round a source lane and two 0/1 weights,
  // into the receiver's y (parent sum) or its own t (sibling pre-accumulation)
  int gather_rounds;
  int gather_has_t[4];
  int gather_src[4][32];
  T gather_wy[4][32], gather_wt[4][32];
  int lane_of_joint[STP_MAX_JOINTS];
  T radius[32], half_len[32], hext[3][32], lpos[3][32], lrot[4][32];
  T mass[32], inv_mass[32], inertia[3][32], inv_inertia[3][32];
  T anc_p[3][32], anc_c[3][32], ax_p[3][32], ax_c[3][32], rest[4][32];
  T lim_lo[32], lim_hi[32], tmax[32];
  T rest_state[13][32];
  T fall_height, alive_bonus;
};

// Scalar physics parameters (StepConfig, types.hpp:92-107).
template <class T>
struct DevCfg {
  T dt, tol, margin, beta, kj, kc, kl, epsf, lim_act;
  T gx, gy, gz;
  int newton, kmax, plane;
};

struct DevTask {
  int kind, episode_cap, fall_grace, target_refresh;
  double target_radius, target_tolerance, spacing;
  int perturb_min, perturb_max;
  double force_lo, force_hi, reset_noise;
  int auto_reset, height_map;
};

// ---------------------------------------------------------------------------
// small vector math (restating vec.hpp:21-190 for device use)
// ---------------------------------------------------------------------------
template <class T>
struct v3 {
  T x, y, z;
};
template <class T>
struct qt {
  T w, x, y, z;
};

template <class T> __device__ __forceinline__ v3<T> mk(T a, T b, T c) { return {a, b, c}; }
template <class T> __device__ __forceinline__ v3<T> operator+(v3<T> a, v3<T> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class T> __device__ __forceinline__ v3<T> operator-(v3<T> a, v3<T> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class T> __device__ __forceinline__ v3<T> operator-(v3<T> a) { return {-a.x, -a.y, -a.z}; }
template <class T> __device__ __forceinline__ v3<T> operator*(v3<T> a, T s) { return {a.x * s, a.y * s, a.z * s}; }
template <class T> __device__ __forceinline__ T dot(v3<T> a, v3<T> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class T> __device__ __forceinline__ v3<T> cross(v3<T> a, v3<T> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class T> __device__ __forceinline__ T vnorm(v3<T> a) { return sqrt(dot(a, a)); }
template <class T> __device__ __forceinline__ v3<T> vunit(v3<T> a) {  // vec.hpp:42-45
  const T n = vnorm(a);
  return n > T(0) ? v3<T>{a.x / n, a.y / n, a.z / n} : v3<T>{0, 0, 0};
}
template <class T> __device__ __forceinline__ bool vfinite(v3<T> a) {
  return isfinite(a.x) && isfinite(a.y) && isfinite(a.z);
}
// finiteness of many values with one test: x * 0 is NaN exactly when x is
// +-inf or NaN, so a chain of fma(x, 0, z) from 0 stays +-0 unless some x is
// not finite (one FMA per value instead of a compare and a predicate op)
template <class T> __device__ __forceinline__ T nf_acc(T z, T x) { return fma(x, T(0), z); }
template <class T> __device__ __forceinline__ T comp(v3<T> a, int k) { return k == 0 ? a.x : (k == 1 ? a.y : a.z); }

// fp32 sine / cosine without sincosf's Payne-Hanek branch (a local-memory
// table and ~100 instructions inlined at every call site of an
// instruction-fetch-bound kernel): Cody-Waite reduction by pi/2 in three FMA
// steps, then the Cephes single-precision polynomials on [-pi/4, pi/4]
// (<= 1.5 ulp against libm for |a| < 1e4, checked in numpy; the step sees: half rotation angles, yaw and
// heading differences).  NaN / inf propagate as NaN, so divergence checks hold.
__device__ __forceinline__ void sincos_(float a, float* s, float* c) {
  const float k = rintf(a * 0.636619772f);
  float r = fmaf(k, -1.57079637f, a);
  r = fmaf(k, 4.37113883e-8f, r);
  r = fmaf(k, 1.77635684e-15f, r);
  const float z = r * r;
  const float sp = fmaf(fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f), z * r, r);
  const float cp = fmaf(fmaf(fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z,
                                   4.166664568298827e-2f), z, -0.5f), z, 1.0f);
  const int q = int(k) & 3;
  const float ss = (q & 1) ? cp : sp, cc = (q & 1) ? sp : cp;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}
__device__ __forceinline__ void sincos_(double a, double* s, double* c) { sincos(a, s, c); }
// (sin, cos) of atan2(y, x) without forming the angle: (y, x) / |(x, y)|, with
// atan2(0, 0) = 0.  fp32 step only (the f64 instrument keeps the reference's
// atan2 -> sin / cos; the two agree to a few ulp).
__device__ __forceinline__ void unit_dir(float y, float x, float* s, float* c) {
  const float r2 = x * x + y * y;
  const bool z = !(r2 > 0.f);
  const float inv = rsqrtf(z ? 1.f : r2);
  *c = z ? 1.f : x * inv;
  *s = z ? 0.f : y * inv;
}
template <class T> __device__ __forceinline__ T cos_(T a) {
  T s, c;
  sincos_(a, &s, &c);
  return c;
}

template <class T> __device__ __forceinline__ qt<T> qmul(qt<T> a, qt<T> b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
template <class T> __device__ __forceinline__ qt<T> qconj(qt<T> q) { return {q.w, -q.x, -q.y, -q.z}; }
template <class T> __device__ __forceinline__ qt<T> qunit(qt<T> q) {
  const T n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  return {q.w / n, q.x / n, q.y / n, q.z / n};
}
// v' = v + 2 q_v x (q_v x v + w v), vec.hpp:163-168
template <class T> __device__ __forceinline__ v3<T> qrot(qt<T> q, v3<T> v) {
  const v3<T> u{q.x, q.y, q.z};
  const v3<T> t = cross(u, v) * T(2);
  return v + t * q.w + cross(u, t);
}
template <class T> __device__ __forceinline__ bool qfinite(qt<T> q) {
  return isfinite(q.w) && isfinite(q.x) && isfinite(q.y) && isfinite(q.z);
}
// Quat::exp_map, vec.hpp:138-145
template <class T> __device__ __forceinline__ qt<T> qexp(v3<T> rv) {
  const T ang = vnorm(rv);
  if (ang < T(1e-12)) return qunit(qt<T>{T(1), T(0.5) * rv.x, T(0.5) * rv.y, T(0.5) * rv.z});
  const T h = T(0.5) * ang;
  T s, c;
  sincos_(h, &s, &c);
  const v3<T> a = vunit(rv);
  return {c, a.x * s, a.y * s, a.z * s};
}


// symmetric 3x3 stored as xx yy zz xy xz yz
template <class T>
struct sym3 {
  T xx, yy, zz, xy, xz, yz;
};
template <class T> __device__ __forceinline__ v3<T> smul(const sym3<T>& m, v3<T> v) {
  return {m.xx * v.x + m.xy * v.y + m.xz * v.z, m.xy * v.x + m.yy * v.y + m.yz * v.z,
          m.xz * v.x + m.yz * v.y + m.zz * v.z};
}
// R diag(d) R^T with R = to_matrix(q) (vec.hpp:171-180; solver.cpp:250-252)
template <class T> __device__ __forceinline__ void rot_mat(qt<T> q, T r[9]) {
  const T xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
  const T xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
  const T wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
  r[0] = 1 - 2 * (yy + zz); r[1] = 2 * (xy - wz); r[2] = 2 * (xz + wy);
  r[3] = 2 * (xy + wz); r[4] = 1 - 2 * (xx + zz); r[5] = 2 * (yz - wx);
  r[6] = 2 * (xz - wy); r[7] = 2 * (yz + wx); r[8] = 1 - 2 * (xx + yy);
}
template <class T> __device__ __forceinline__ sym3<T> rdrt(const T r[9], T d0, T d1, T d2) {
  sym3<T> s;
  s.xx = r[0] * d0 * r[0] + r[1] * d1 * r[1] + r[2] * d2 * r[2];
  s.yy = r[3] * d0 * r[3] + r[4] * d1 * r[4] + r[5] * d2 * r[5];
  s.zz = r[6] * d0 * r[6] + r[7] * d1 * r[7] + r[8] * d2 * r[8];
  s.xy = r[0] * d0 * r[3] + r[1] * d1 * r[4] + r[2] * d2 * r[5];
  s.xz = r[0] * d0 * r[6] + r[1] * d1 * r[7] + r[2] * d2 * r[8];
  s.yz = r[3] * d0 * r[6] + r[4] * d1 * r[7] + r[5] * d2 * r[8];
  return s;
}

// 6x6 symmetric packed lower triangle: index(i, j) with i >= j
__host__ __device__ constexpr int tri(int i, int j) { return i * (i + 1) / 2 + j; }
__host__ __device__ constexpr int sidx(int i, int j) { return i >= j ? tri(i, j) : tri(j, i); }

}  // namespace stp
