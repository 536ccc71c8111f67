// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
//
// CPU restatement of the reference physics step (stampede::physics::step,
// /root/reference/proj/src/physics/solver.cpp:448-597) for ONE environment,
// templated on the scalar type so the same code yields
//   * T = double : the parity oracle (pinned against the compiled reference
//                  in oracle/_ref, see tests/test_oracle_pin.py), and
//   * T = float  : the fp32 envelope of the reference algorithm, used to set
//                  the GPU tolerances.
// Every function cites the reference lines it restates.  Arithmetic order
// follows the reference (row order, block accumulation order, dot order) so
// that the double instantiation tracks the reference to rounding.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "stampede_sim.h"

namespace orc {

template <class T>
struct V {
  T x = 0, y = 0, z = 0;
  V() = default;
  V(T a, T b, T c) : x(a), y(b), z(c) {}
  V operator+(const V& o) const { return {x + o.x, y + o.y, z + o.z}; }
  V operator-(const V& o) const { return {x - o.x, y - o.y, z - o.z}; }
  V operator-() const { return {-x, -y, -z}; }
  V operator*(T s) const { return {x * s, y * s, z * s}; }
  V operator/(T s) const { return {x / s, y / s, z / s}; }
  T dot(const V& o) const { return x * o.x + y * o.y + z * o.z; }
  V cross(const V& o) const { return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x}; }
  T norm2() const { return dot(*this); }
  T norm() const { return std::sqrt(norm2()); }
  // vec.hpp:42-45
  V unit() const {
    const T n = norm();
    return n > 0 ? (*this) / n : V{};
  }
  T& operator[](int i) { return (&x)[i]; }
  T operator[](int i) const { return (&x)[i]; }
  bool finite() const { return std::isfinite(x) && std::isfinite(y) && std::isfinite(z); }
};

// row-major 3x3, vec.hpp:51-121
template <class T>
struct M3 {
  T a[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  T operator()(int r, int c) const { return a[3 * r + c]; }
  T& operator()(int r, int c) { return a[3 * r + c]; }
  static M3 diag(const V<T>& d) {
    M3 m;
    m.a[0] = d.x; m.a[4] = d.y; m.a[8] = d.z;
    m.a[1] = m.a[2] = m.a[3] = m.a[5] = m.a[6] = m.a[7] = 0;
    return m;
  }
  static M3 skew(const V<T>& v) {
    M3 m;
    m.a[0] = 0; m.a[1] = -v.z; m.a[2] = v.y;
    m.a[3] = v.z; m.a[4] = 0; m.a[5] = -v.x;
    m.a[6] = -v.y; m.a[7] = v.x; m.a[8] = 0;
    return m;
  }
  V<T> operator*(const V<T>& v) const {
    return {a[0] * v.x + a[1] * v.y + a[2] * v.z, a[3] * v.x + a[4] * v.y + a[5] * v.z,
            a[6] * v.x + a[7] * v.y + a[8] * v.z};
  }
  M3 operator*(const M3& o) const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        T s = 0;
        for (int k = 0; k < 3; ++k) s += (*this)(i, k) * o(k, j);
        r(i, j) = s;
      }
    return r;
  }
  M3 operator+(const M3& o) const {
    M3 r;
    for (int i = 0; i < 9; ++i) r.a[i] = a[i] + o.a[i];
    return r;
  }
  M3 operator*(T s) const {
    M3 r;
    for (int i = 0; i < 9; ++i) r.a[i] = a[i] * s;
    return r;
  }
  M3 T_() const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r(i, j) = (*this)(j, i);
    return r;
  }
  // adjugate inverse, vec.hpp:107-120
  M3 inv() const {
    const T A = a[4] * a[8] - a[5] * a[7], B = a[2] * a[7] - a[1] * a[8], C = a[1] * a[5] - a[2] * a[4];
    const T D = a[5] * a[6] - a[3] * a[8], E = a[0] * a[8] - a[2] * a[6], F = a[2] * a[3] - a[0] * a[5];
    const T G = a[3] * a[7] - a[4] * a[6], H = a[1] * a[6] - a[0] * a[7], I = a[0] * a[4] - a[1] * a[3];
    const T det = a[0] * A + a[1] * D + a[2] * G;
    M3 r;
    r.a[0] = A / det; r.a[1] = B / det; r.a[2] = C / det;
    r.a[3] = D / det; r.a[4] = E / det; r.a[5] = F / det;
    r.a[6] = G / det; r.a[7] = H / det; r.a[8] = I / det;
    return r;
  }
};

// unit quaternion (w, x, y, z), vec.hpp:124-190
template <class T>
struct Q {
  T w = 1, x = 0, y = 0, z = 0;
  Q() = default;
  Q(T a, T b, T c, T d) : w(a), x(b), y(c), z(d) {}
  Q operator*(const Q& o) const {
    return {w * o.w - x * o.x - y * o.y - z * o.z, w * o.x + x * o.w + y * o.z - z * o.y,
            w * o.y - x * o.z + y * o.w + z * o.x, w * o.z + x * o.y - y * o.x + z * o.w};
  }
  Q conj() const { return {w, -x, -y, -z}; }
  Q unit() const {
    const T n = std::sqrt(w * w + x * x + y * y + z * z);
    return {w / n, x / n, y / n, z / n};
  }
  // v' = v + 2 q_v x (q_v x v + w v), vec.hpp:163-168
  V<T> rot(const V<T>& v) const {
    const V<T> u{x, y, z};
    const V<T> t = u.cross(v) * T(2);
    return v + t * w + u.cross(t);
  }
  M3<T> mat() const {  // vec.hpp:171-180
    M3<T> r;
    const T xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
    const T wx = w * x, wy = w * y, wz = w * z;
    r.a[0] = 1 - 2 * (yy + zz); r.a[1] = 2 * (xy - wz); r.a[2] = 2 * (xz + wy);
    r.a[3] = 2 * (xy + wz); r.a[4] = 1 - 2 * (xx + zz); r.a[5] = 2 * (yz - wx);
    r.a[6] = 2 * (xz - wy); r.a[7] = 2 * (yz + wx); r.a[8] = 1 - 2 * (xx + yy);
    return r;
  }
  // exp_map, vec.hpp:130-145
  static Q expmap(const V<T>& rv) {
    const T ang = rv.norm();
    if (ang < T(1e-12)) return Q{1, T(0.5) * rv.x, T(0.5) * rv.y, T(0.5) * rv.z}.unit();
    const T h = T(0.5) * ang;
    const T s = std::sin(h);
    const V<T> a = rv.unit();
    return {std::cos(h), a.x * s, a.y * s, a.z * s};
  }
  bool finite() const { return std::isfinite(w) && std::isfinite(x) && std::isfinite(y) && std::isfinite(z); }
};

template <class T>
struct Body {  // RigidBodyState, types.hpp:28-38
  V<T> x;
  Q<T> q;
  V<T> v, w;
  bool finite() const { return x.finite() && q.finite() && v.finite() && w.finite(); }
};

template <class T>
struct Contact {  // ContactPoint + SolvedContact, types.hpp:76-83, :109-113
  int a = 0, b = -1;
  V<T> p, n;
  T sep = 0, mu = 1;
  T pn = 0;
  V<T> pt;
};

struct StepStats {
  int newton = 0, krylov = 0;
  bool failed = false;
};

// Scene constants of one env converted to T.
template <class T>
struct Model {
  int nb = 0, nj = 0;
  int shape[STP_MAX_BODIES];
  bool is_static[STP_MAX_BODIES];
  T radius[STP_MAX_BODIES], half_len[STP_MAX_BODIES];
  V<T> half_ext[STP_MAX_BODIES], local_pos[STP_MAX_BODIES];
  Q<T> local_rot[STP_MAX_BODIES];
  T mass[STP_MAX_BODIES];
  V<T> inertia[STP_MAX_BODIES];
  int jp[STP_MAX_JOINTS], jc[STP_MAX_JOINTS];
  V<T> anc_p[STP_MAX_JOINTS], anc_c[STP_MAX_JOINTS], ax_p[STP_MAX_JOINTS], ax_c[STP_MAX_JOINTS];
  Q<T> rest[STP_MAX_JOINTS];
  T lim_lo[STP_MAX_JOINTS], lim_hi[STP_MAX_JOINTS], tmax[STP_MAX_JOINTS];

  void load(const stp_model& m) {
    nb = m.n_bodies;
    nj = m.n_joints;
    for (int b = 0; b < nb; ++b) {
      const stp_body& d = m.bodies[b];
      shape[b] = d.shape;
      is_static[b] = d.is_static != 0;
      radius[b] = T(d.radius);
      half_len[b] = T(d.half_length);
      half_ext[b] = {T(d.half_extents[0]), T(d.half_extents[1]), T(d.half_extents[2])};
      local_pos[b] = {T(d.local_pos[0]), T(d.local_pos[1]), T(d.local_pos[2])};
      local_rot[b] = {T(d.local_rot[0]), T(d.local_rot[1]), T(d.local_rot[2]), T(d.local_rot[3])};
      mass[b] = T(d.mass);
      inertia[b] = {T(d.inertia_diag[0]), T(d.inertia_diag[1]), T(d.inertia_diag[2])};
    }
    for (int j = 0; j < nj; ++j) {
      const stp_joint& d = m.joints[j];
      jp[j] = d.parent;
      jc[j] = d.child;
      anc_p[j] = {T(d.anchor_parent[0]), T(d.anchor_parent[1]), T(d.anchor_parent[2])};
      anc_c[j] = {T(d.anchor_child[0]), T(d.anchor_child[1]), T(d.anchor_child[2])};
      ax_p[j] = {T(d.axis_parent[0]), T(d.axis_parent[1]), T(d.axis_parent[2])};
      ax_c[j] = {T(d.axis_child[0]), T(d.axis_child[1]), T(d.axis_child[2])};
      rest[j] = {T(d.rest_relative[0]), T(d.rest_relative[1]), T(d.rest_relative[2]), T(d.rest_relative[3])};
      lim_lo[j] = T(d.limit_lo);
      lim_hi[j] = T(d.limit_hi);
      tmax[j] = T(d.max_torque);
    }
  }
};

template <class T>
struct Cfg {
  T dt, tol, margin, beta, kj, kc, kl, epsf, lim_act;
  int newton, kmax;
  V<T> g;
  bool plane;
  bool alias_quirk;
  void load(const stp_step_config& c) {
    dt = T(c.dt); tol = T(c.krylov_tol); margin = T(c.contact_margin); beta = T(c.baumgarte);
    kj = T(c.joint_hardness); kc = T(c.contact_hardness); kl = T(c.limit_hardness);
    epsf = T(c.friction_smoothing); lim_act = T(c.limit_activation);
    newton = c.newton_iters; kmax = c.krylov_max_iters;
    g = {T(c.gravity[0]), T(c.gravity[1]), T(c.gravity[2])};
    plane = c.has_ground_plane != 0;
    alias_quirk = c.reference_alias_quirk != 0;
  }
};

template <class T>
struct Box {  // ObbFrame, collide.cpp:123-136
  V<T> c, h;
  M3<T> r;
};

// ---------------------------------------------------------------------------
// Contacts (collide.cpp)
// ---------------------------------------------------------------------------
template <class T>
struct Shape {  // WorldShape, collide.cpp:28-36
  int type;
  V<T> p0, p1;
  T r;
  V<T> c;
  M3<T> rot;
  V<T> h;
  V<T> lo, hi;
};

// world_shape, collide.cpp:38-78
template <class T>
Shape<T> world_shape(const Model<T>& m, int b, const Body<T>& s) {
  Shape<T> w{};
  w.type = m.shape[b];
  const Q<T> rot = s.q * m.local_rot[b];
  const V<T> pos = s.x + s.q.rot(m.local_pos[b]);
  const V<T> rr{m.radius[b], m.radius[b], m.radius[b]};
  if (w.type == STP_SPHERE) {
    w.p0 = w.p1 = pos;
    w.r = m.radius[b];
    w.lo = pos - rr;
    w.hi = pos + rr;
  } else if (w.type == STP_CAPSULE) {
    const V<T> ax = rot.rot(V<T>{0, 0, m.half_len[b]});
    w.p0 = pos - ax;
    w.p1 = pos + ax;
    w.r = m.radius[b];
    w.lo = V<T>{std::min(w.p0.x, w.p1.x), std::min(w.p0.y, w.p1.y), std::min(w.p0.z, w.p1.z)} - rr;
    w.hi = V<T>{std::max(w.p0.x, w.p1.x), std::max(w.p0.y, w.p1.y), std::max(w.p0.z, w.p1.z)} + rr;
  } else {
    w.c = pos;
    w.rot = rot.mat();
    w.h = m.half_ext[b];
    V<T> e{};
    for (int i = 0; i < 3; ++i) {
      e.x += std::abs(w.rot(0, i)) * w.h[i];
      e.y += std::abs(w.rot(1, i)) * w.h[i];
      e.z += std::abs(w.rot(2, i)) * w.h[i];
    }
    w.lo = pos - e;
    w.hi = pos + e;
  }
  return w;
}

template <class T>
void push_contact(std::vector<Contact<T>>& out, int a, const V<T>& p, const V<T>& n, T sep) {
  Contact<T> c;
  c.a = a;
  c.b = -1;
  c.p = p;
  c.n = n;
  c.sep = sep;
  c.mu = T(1);  // kDefaultFriction, collide.cpp:25
  out.push_back(c);
}

// collide_plane, collide.cpp:93-119
template <class T>
void plane_contacts(const Shape<T>& s, int b, T margin, std::vector<Contact<T>>& out) {
  const V<T> up{0, 0, 1};
  if (s.type == STP_SPHERE) {
    const T sep = s.p0.z - s.r;
    if (sep < margin) push_contact(out, b, s.p0 - up * s.r, up, sep);
  } else if (s.type == STP_CAPSULE) {
    const V<T> ends[2] = {s.p0, s.p1};
    for (const V<T>& e : ends) {
      const T sep = e.z - s.r;
      if (sep < margin) push_contact(out, b, e - up * s.r, up, sep);
    }
  } else {
    for (int cx = -1; cx <= 1; cx += 2)
      for (int cy = -1; cy <= 1; cy += 2)
        for (int cz = -1; cz <= 1; cz += 2) {
          const V<T> loc{T(cx) * s.h.x, T(cy) * s.h.y, T(cz) * s.h.z};
          const V<T> corner = s.c + s.rot * loc;
          if (corner.z < margin) push_contact(out, b, corner, up, corner.z);
        }
  }
}

// obb_frame, collide.cpp:129-136
template <class T>
Box<T> make_box(const stp_static_box& sb) {
  Box<T> f;
  const T yaw = T(sb.yaw);
  const T c = std::cos(yaw), s = std::sin(yaw);
  f.r.a[0] = c; f.r.a[1] = -s; f.r.a[2] = 0;
  f.r.a[3] = s; f.r.a[4] = c; f.r.a[5] = 0;
  f.r.a[6] = 0; f.r.a[7] = 0; f.r.a[8] = 1;
  f.c = {T(sb.center[0]), T(sb.center[1]), T(sb.center[2])};
  f.h = {T(sb.half_extents[0]), T(sb.half_extents[1]), T(sb.half_extents[2])};
  return f;
}

// point_obb, collide.cpp:140-173: signed distance, outward normal, surface point
template <class T>
T point_box(const Box<T>& bx, const V<T>& p, V<T>& n, V<T>& surf) {
  const V<T> loc = bx.r.T_() * (p - bx.c);
  const V<T> h = bx.h;
  const V<T> cl{std::clamp(loc.x, -h.x, h.x), std::clamp(loc.y, -h.y, h.y), std::clamp(loc.z, -h.z, h.z)};
  const V<T> d = loc - cl;
  const T out = d.norm();
  if (out > T(1e-12)) {
    surf = bx.c + bx.r * cl;
    n = (bx.r * d) / out;
    return out;
  }
  T best = h.x - std::abs(loc.x);
  int axis = 0;
  T sgn = loc.x >= 0 ? T(1) : T(-1);
  if (h.y - std::abs(loc.y) < best) {
    best = h.y - std::abs(loc.y);
    axis = 1;
    sgn = loc.y >= 0 ? T(1) : T(-1);
  }
  if (h.z - std::abs(loc.z) < best) {
    best = h.z - std::abs(loc.z);
    axis = 2;
    sgn = loc.z >= 0 ? T(1) : T(-1);
  }
  V<T> ln{};
  ln[axis] = sgn;
  V<T> ls = loc;
  ls[axis] = sgn * h[axis];
  surf = bx.c + bx.r * ls;
  n = bx.r * ln;
  return -best;
}

// collide_sphere_obb / collide_capsule_obb, collide.cpp:175-214
template <class T>
void box_contacts(const Shape<T>& s, const Box<T>& bx, int b, T margin, std::vector<Contact<T>>& out) {
  V<T> n, surf;
  if (s.type == STP_SPHERE) {
    const T d = point_box(bx, s.p0, n, surf);
    const T sep = d - s.r;
    if (sep < margin) push_contact(out, b, surf, n, sep);
    return;
  }
  const V<T> seg = s.p1 - s.p0;
  auto dist_at = [&](T t) {
    V<T> nn, ss;
    return point_box(bx, s.p0 + seg * t, nn, ss);
  };
  T lo = 0, hi = 1;
  for (int i = 0; i < 32; ++i) {  // ternary search, collide.cpp:193-197
    const T m1 = lo + (hi - lo) / 3, m2 = hi - (hi - lo) / 3;
    if (dist_at(m1) <= dist_at(m2)) hi = m2;
    else lo = m1;
  }
  const T tmid = T(0.5) * (lo + hi);
  bool mid_added = false;
  {
    const T d = point_box(bx, s.p0 + seg * tmid, n, surf);
    if (d - s.r < margin) {
      push_contact(out, b, surf, n, d - s.r);
      mid_added = true;
    }
  }
  const T ts[2] = {T(0), T(1)};
  for (T t : ts) {
    if (mid_added && std::abs(t - tmid) < T(0.05)) continue;
    const T d = point_box(bx, s.p0 + seg * t, n, surf);
    if (d - s.r < margin) push_contact(out, b, surf, n, d - s.r);
  }
}

// detect_contacts static part, collide.cpp:270-299 (inter-agent pairs are
// off for every parity workload)
template <class T>
void detect(const Model<T>& m, const Body<T>* st, const std::vector<Box<T>>& boxes, bool plane, T margin,
            std::vector<Contact<T>>& out) {
  out.clear();
  for (int b = 0; b < m.nb; ++b) {
    if (m.is_static[b]) continue;
    const Shape<T> ws = world_shape(m, b, st[b]);
    if (plane && ws.lo.z < margin) plane_contacts(ws, b, margin, out);
    for (const Box<T>& bx : boxes) {
      const T ex = bx.h.x + bx.h.y;
      const V<T> bmin = bx.c - V<T>{ex, ex, bx.h.z};
      const V<T> bmax = bx.c + V<T>{ex, ex, bx.h.z};
      if (ws.hi.x + margin < bmin.x || ws.lo.x - margin > bmax.x || ws.hi.y + margin < bmin.y ||
          ws.lo.y - margin > bmax.y || ws.hi.z + margin < bmin.z || ws.lo.z - margin > bmax.z)
        continue;
      if (ws.type == STP_SPHERE || ws.type == STP_CAPSULE) box_contacts(ws, bx, b, margin, out);
    }
  }
}

// ---------------------------------------------------------------------------
// Rows + dynamics (solver.cpp:27-276)
// ---------------------------------------------------------------------------
enum { kEq = 0, kUni = 1, kFric = 2 };

template <class T>
struct Row {  // solver.cpp:38-49
  int a = -1, b = -1;
  T ja[6] = {0, 0, 0, 0, 0, 0};
  T jb[6] = {0, 0, 0, 0, 0, 0};
  T bias = 0, reg = 0;
  int kind = kEq;
  bool active = true;
  int contact = -1, fpair = -1;
};

template <class T>
struct Dyn {  // BodyDyn, solver.cpp:51-56
  T inv_m = 0;
  M3<T> I, Iinv;
  T vfree[6] = {0, 0, 0, 0, 0, 0};
};

template <class T>
T dot6(const T* j, const T* u) {
  return j[0] * u[0] + j[1] * u[1] + j[2] * u[2] + j[3] * u[3] + j[4] * u[4] + j[5] * u[5];
}
template <class T>
void set6(T* j, const V<T>& l, const V<T>& a) {
  j[0] = l.x; j[1] = l.y; j[2] = l.z;
  j[3] = a.x; j[4] = a.y; j[5] = a.z;
}

// effective_mass, solver.cpp:69-80
template <class T>
T eff_mass(const Row<T>& r, const Model<T>& m, const Dyn<T>* dyn) {
  T w = 0;
  const int bodies[2] = {r.a, r.b};
  const T* js[2] = {r.ja, r.jb};
  for (int k = 0; k < 2; ++k) {
    const int body = bodies[k];
    if (body < 0 || m.is_static[body]) continue;
    const T* j = js[k];
    const Dyn<T>& d = dyn[body];
    w += d.inv_m * (j[0] * j[0] + j[1] * j[1] + j[2] * j[2]);
    const V<T> ang{j[3], j[4], j[5]};
    w += ang.dot(d.Iinv * ang);
  }
  return w > T(1e-12) ? T(1) / w : T(0);
}

// unilateral_bias, solver.cpp:84-87
template <class T>
T uni_bias(T gap, T beta, T dt) {
  if (gap < 0) return -(beta / dt) * gap;
  return -gap / dt;
}

// joint_angle / joint_velocity, solver.cpp:405-417
template <class T>
T hinge_angle(const Body<T>& p, const Body<T>& c, const Q<T>& rest, const V<T>& axc) {
  const Q<T> rel = p.q.conj() * c.q;
  Q<T> d = rest.conj() * rel;
  if (d.w < 0) d = Q<T>{-d.w, -d.x, -d.y, -d.z};
  const T proj = d.x * axc.x + d.y * axc.y + d.z * axc.z;
  return T(2) * std::atan2(proj, d.w);
}
template <class T>
T hinge_rate(const Body<T>& p, const Body<T>& c, const V<T>& axc) {
  return c.q.rot(axc).dot(c.w - p.w);
}

// build_rows, solver.cpp:98-212
template <class T>
void build_rows(const Model<T>& m, const Body<T>* st, const std::vector<int>& joints,
                const std::vector<Contact<T>*>& cts, const Dyn<T>* dyn, const Cfg<T>& cf,
                std::vector<Row<T>>& rows) {
  rows.clear();
  const T beta = cf.beta, dt = cf.dt;
  for (int j : joints) {
    const Body<T>& sp = st[m.jp[j]];
    const Body<T>& sc = st[m.jc[j]];
    const V<T> ra = sp.q.rot(m.anc_p[j]);
    const V<T> rb = sc.q.rot(m.anc_c[j]);
    const V<T> cpos = (sc.x + rb) - (sp.x + ra);
    for (int k = 0; k < 3; ++k) {
      V<T> e{};
      e[k] = T(1);
      Row<T> r;
      r.a = m.jp[j];
      r.b = m.jc[j];
      set6(r.ja, -e, -(ra.cross(e)));
      set6(r.jb, e, rb.cross(e));
      r.bias = -(beta / dt) * cpos[k];
      r.reg = cf.kj * eff_mass(r, m, dyn);
      rows.push_back(r);
    }
    const V<T> aw = sp.q.rot(m.ax_p[j]);
    const V<T> bw = sc.q.rot(m.ax_c[j]);
    const V<T> ref = std::abs(aw.z) < T(0.9) ? V<T>{0, 0, 1} : V<T>{1, 0, 0};
    const V<T> t1 = aw.cross(ref).unit();
    const V<T> t2 = aw.cross(t1);
    const V<T> err = aw.cross(bw);
    const V<T> ts[2] = {t1, t2};
    for (const V<T>& t : ts) {
      Row<T> r;
      r.a = m.jp[j];
      r.b = m.jc[j];
      set6(r.ja, V<T>{}, -t);
      set6(r.jb, V<T>{}, t);
      r.bias = -(beta / dt) * t.dot(err);
      r.reg = cf.kj * eff_mass(r, m, dyn);
      rows.push_back(r);
    }
    const T angle = hinge_angle(sp, sc, m.rest[j], m.ax_c[j]);
    const T rate = hinge_rate(sp, sc, m.ax_c[j]);
    const V<T> axw = sc.q.rot(m.ax_c[j]);
    const T lo_gap = angle - m.lim_lo[j];
    const T hi_gap = m.lim_hi[j] - angle;
    const T travel = T(1.5) * std::abs(rate) * dt;
    const T thresh = std::max(cf.lim_act, travel);
    if (lo_gap < thresh) {
      Row<T> r;
      r.a = m.jp[j];
      r.b = m.jc[j];
      set6(r.ja, V<T>{}, -axw);
      set6(r.jb, V<T>{}, axw);
      r.bias = uni_bias(lo_gap, beta, dt);
      r.reg = cf.kl * eff_mass(r, m, dyn);
      r.kind = kUni;
      rows.push_back(r);
    }
    if (hi_gap < thresh) {
      Row<T> r;
      r.a = m.jp[j];
      r.b = m.jc[j];
      set6(r.ja, V<T>{}, axw);
      set6(r.jb, V<T>{}, -axw);
      r.bias = uni_bias(hi_gap, beta, dt);
      r.reg = cf.kl * eff_mass(r, m, dyn);
      r.kind = kUni;
      rows.push_back(r);
    }
  }
  for (size_t ci = 0; ci < cts.size(); ++ci) {
    const Contact<T>& c = *cts[ci];
    const V<T> ra = c.p - st[c.a].x;
    Row<T> nr;
    nr.a = c.a;
    nr.b = c.b;
    set6(nr.ja, c.n, ra.cross(c.n));
    nr.bias = uni_bias(c.sep, beta, dt);
    nr.reg = cf.kc * eff_mass(nr, m, dyn);
    nr.kind = kUni;
    nr.contact = int(ci);
    nr.fpair = int(rows.size()) + 1;
    rows.push_back(nr);
    const V<T> ref = std::abs(c.n.z) < T(0.9) ? V<T>{0, 0, 1} : V<T>{1, 0, 0};
    const V<T> t1 = c.n.cross(ref).unit();
    const V<T> t2 = c.n.cross(t1);
    const V<T> ts[2] = {t1, t2};
    for (const V<T>& t : ts) {
      Row<T> f;
      f.a = c.a;
      f.b = c.b;
      set6(f.ja, t, ra.cross(t));
      f.kind = kFric;
      f.contact = int(ci);
      f.active = false;
      rows.push_back(f);
    }
  }
}

// implicit_gyro, solver.cpp:216-226
template <class T>
V<T> gyro(const M3<T>& I, const V<T>& w0, const V<T>& tau, T dt) {
  V<T> w = w0;
  const V<T> mom = I * w0 + tau * dt;
  for (int it = 0; it < 2; ++it) {
    const V<T> iw = I * w;
    const V<T> f = iw + w.cross(iw) * dt - mom;
    const M3<T> jac = I + (M3<T>::skew(w) * I + M3<T>::skew(iw) * T(-1)) * dt;
    w = w - jac.inv() * f;
  }
  return w.finite() ? w : w0;
}

// body_dynamics, solver.cpp:230-262
template <class T>
void dynamics(const Model<T>& m, const Body<T>* st, const T* tau, const V<T>* fext, const V<T>* text,
              const Cfg<T>& cf, Dyn<T>* dyn) {
  V<T> torque[STP_MAX_BODIES];
  for (int b = 0; b < m.nb; ++b) {
    dyn[b] = Dyn<T>{};
    torque[b] = text[b];
  }
  for (int j = 0; j < m.nj; ++j) {
    const V<T> axw = st[m.jp[j]].q.rot(m.ax_p[j]);
    torque[m.jc[j]] = torque[m.jc[j]] + axw * tau[j];
    torque[m.jp[j]] = torque[m.jp[j]] - axw * tau[j];
  }
  for (int b = 0; b < m.nb; ++b) {
    if (m.is_static[b]) continue;
    Dyn<T>& d = dyn[b];
    d.inv_m = T(1) / m.mass[b];
    const M3<T> r = st[b].q.mat();
    d.I = r * M3<T>::diag(m.inertia[b]) * r.T_();
    const V<T> invd{T(1) / m.inertia[b].x, T(1) / m.inertia[b].y, T(1) / m.inertia[b].z};
    d.Iinv = r * M3<T>::diag(invd) * r.T_();
    V<T> force = cf.g * m.mass[b];
    force = force + fext[b];
    const V<T> v = st[b].v + force * (cf.dt * d.inv_m);
    const V<T> w = gyro(d.I, st[b].w, torque[b], cf.dt);
    d.vfree[0] = v.x; d.vfree[1] = v.y; d.vfree[2] = v.z;
    d.vfree[3] = w.x; d.vfree[4] = w.y; d.vfree[5] = w.z;
  }
}

// friction_weight, solver.cpp:267-270
template <class T>
T fric_w(T mu, T pn, T vt, T eps) {
  const T s = vt / eps;
  return mu * pn / (eps * std::sqrt(T(1) + s * s));
}

// ---------------------------------------------------------------------------
// Block-sparse system + preconditioned conjugate residual
// (block_sparse.cpp:28-67, krylov.cpp:27-174)
// ---------------------------------------------------------------------------
template <class T>
struct BlockSys {
  int k = 0;
  bool present[STP_MAX_BODIES][STP_MAX_BODIES];
  T blk[STP_MAX_BODIES][STP_MAX_BODIES][36];
  void reset(int n) {
    k = n;
    nblocks = 0;
    capacity = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) present[i][j] = false;
  }
  // Block-pool bookkeeping of BlockSparseSym (block_sparse.cpp:212-223):
  // blocks live in one std::vector<double> grown by 36 doubles per new
  // block, so libstdc++ doubles its capacity (1, 2, 4, 8, ... blocks).
  int nblocks = 0, capacity = 0;
  T* at(int i, int j) {  // BlockSparseSym::block: zero block on first touch
    if (!present[i][j]) {
      present[i][j] = true;
      std::memset(blk[i][j], 0, sizeof(blk[i][j]));
      if (nblocks + 1 > capacity) capacity = capacity == 0 ? 1 : 2 * capacity;
      ++nblocks;
    }
    return blk[i][j];
  }
  // True when creating block (i, j) now reallocates the pool, which
  // invalidates every block pointer handed out before (see assemble()).
  bool create_reallocates(int i, int j) const { return !present[i][j] && nblocks + 1 > capacity; }
  // y = A x with the reference's accumulation order (block rows, cols ascending)
  void apply(const T* x, T* y) const {
    for (int i = 0; i < 6 * k; ++i) y[i] = 0;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {
        if (!present[i][j]) continue;
        const T* b = blk[i][j];
        for (int r = 0; r < 6; ++r) {
          T s = 0;
          for (int c = 0; c < 6; ++c) s += b[r * 6 + c] * x[6 * j + c];
          y[6 * i + r] += s;
        }
      }
  }
  bool finite() const {
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        if (present[i][j])
          for (int e = 0; e < 36; ++e)
            if (!std::isfinite(blk[i][j][e])) return false;
    return true;
  }
};

// cholesky / cholesky_solve, krylov.cpp:27-56
template <class T>
bool chol6(T* a) {
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      T s = a[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= a[i * 6 + k] * a[j * 6 + k];
      if (i == j) {
        if (s <= 0) return false;
        a[i * 6 + i] = std::sqrt(s);
      } else {
        a[i * 6 + j] = s / a[j * 6 + j];
      }
    }
  return true;
}
template <class T>
void chol6_solve(const T* l, const T* rhs, T* out) {
  for (int i = 0; i < 6; ++i) {
    T s = rhs[i];
    for (int k = 0; k < i; ++k) s -= l[i * 6 + k] * out[k];
    out[i] = s / l[i * 6 + i];
  }
  for (int i = 5; i >= 0; --i) {
    T s = out[i];
    for (int k = i + 1; k < 6; ++k) s -= l[k * 6 + i] * out[k];
    out[i] = s / l[i * 6 + i];
  }
}

template <class T>
T vdot(const T* a, const T* b, int n) {
  T s = 0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

struct KrylovResult {
  int iters = 0;
  bool nonfinite_input = false;
};

// solve_krylov_inplace, krylov.cpp:106-174 (the reference throws on
// non-finite A/b, :113-114; here the caller marks the island failed)
template <class T>
KrylovResult pcr(const BlockSys<T>& A, const T* b, T* x, T tol, int max_iters) {
  KrylovResult res;
  const int n = 6 * A.k;
  bool fin = A.finite();
  for (int i = 0; i < n && fin; ++i) fin = std::isfinite(b[i]);
  if (!fin) {
    res.nonfinite_input = true;
    return res;
  }
  const T bn = std::sqrt(vdot(b, b, n));
  if (bn == T(0)) {
    for (int i = 0; i < n; ++i) x[i] = 0;
    return res;
  }
  // BlockJacobi, krylov.cpp:60-88
  T fac[STP_MAX_BODIES][36];
  bool ok[STP_MAX_BODIES];
  for (int i = 0; i < A.k; ++i) {
    ok[i] = false;
    if (!A.present[i][i]) continue;
    std::memcpy(fac[i], A.blk[i][i], sizeof(fac[i]));
    ok[i] = chol6(fac[i]);
  }
  auto precond = [&](const T* r, T* z) {
    for (int i = 0; i < A.k; ++i) {
      if (ok[i]) chol6_solve(fac[i], r + 6 * i, z + 6 * i);
      else
        for (int c = 0; c < 6; ++c) z[6 * i + c] = r[6 * i + c];
    }
  };
  const int N = 6 * STP_MAX_BODIES;
  T r[N], z[N], p[N], az[N], ap[N], map[N], tmp[N];
  A.apply(x, tmp);
  for (int i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
  precond(r, z);
  for (int i = 0; i < n; ++i) p[i] = z[i];
  A.apply(z, az);
  for (int i = 0; i < n; ++i) ap[i] = az[i];
  T zaz = vdot(z, az, n);
  const T tol_abs = tol * bn;
  T rn = std::sqrt(vdot(r, r, n));
  int k = 0;
  while (k < max_iters && rn > tol_abs) {
    precond(ap, map);
    const T denom = vdot(ap, map, n);
    if (!(denom > 0) || !(zaz > 0)) break;
    const T alpha = zaz / denom;
    for (int i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    ++k;
    precond(r, z);
    rn = std::sqrt(vdot(r, r, n));
    if (rn <= tol_abs) break;
    A.apply(z, az);
    const T zn = vdot(z, az, n);
    const T beta = zn / zaz;
    zaz = zn;
    for (int i = 0; i < n; ++i) {
      p[i] = z[i] + beta * p[i];
      ap[i] = az[i] + beta * ap[i];
    }
  }
  res.iters = k;
  bool xf = true;
  for (int i = 0; i < n; ++i) xf = xf && std::isfinite(x[i]);
  if (!xf)
    for (int i = 0; i < n; ++i) x[i] = 0;
  return res;
}

// assemble, solver.cpp:281-360
template <class T>
void assemble(const Model<T>& m, const Dyn<T>* dyn, std::vector<Row<T>>& rows, std::vector<Contact<T>*>& cts,
              const int* slot, const std::vector<int>& slot_body, const T* u, const Cfg<T>& cf,
              BlockSys<T>& H, T* rhs) {
  const int k = int(slot_body.size());
  H.reset(k);
  for (int i = 0; i < 6 * k; ++i) rhs[i] = 0;
  static const T zeros[6] = {0, 0, 0, 0, 0, 0};
  auto vel = [&](int body) -> const T* {
    const int s = body < 0 ? -1 : slot[body];
    return s < 0 ? zeros : u + 6 * s;
  };
  for (int s = 0; s < k; ++s) {
    const int b = slot_body[s];
    const Dyn<T>& d = dyn[b];
    T* blk = H.at(s, s);
    const T ms = m.mass[b];
    blk[0] += ms;
    blk[7] += ms;
    blk[14] += ms;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) blk[(3 + r) * 6 + 3 + c] += d.I(r, c);
    T* o = rhs + 6 * s;
    for (int q = 0; q < 3; ++q) o[q] = ms * d.vfree[q];
    const V<T> iw = d.I * V<T>{d.vfree[3], d.vfree[4], d.vfree[5]};
    o[3] = iw.x; o[4] = iw.y; o[5] = iw.z;
  }
  for (auto& row : rows) {
    if (row.kind != kUni) continue;
    const T rate = dot6(row.ja, vel(row.a)) + dot6(row.jb, vel(row.b));
    const T pred = row.reg * (row.bias - rate);
    row.active = pred > 0;
    if (row.contact >= 0) {
      Row<T>& f1 = rows[row.fpair];
      Row<T>& f2 = rows[row.fpair + 1];
      if (row.active) {
        const T v1 = dot6(f1.ja, vel(f1.a)) + dot6(f1.jb, vel(f1.b));
        const T v2 = dot6(f2.ja, vel(f2.a)) + dot6(f2.jb, vel(f2.b));
        const T vt = std::sqrt(v1 * v1 + v2 * v2);
        const T w = fric_w(cts[row.contact]->mu, pred, vt, cf.epsf);
        f1.active = f2.active = true;
        f1.reg = f2.reg = w;
      } else {
        f1.active = f2.active = false;
      }
    }
  }
  for (const auto& row : rows) {
    if (!row.active || row.reg <= 0) continue;
    const T d = row.reg;
    const int sa = row.a < 0 ? -1 : slot[row.a];
    const int sb = row.b < 0 ? -1 : slot[row.b];
    if (sa >= 0) {
      T* blk = H.at(sa, sa);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) blk[r * 6 + c] += d * row.ja[r] * row.ja[c];
      T* o = rhs + 6 * sa;
      for (int r = 0; r < 6; ++r) o[r] += row.ja[r] * d * row.bias;
    }
    if (sb >= 0) {
      T* blk = H.at(sb, sb);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) blk[r * 6 + c] += d * row.jb[r] * row.jb[c];
      T* o = rhs + 6 * sb;
      for (int r = 0; r < 6; ++r) o[r] += row.jb[r] * d * row.bias;
    }
    if (sa >= 0 && sb >= 0) {
      T* ab = H.at(sa, sb);
      // Reference quirk (solver.cpp:350-351): `ab` is taken before
      // h.block(sb, sa) may grow the pool (block_sparse.cpp:33-37); when that
      // reallocates, the writes through `ab` land in freed memory and this
      // row's contribution to block (sa, sb) is lost.  Emulated so the
      // oracle reproduces the reference's actual output.
      T lost[36];
      if (cf.alias_quirk && H.create_reallocates(sb, sa)) ab = lost;
      T* ba = H.at(sb, sa);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) {
          const T v = d * row.ja[r] * row.jb[c];
          ab[r * 6 + c] += v;
          ba[c * 6 + r] += v;
        }
    }
  }
}

// report_impulses, solver.cpp:365-391
template <class T>
void report(const std::vector<Row<T>>& rows, std::vector<Contact<T>*>& cts, const int* slot, const T* u,
            const Cfg<T>& cf) {
  static const T zeros[6] = {0, 0, 0, 0, 0, 0};
  auto vel = [&](int body) -> const T* {
    const int s = body < 0 ? -1 : slot[body];
    return s < 0 ? zeros : u + 6 * s;
  };
  for (const auto& row : rows) {
    if (row.kind != kUni || row.contact < 0) continue;
    const T rate = dot6(row.ja, vel(row.a)) + dot6(row.jb, vel(row.b));
    const T pn = std::max(T(0), row.reg * (row.bias - rate));
    Contact<T>& c = *cts[row.contact];
    c.pn = pn;
    if (pn <= 0) {
      c.pt = V<T>{};
      continue;
    }
    const Row<T>& f1 = rows[row.fpair];
    const Row<T>& f2 = rows[row.fpair + 1];
    const T v1 = dot6(f1.ja, vel(f1.a)) + dot6(f1.jb, vel(f1.b));
    const T v2 = dot6(f2.ja, vel(f2.a)) + dot6(f2.jb, vel(f2.b));
    const T vt = std::sqrt(v1 * v1 + v2 * v2);
    const T w = fric_w(c.mu, pn, vt, cf.epsf);
    const V<T> t1{f1.ja[0], f1.ja[1], f1.ja[2]};
    const V<T> t2{f2.ja[0], f2.ja[1], f2.ja[2]};
    c.pt = t1 * (-w * v1) + t2 * (-w * v2);
  }
}

// One environment's physics::step (solver.cpp:448-597): islands are the
// joint-connected components of its dynamic bodies (no dynamic contacts
// because inter-agent collisions are off and agents never self-collide).
template <class T>
StepStats step_env(const Model<T>& m, const Cfg<T>& cf, const std::vector<Box<T>>& boxes, Body<T>* st,
                   const T* tau_in, const V<T>* fext, const V<T>* text, std::vector<Contact<T>>& contacts) {
  StepStats stats;
  const int n = m.nb;
  T tau[STP_MAX_JOINTS];
  for (int j = 0; j < m.nj; ++j) tau[j] = std::clamp(tau_in[j], -m.tmax[j], m.tmax[j]);  // :395-403
  detect(m, st, boxes, cf.plane, cf.margin, contacts);
  Dyn<T> dyn[STP_MAX_BODIES];
  dynamics(m, st, tau, fext, text, cf, dyn);

  // islands (union-find over dynamic-dynamic joints), solver.cpp:458-502
  int par[STP_MAX_BODIES];
  for (int b = 0; b < n; ++b) par[b] = b;
  auto find = [&](int x) {
    while (par[x] != x) {
      par[x] = par[par[x]];
      x = par[x];
    }
    return x;
  };
  for (int j = 0; j < m.nj; ++j)
    if (!m.is_static[m.jp[j]] && !m.is_static[m.jc[j]]) par[find(m.jp[j])] = find(m.jc[j]);
  int island_of[STP_MAX_BODIES];
  std::vector<std::vector<int>> isl_bodies;
  for (int b = 0; b < n; ++b) island_of[b] = -1;
  for (int b = 0; b < n; ++b) {
    if (m.is_static[b]) continue;
    const int root = find(b);
    if (island_of[root] < 0) {
      island_of[root] = int(isl_bodies.size());
      isl_bodies.emplace_back();
    }
    island_of[b] = island_of[root];
    isl_bodies[island_of[b]].push_back(b);
  }
  const int ni = int(isl_bodies.size());
  std::vector<std::vector<int>> isl_joints(ni);
  std::vector<std::vector<Contact<T>*>> isl_cts(ni);
  for (int j = 0; j < m.nj; ++j) {
    int isl = island_of[m.jp[j]];
    if (isl < 0) isl = island_of[m.jc[j]];
    if (isl >= 0) isl_joints[isl].push_back(j);
  }
  for (auto& c : contacts) {
    const int isl = island_of[c.a];
    if (isl >= 0) isl_cts[isl].push_back(&c);
  }

  Body<T> saved[STP_MAX_BODIES];
  for (int b = 0; b < n; ++b) saved[b] = st[b];
  int slot[STP_MAX_BODIES];
  for (int b = 0; b < n; ++b) slot[b] = -1;
  std::vector<Row<T>> rows;
  static thread_local BlockSys<T> H;
  T u[6 * STP_MAX_BODIES], rhs[6 * STP_MAX_BODIES];

  for (int isl = 0; isl < ni; ++isl) {
    const std::vector<int>& bodies = isl_bodies[isl];
    const int k = int(bodies.size());
    bool failed = false;
    if (isl_joints[isl].empty() && isl_cts[isl].empty()) {  // :517-523
      for (int b : bodies) {
        st[b].v = {dyn[b].vfree[0], dyn[b].vfree[1], dyn[b].vfree[2]};
        st[b].w = {dyn[b].vfree[3], dyn[b].vfree[4], dyn[b].vfree[5]};
      }
    } else {
      for (int i = 0; i < k; ++i) slot[bodies[i]] = i;
      build_rows(m, st, isl_joints[isl], isl_cts[isl], dyn, cf, rows);
      for (int i = 0; i < k; ++i) {
        const Body<T>& s = st[bodies[i]];
        T* ub = u + 6 * i;
        ub[0] = s.v.x; ub[1] = s.v.y; ub[2] = s.v.z;
        ub[3] = s.w.x; ub[4] = s.w.y; ub[5] = s.w.z;
      }
      for (int it = 0; it < cf.newton; ++it) {  // :541-548
        assemble(m, dyn, rows, isl_cts[isl], slot, bodies, u, cf, H, rhs);
        const KrylovResult kr = pcr(H, rhs, u, cf.tol, cf.kmax);
        if (kr.nonfinite_input) failed = true;  // reference: throws (krylov.cpp:113-114)
        stats.krylov += kr.iters;
        ++stats.newton;
        if (failed) break;
      }
      report(rows, isl_cts[isl], slot, u, cf);
      for (int i = 0; i < k; ++i) {
        Body<T>& s = st[bodies[i]];
        const T* ub = u + 6 * i;
        s.v = {ub[0], ub[1], ub[2]};
        s.w = {ub[3], ub[4], ub[5]};
      }
    }
    for (int b : bodies) {  // integrate, :562-569
      Body<T>& s = st[b];
      s.x = s.x + s.v * cf.dt;
      s.q = (Q<T>::expmap(s.w * cf.dt) * s.q).unit();
      if (!s.finite()) failed = true;
    }
    if (failed) {  // rollback, :580-593
      for (int b : bodies) st[b] = saved[b];
      stats.failed = true;
    }
  }
  return stats;
}

}  // namespace orc
