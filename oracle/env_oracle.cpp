// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
// reference arm may load the library built from this file.
//
// Env layer restatement + the `orc_*`
// C API shared by liboracle.so (restated physics) and
// oracle/_ref/libstampede_ref.so (the compiled reference physics).
// The design decisions for every gap SPEC leaves open are listed in
// DESIGN.md §"Env layer"; the GPU epilogue kernel implements the same ones.
#include "env_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

#include "phys_oracle.hpp"

namespace orc {

// terrain_height restated, collide.cpp:348-359
double stp_terrain_height_orc(const stp_static_box* boxes, int n, double x, double y) {
  double h = 0.0;
  for (int i = 0; i < n; ++i) {
    const stp_static_box& b = boxes[i];
    const double c = std::cos(b.yaw), s = std::sin(b.yaw);
    const double dx = x - b.center[0], dy = y - b.center[1];
    const double lx = c * dx + s * dy;
    const double ly = -s * dx + c * dy;
    if (std::abs(lx) <= b.half_extents[0] && std::abs(ly) <= b.half_extents[1])
      h = std::max(h, b.center[2] + b.half_extents[2]);
  }
  return h;
}

namespace {

thread_local std::string g_err;

int err(const std::string& m) {
  g_err = m;
  return STP_EINVAL;
}

// splitmix64 helpers restated from rng.hpp:25-37; draws are the 24-bit
// counter-based uniforms defined in DESIGN.md §RNG.
uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
uint64_t derive(uint64_t seed, uint64_t a, uint64_t b) { return mix64(mix64(mix64(seed) ^ a) ^ b); }
double unif(uint64_t stream, uint32_t k) { return double(mix64(stream + k) >> 40) * (1.0 / 16777216.0); }

enum : uint64_t { TAG_RESET = 1, TAG_FLAG = 2, TAG_PERTURB = 3, TAG_ACTION = 4 };
enum { C_FRAME = 0, C_FLAG = 1, C_FALL = 2, C_NEXTP = 3, C_EPISODE = 4, C_FLAGDRAW = 5, C_PERTDRAW = 6 };
constexpr int kGridCols = 64;

using V3 = V<double>;
using Q4 = Q<double>;

V3 v3(const double* p) { return {p[0], p[1], p[2]}; }
Q4 q4(const double* p) { return {p[0], p[1], p[2], p[3]}; }

// Quat::from_axis_angle, vec.hpp:130-135
Q4 axis_angle(const V3& axis, double ang) {
  const double h = 0.5 * ang;
  const double s = std::sin(h);
  const V3 a = axis.unit();
  return {std::cos(h), a.x * s, a.y * s, a.z * s};
}

// roll/pitch/yaw, vec.hpp:182-189
double yaw_of(const Q4& q) { return std::atan2(2 * (q.w * q.z + q.x * q.y), 1 - 2 * (q.y * q.y + q.z * q.z)); }
double roll_of(const Q4& q) { return std::atan2(2 * (q.w * q.x + q.y * q.z), 1 - 2 * (q.x * q.x + q.y * q.y)); }
double pitch_of(const Q4& q) {
  double s = 2 * (q.w * q.y - q.z * q.x);
  if (s > 1) s = 1;
  if (s < -1) s = -1;
  return std::asin(s);
}

// geometric height-map offsets: ratio 1.3 starting at 0.2 m
double geo_offset(int k) {
  const int a = k < 0 ? -k : k;
  const double d = 0.2 * (std::pow(1.3, a) - 1.0) / 0.3;
  return k < 0 ? -d : d;
}

int perturb_interval(const World& w, uint64_t stream) {
  const int span = w.task.perturb_max - w.task.perturb_min + 1;
  int k = int(std::floor(unif(stream, 0) * span));
  if (k >= span) k = span - 1;
  return w.task.perturb_min + k;
}

bool perturb_enabled(const World& w) { return w.task.perturb_max > 0 && w.task.perturb_max >= w.task.perturb_min; }

void draw_flag_target(World& w, int e) {
  const uint64_t genv = uint64_t(w.env_offset + e);
  int32_t* c = &w.counters[size_t(e) * 8];
  const uint64_t s = derive(w.seed, TAG_FLAG, (genv << 32) | uint32_t(c[C_FLAGDRAW]));
  c[C_FLAGDRAW] += 1;
  const double r = w.task.target_radius * std::sqrt(unif(s, 0));
  const double phi = 2.0 * M_PI * unif(s, 1);
  const double* root = w.body(e, w.model.root);
  w.target[2 * e] = root[0] + r * std::cos(phi);
  w.target[2 * e + 1] = root[1] + r * std::sin(phi);
}

// reset: grid placement + uniform noise on every DoF,
// propagated through hinge forward kinematics.
void reset_env(World& w, int e) {
  const stp_model& m = w.model;
  const int B = m.n_bodies, J = m.n_joints;
  const uint64_t genv = uint64_t(w.env_offset + e);
  int32_t* c = &w.counters[size_t(e) * 8];
  const uint64_t s = derive(w.seed, TAG_RESET, (genv << 32) | uint32_t(c[C_EPISODE]));
  c[C_EPISODE] += 1;
  const double a = w.task.reset_noise;
  auto noise = [&](uint32_t k) { return a * (2.0 * unif(s, k) - 1.0); };
  const double gx = double(genv % kGridCols) * w.task.spacing;
  const double gy = double(genv / kGridCols) * w.task.spacing;

  V3 x[STP_MAX_BODIES], v[STP_MAX_BODIES], om[STP_MAX_BODIES];
  Q4 q[STP_MAX_BODIES];
  const int r = m.root;
  const double* rs = m.rest_state[r];
  x[r] = {rs[0] + gx + noise(0), rs[1] + gy + noise(1), rs[2] + noise(2)};
  const V3 rv{noise(3), noise(4), noise(5)};
  q[r] = (Q4::expmap(rv) * q4(rs + 3)).unit();
  v[r] = {noise(6 + J), noise(7 + J), noise(8 + J)};
  om[r] = {noise(9 + J), noise(10 + J), noise(11 + J)};
  for (int j = 0; j < J; ++j) {
    const stp_joint& d = m.joints[j];
    const int p = d.parent, ch = d.child;
    const double th = noise(6 + j);
    const double thd = noise(12 + J + j);
    const V3 axc = v3(d.axis_child);
    q[ch] = q[p] * q4(d.rest_relative) * axis_angle(axc, th);
    const V3 anchor = x[p] + q[p].rot(v3(d.anchor_parent));
    x[ch] = anchor - q[ch].rot(v3(d.anchor_child));
    om[ch] = om[p] + q[ch].rot(axc) * thd;
    v[ch] = v[p] + om[p].cross(anchor - x[p]) - om[ch].cross(anchor - x[ch]);
  }
  for (int b = 0; b < B; ++b) {
    double* st = w.body(e, b);
    if (b != r && m.bodies[b].is_static) {  // static bodies keep the rest pose
      std::memcpy(st, m.rest_state[b], sizeof(double) * STP_STATE_STRIDE);
      st[0] += gx;
      st[1] += gy;
      continue;
    }
    st[0] = x[b].x; st[1] = x[b].y; st[2] = x[b].z;
    st[3] = q[b].w; st[4] = q[b].x; st[5] = q[b].y; st[6] = q[b].z;
    st[7] = v[b].x; st[8] = v[b].y; st[9] = v[b].z;
    st[10] = om[b].x; st[11] = om[b].y; st[12] = om[b].z;
  }
  c[C_FRAME] = 0;
  c[C_FLAG] = 0;
  c[C_FALL] = 0;
  if (w.task.target_refresh > 0) {
    draw_flag_target(w, e);
  } else {  // Ant / Humanoid: a point 1000 m straight ahead of spawn
    w.target[2 * e] = x[r].x + 1000.0;
    w.target[2 * e + 1] = x[r].y;
  }
  if (perturb_enabled(w)) {
    const uint64_t ps = derive(w.seed, TAG_PERTURB, (genv << 32) | uint32_t(c[C_PERTDRAW]));
    c[C_NEXTP] = perturb_interval(w, ps);
  } else {
    c[C_NEXTP] = -1;
  }
  for (int j = 0; j < J; ++j) w.last_tau[size_t(e) * J + j] = 0.0;
  for (int f = 0; f < STP_MAX_FEET; ++f) w.feet[size_t(e) * STP_MAX_FEET + f] = 0;
}

int obs_dim(const World& w) {
  return 11 + 3 * w.model.n_joints + w.model.n_feet + (w.task.height_map ? 165 : 0);
}

// observation, SPEC.md:243-246 / PAPER.md Table 2
void make_obs(World& w, int e, double* o) {
  const stp_model& m = w.model;
  const int J = m.n_joints;
  const double* rs = w.body(e, m.root);
  const Q4 q = q4(rs + 3);
  const double yaw = yaw_of(q);
  const double cy = std::cos(yaw), sy = std::sin(yaw);
  int k = 0;
  o[k++] = rs[2];
  o[k++] = roll_of(q);
  o[k++] = pitch_of(q);
  o[k++] = cy * rs[7] + sy * rs[8];
  o[k++] = -sy * rs[7] + cy * rs[8];
  o[k++] = rs[9];
  o[k++] = cy * rs[10] + sy * rs[11];
  o[k++] = -sy * rs[10] + cy * rs[11];
  o[k++] = rs[12];
  const double dx = w.target[2 * e] - rs[0], dy = w.target[2 * e + 1] - rs[1];
  const double th = std::atan2(dy, dx) - yaw;
  o[k++] = std::sin(th);
  o[k++] = std::cos(th);
  for (int j = 0; j < J; ++j) {
    const stp_joint& d = m.joints[j];
    const double* p = w.body(e, d.parent);
    const double* c = w.body(e, d.child);
    const Q4 rel = q4(p + 3).conj() * q4(c + 3);  // joint_angle, solver.cpp:405-411
    Q4 dq = q4(d.rest_relative).conj() * rel;
    if (dq.w < 0) dq = {-dq.w, -dq.x, -dq.y, -dq.z};
    const double proj = dq.x * d.axis_child[0] + dq.y * d.axis_child[1] + dq.z * d.axis_child[2];
    o[k + j] = 2.0 * std::atan2(proj, dq.w);
    const V3 axw = q4(c + 3).rot(v3(d.axis_child));  // joint_velocity, :413-417
    o[k + J + j] = axw.dot(v3(c + 10) - v3(p + 10));
    o[k + 2 * J + j] = w.last_tau[size_t(e) * J + j];
  }
  k += 3 * J;
  for (int f = 0; f < m.n_feet; ++f) o[k++] = w.feet[size_t(e) * STP_MAX_FEET + f] ? 1.0 : 0.0;
  if (w.task.height_map) {
    for (int i = 0; i < 15; ++i)
      for (int jj = 0; jj < 11; ++jj) {
        const double fx = geo_offset(i - 7), fy = geo_offset(jj - 5);
        const double px = rs[0] + cy * fx - sy * fy;
        const double py = rs[1] + sy * fx + cy * fy;
        o[k++] = stp_terrain_height_orc(w.boxes.data(), int(w.boxes.size()), px, py) - rs[2];
      }
  }
}

}  // namespace

namespace {

// Restated physics backend: per env step_env<T> on a few host threads.
template <class T>
struct Restated {
  static void run(World& w, const double* torques, int e0, int e1) {
    Model<T> m;
    m.load(w.model);
    Cfg<T> cf;
    cf.load(w.cfg);
    std::vector<Box<T>> boxes;
    for (const auto& b : w.boxes) boxes.push_back(make_box<T>(b));
    const int B = w.nb(), J = w.nj();
    std::vector<Contact<T>> cts;
    for (int e = e0; e < e1; ++e) {
      Body<T> st[STP_MAX_BODIES];
      V<T> fext[STP_MAX_BODIES], text[STP_MAX_BODIES];
      for (int b = 0; b < B; ++b) {
        const double* s = w.body(e, b);
        st[b].x = {T(s[0]), T(s[1]), T(s[2])};
        st[b].q = {T(s[3]), T(s[4]), T(s[5]), T(s[6])};
        st[b].v = {T(s[7]), T(s[8]), T(s[9])};
        st[b].w = {T(s[10]), T(s[11]), T(s[12])};
        const double* l = w.loads.data() + (size_t(e) * B + b) * 6;
        fext[b] = {T(l[0]), T(l[1]), T(l[2])};
        text[b] = {T(l[3]), T(l[4]), T(l[5])};
      }
      T tau[STP_MAX_JOINTS];
      for (int j = 0; j < J; ++j) tau[j] = T(torques[size_t(e) * J + j]);
      const StepStats ss = step_env(m, cf, boxes, st, tau, fext, text, cts);
      for (int b = 0; b < B; ++b) {
        double* s = w.body(e, b);
        s[0] = st[b].x.x; s[1] = st[b].x.y; s[2] = st[b].x.z;
        s[3] = st[b].q.w; s[4] = st[b].q.x; s[5] = st[b].q.y; s[6] = st[b].q.z;
        s[7] = st[b].v.x; s[8] = st[b].v.y; s[9] = st[b].v.z;
        s[10] = st[b].w.x; s[11] = st[b].w.y; s[12] = st[b].w.z;
      }
      auto& out = w.contacts[e];
      out.clear();
      for (const auto& c : cts) {
        ContactRec r{};
        r.a = c.a;
        r.b = c.b;
        for (int i = 0; i < 3; ++i) {
          r.p[i] = c.p[i];
          r.n[i] = c.n[i];
          r.pt[i] = c.pt[i];
        }
        r.sep = c.sep;
        r.pn = c.pn;
        out.push_back(r);
      }
      w.newton[e] = ss.newton;
      w.krylov[e] = ss.krylov;
      w.failed[e] = ss.failed ? 1 : 0;
    }
  }
};

// closest points between segments (collide.cpp:219-249, Ericson)
void seg_closest(const V<double>& p1, const V<double>& q1, const V<double>& p2, const V<double>& q2,
                 V<double>& c1, V<double>& c2) {
  const V<double> d1 = q1 - p1, d2 = q2 - p2, r = p1 - p2;
  const double a = d1.dot(d1), e = d2.dot(d2), f = d2.dot(r);
  auto cl = [](double v) { return std::min(std::max(v, 0.0), 1.0); };
  double s = 0, t = 0;
  if (a <= 1e-12 && e <= 1e-12) {
  } else if (a <= 1e-12) {
    t = cl(f / e);
  } else {
    const double c = d1.dot(r);
    if (e <= 1e-12) {
      s = cl(-c / a);
    } else {
      const double b = d1.dot(d2), den = a * e - b * b;
      if (den > 1e-12) s = cl((b * f - c * e) / den);
      t = (b * s + f) / e;
      if (t < 0) {
        t = 0;
        s = cl(-c / a);
      } else if (t > 1) {
        t = 1;
        s = cl((b - c) / a);
      }
    }
  }
  c1 = p1 + d1 * s;
  c2 = p2 + d2 * t;
}

// The restatement solves every env as its own island.  With
// Scene::inter_agent_collisions on (HFH) that is the reference's
// behaviour only while no two agents touch (collide.cpp:300-343 finds no
// pair): check exactly that, and fail loudly otherwise (contact-merged
// islands are checked against the compiled reference instead).
void require_no_inter_agent_contacts(const World& w) {
  Model<double> m;
  m.load(w.model);
  const double margin = w.cfg.contact_margin;
  const int B = w.nb();
  std::vector<Shape<double>> sh(size_t(w.n) * B);
  std::vector<char> ok(size_t(w.n) * B);
  std::vector<V<double>> lo(w.n, V<double>{1e300, 1e300, 1e300}), hi(w.n, V<double>{-1e300, -1e300, -1e300});
  for (int e = 0; e < w.n; ++e)
    for (int b = 0; b < B; ++b) {
      const double* s = w.state.data() + (size_t(e) * B + b) * STP_STATE_STRIDE;
      Body<double> st;
      st.x = {s[0], s[1], s[2]};
      st.q = {s[3], s[4], s[5], s[6]};
      const size_t i = size_t(e) * B + b;
      sh[i] = world_shape(m, b, st);
      ok[i] = !m.is_static[b] && m.shape[b] != STP_BOX;
      if (ok[i]) {
        lo[e] = {std::min(lo[e].x, sh[i].lo.x), std::min(lo[e].y, sh[i].lo.y), std::min(lo[e].z, sh[i].lo.z)};
        hi[e] = {std::max(hi[e].x, sh[i].hi.x), std::max(hi[e].y, sh[i].hi.y), std::max(hi[e].z, sh[i].hi.z)};
      }
    }
  auto over = [&](const V<double>& al, const V<double>& ah, const V<double>& bl, const V<double>& bh) {
    return al.x <= bh.x + margin && bl.x <= ah.x + margin && al.y <= bh.y + margin && bl.y <= ah.y + margin &&
           al.z <= bh.z + margin && bl.z <= ah.z + margin;  // aabb_overlap, collide.cpp:80-84
  };
  for (int e1 = 0; e1 < w.n; ++e1)
    for (int e2 = e1 + 1; e2 < w.n; ++e2) {
      if (!over(lo[e1], hi[e1], lo[e2], hi[e2])) continue;
      for (int a = 0; a < B; ++a)
        for (int b = 0; b < B; ++b) {
          const Shape<double>& A = sh[size_t(e1) * B + a];
          const Shape<double>& Bs = sh[size_t(e2) * B + b];
          if (!ok[size_t(e1) * B + a] || !ok[size_t(e2) * B + b] || !over(A.lo, A.hi, Bs.lo, Bs.hi)) continue;
          V<double> ca, cb;
          seg_closest(A.p0, A.p1, Bs.p0, Bs.p1, ca, cb);
          const V<double> d = ca - cb;
          if (d.norm() - A.r - Bs.r < margin)
            throw std::runtime_error("restated physics: agents " + std::to_string(e1) + " and " + std::to_string(e2) +
                                     " touch; contact-merged islands are only in the compiled reference backend");
        }
    }
}

struct RestatedPhysics : PhysicsBackend {
  const char* name() const override { return "restatement"; }
  void step(World& w, const double* torques) override {
    if (w.task.inter_agent_collisions) require_no_inter_agent_contacts(w);
    const int nt = std::max(1, std::min(w.nthreads, w.n));
    auto body = [&](int e0, int e1) {
      if (w.precision == 0) Restated<float>::run(w, torques, e0, e1);
      else Restated<double>::run(w, torques, e0, e1);
    };
    if (nt == 1) {
      body(0, w.n);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < nt; ++t) {
        const int e0 = int(int64_t(w.n) * t / nt), e1 = int(int64_t(w.n) * (t + 1) / nt);
        th.emplace_back(body, e0, e1);
      }
      for (auto& t : th) t.join();
    }
    std::fill(w.loads.begin(), w.loads.end(), 0.0);  // clear_external_loads, scene.cpp:75-78
  }
};

}  // namespace

int set_error(const std::string& message) { return err(message); }

std::unique_ptr<PhysicsBackend> make_restated_backend() { return std::make_unique<RestatedPhysics>(); }

}  // namespace orc

// ---------------------------------------------------------------------------
// C API
// ---------------------------------------------------------------------------
using orc::World;

extern "C" {

typedef struct orc_world orc_world;

const char* orc_last_error(void) { return orc::g_err.c_str(); }

orc_world* orc_create(const stp_model* model, const stp_task* task, const stp_step_config* cfg, int32_t n_envs,
                      uint64_t seed, int64_t env_offset, int32_t nthreads, int32_t precision,
                      int32_t use_reference) {
  if (!model || !task || !cfg || n_envs <= 0) {
    orc::err("orc_create: bad arguments");
    return nullptr;
  }
  auto* w = new World();
  w->model = *model;
  w->task = *task;
  w->cfg = *cfg;
  w->n = n_envs;
  w->seed = seed;
  w->env_offset = env_offset;
  w->nthreads = std::max(1, nthreads);
  w->precision = precision;
  const int B = model->n_bodies, J = model->n_joints;
  w->state.assign(size_t(n_envs) * B * STP_STATE_STRIDE, 0.0);
  w->loads.assign(size_t(n_envs) * B * 6, 0.0);
  w->contacts.assign(n_envs, {});
  w->newton.assign(n_envs, 0);
  w->krylov.assign(n_envs, 0);
  w->failed.assign(n_envs, 0);
  w->target.assign(size_t(n_envs) * 2, 0.0);
  w->counters.assign(size_t(n_envs) * 8, 0);
  w->last_tau.assign(size_t(n_envs) * J, 0.0);
  w->feet.assign(size_t(n_envs) * STP_MAX_FEET, 0);
  try {
    w->physics = use_reference ? orc::make_reference_backend() : orc::make_restated_backend();
  } catch (const std::exception& ex) {
    orc::err(std::string("orc_create: ") + ex.what());
    delete w;
    return nullptr;
  }
  if (!w->physics) {
    orc::err("orc_create: reference backend not built into this library");
    delete w;
    return nullptr;
  }
  for (int e = 0; e < n_envs; ++e) orc::reset_env(*w, e);
  return reinterpret_cast<orc_world*>(w);
}

void orc_destroy(orc_world* h) { delete reinterpret_cast<World*>(h); }

const char* orc_backend(orc_world* h) { return reinterpret_cast<World*>(h)->physics->name(); }

int32_t orc_obs_dim(orc_world* h) { return orc::obs_dim(*reinterpret_cast<World*>(h)); }

int orc_set_terrain(orc_world* h, const stp_static_box* boxes, int32_t n) {
  auto* w = reinterpret_cast<World*>(h);
  w->boxes.assign(boxes, boxes + n);
  return STP_OK;
}

int orc_set_state(orc_world* h, const double* s) {
  auto* w = reinterpret_cast<World*>(h);
  std::memcpy(w->state.data(), s, w->state.size() * sizeof(double));
  return STP_OK;
}
int orc_get_state(orc_world* h, double* s) {
  auto* w = reinterpret_cast<World*>(h);
  std::memcpy(s, w->state.data(), w->state.size() * sizeof(double));
  return STP_OK;
}
int orc_set_external_loads(orc_world* h, const double* l) {
  auto* w = reinterpret_cast<World*>(h);
  std::memcpy(w->loads.data(), l, w->loads.size() * sizeof(double));
  return STP_OK;
}

int orc_physics_step(orc_world* h, const double* torques) {
  auto* w = reinterpret_cast<World*>(h);
  try {
    w->physics->step(*w, torques);
  } catch (const std::exception& ex) {
    return orc::err(std::string("orc_physics_step: ") + ex.what());
  }
  return STP_OK;
}

int orc_reset(orc_world* h, const uint8_t* mask, double* obs) {
  auto* w = reinterpret_cast<World*>(h);
  const int od = orc::obs_dim(*w);
  for (int e = 0; e < w->n; ++e) {
    if (!mask || mask[e]) orc::reset_env(*w, e);
    if (obs) orc::make_obs(*w, e, obs + size_t(e) * od);
  }
  return STP_OK;
}

// env_step, SPEC.md:270-278 (+ compute_reward :279-305, flagrun :306-314,
// perturbations :324-332, termination :334-343); order documented in
// DESIGN.md §"Env layer".
int orc_step(orc_world* h, const double* actions, double* obs, double* reward, uint8_t* done) {
  auto* w = reinterpret_cast<World*>(h);
  const stp_model& m = w->model;
  const int N = w->n, B = m.n_bodies, J = m.n_joints, R = m.root;
  const double dt = w->cfg.dt;
  std::vector<double> tau(size_t(N) * J);
  std::vector<double> prev_xy(size_t(N) * 2);
  std::vector<uint8_t> perturbed(N, 0);
  for (int e = 0; e < N; ++e) {
    for (int j = 0; j < J; ++j) tau[size_t(e) * J + j] = actions[size_t(e) * J + j] * m.joints[j].max_torque;
    int32_t* c = &w->counters[size_t(e) * 8];
    if (orc::perturb_enabled(*w) && c[orc::C_FRAME] == c[orc::C_NEXTP]) {
      const uint64_t genv = uint64_t(w->env_offset + e);
      const uint64_t ps = orc::derive(w->seed, orc::TAG_PERTURB, (genv << 32) | uint32_t(c[orc::C_PERTDRAW]));
      const double f = w->task.perturb_force_lo + (w->task.perturb_force_hi - w->task.perturb_force_lo) * orc::unif(ps, 1);
      const double phi = 2.0 * M_PI * orc::unif(ps, 2);
      double* l = w->loads.data() + (size_t(e) * B + R) * 6;
      l[0] += f * std::cos(phi);
      l[1] += f * std::sin(phi);
      perturbed[e] = 1;
    }
    const double* rs = w->body(e, R);
    prev_xy[2 * e] = rs[0];
    prev_xy[2 * e + 1] = rs[1];
  }
  int rc = orc_physics_step(h, tau.data());
  if (rc) return rc;
  const int od = orc::obs_dim(*w);
  for (int e = 0; e < N; ++e) {
    int32_t* c = &w->counters[size_t(e) * 8];
    const double* rs = w->body(e, R);
    // feet flags: foot has >= 1 contact against static geometry this step
    for (int f = 0; f < STP_MAX_FEET; ++f) w->feet[size_t(e) * STP_MAX_FEET + f] = 0;
    for (const auto& ct : w->contacts[e])
      for (int f = 0; f < m.n_feet; ++f)
        if (ct.a == m.feet[f] && ct.b < 0) w->feet[size_t(e) * STP_MAX_FEET + f] = 1;
    double r = 0.0;
    const bool failed = w->failed[e] != 0;
    if (!failed) {
      // compute_reward, PAPER.md:463-483 / SPEC.md:279-305
      const double tx = w->target[2 * e], ty = w->target[2 * e + 1];
      const double ox = tx - prev_xy[2 * e], oy = ty - prev_xy[2 * e + 1];
      const double od0 = std::sqrt(ox * ox + oy * oy);
      double S = 0.0;
      if (od0 > 0) S = ((rs[0] - prev_xy[2 * e]) * ox + (rs[1] - prev_xy[2 * e + 1]) * oy) / od0 / dt;
      const orc::Q4 q = orc::q4(rs + 3);
      const double yaw = orc::yaw_of(q);
      const double cth = std::cos(std::atan2(ty - rs[1], tx - rs[0]) - yaw);
      const double rhead = cth > 0.8 ? 1.0 : cth / 0.8;
      const double cvert = 1.0 - 2.0 * (q.x * q.x + q.y * q.y);
      const double rstand = cvert > 0.93 ? 1.0 : 0.0;
      double tcost = 0.0, ucost = 0.0;
      int nlim = 0;
      for (int j = 0; j < J; ++j) {
        const double u = actions[size_t(e) * J + j];
        tcost += std::abs(std::clamp(u, -1.0, 1.0));
        ucost += u * u;
        const stp_joint& d = m.joints[j];
        const double* p = w->body(e, d.parent);
        const double* ch = w->body(e, d.child);
        const orc::Q4 rel = orc::q4(p + 3).conj() * orc::q4(ch + 3);
        orc::Q4 dq = orc::q4(d.rest_relative).conj() * rel;
        if (dq.w < 0) dq = {-dq.w, -dq.x, -dq.y, -dq.z};
        const double proj = dq.x * d.axis_child[0] + dq.y * d.axis_child[1] + dq.z * d.axis_child[2];
        const double ang = 2.0 * std::atan2(proj, dq.w);
        if (ang - d.limit_lo < w->cfg.limit_activation || d.limit_hi - ang < w->cfg.limit_activation) ++nlim;
      }
      int nfeet = 0;
      for (int f = 0; f < m.n_feet; ++f) nfeet += w->feet[size_t(e) * STP_MAX_FEET + f];
      r = m.alive_bonus + S + 0.5 * rhead + 0.05 * rstand - 4.0 * tcost - 0.5 * ucost - 0.2 * nlim - double(nfeet);
    }
    const int frame_before = c[orc::C_FRAME];
    c[orc::C_FRAME] += 1;
    const bool low = rs[2] < m.fall_height;
    c[orc::C_FALL] = low ? c[orc::C_FALL] + 1 : 0;
    const bool fell = w->task.fall_grace > 0 ? c[orc::C_FALL] >= w->task.fall_grace : low;
    const bool d = failed || fell || c[orc::C_FRAME] >= w->task.episode_cap;
    if (perturbed[e]) {
      c[orc::C_PERTDRAW] += 1;
      const uint64_t genv = uint64_t(w->env_offset + e);
      const uint64_t ps = orc::derive(w->seed, orc::TAG_PERTURB, (genv << 32) | uint32_t(c[orc::C_PERTDRAW]));
      c[orc::C_NEXTP] = frame_before + orc::perturb_interval(*w, ps);
    }
    if (w->task.target_refresh > 0) {  // update_flagrun_targets
      c[orc::C_FLAG] += 1;
      const double dx = w->target[2 * e] - rs[0], dy = w->target[2 * e + 1] - rs[1];
      if (c[orc::C_FLAG] >= w->task.target_refresh || std::sqrt(dx * dx + dy * dy) < w->task.target_tolerance) {
        orc::draw_flag_target(*w, e);
        c[orc::C_FLAG] = 0;
      }
    }
    for (int j = 0; j < J; ++j)
      w->last_tau[size_t(e) * J + j] = std::clamp(actions[size_t(e) * J + j], -1.0, 1.0);
    if (reward) reward[e] = r;
    if (done) done[e] = d ? 1 : 0;
    if (d && w->task.auto_reset) orc::reset_env(*w, e);
    if (obs) orc::make_obs(*w, e, obs + size_t(e) * od);
  }
  return STP_OK;
}

int orc_random_actions(orc_world* h, double* actions, uint64_t step) {
  auto* w = reinterpret_cast<World*>(h);
  const int J = w->model.n_joints;
  for (int e = 0; e < w->n; ++e) {
    const uint64_t genv = uint64_t(w->env_offset + e);
    const uint64_t s = orc::derive(w->seed, orc::TAG_ACTION, (genv << 32) | uint32_t(step));
    for (int j = 0; j < J; ++j) actions[size_t(e) * J + j] = 2.0 * orc::unif(s, j) - 1.0;
  }
  return STP_OK;
}

int32_t orc_get_contacts(orc_world* h, int32_t capacity, int32_t* count, int32_t* body_a, int32_t* body_b,
                         double* point, double* normal, double* sep, double* pn, double* pt) {
  auto* w = reinterpret_cast<World*>(h);
  int32_t maxc = 0;
  for (int e = 0; e < w->n; ++e) {
    const auto& cs = w->contacts[e];
    maxc = std::max<int32_t>(maxc, int32_t(cs.size()));
    if (count) count[e] = int32_t(cs.size());
    for (int i = 0; i < int(cs.size()) && i < capacity; ++i) {
      const size_t s = size_t(e) * capacity + i;
      const auto& c = cs[i];
      if (body_a) body_a[s] = c.a;
      if (body_b) body_b[s] = c.b;
      for (int k = 0; k < 3; ++k) {
        if (point) point[3 * s + k] = c.p[k];
        if (normal) normal[3 * s + k] = c.n[k];
        if (pt) pt[3 * s + k] = c.pt[k];
      }
      if (sep) sep[s] = c.sep;
      if (pn) pn[s] = c.pn;
    }
  }
  return maxc;
}

int orc_get_report(orc_world* h, int32_t* newton, int32_t* krylov, uint8_t* failed) {
  auto* w = reinterpret_cast<World*>(h);
  for (int e = 0; e < w->n; ++e) {
    if (newton) newton[e] = w->newton[e];
    if (krylov) krylov[e] = w->krylov[e];
    if (failed) failed[e] = w->failed[e];
  }
  return STP_OK;
}

int orc_get_task_state(orc_world* h, double* target, int32_t* counters, double* last_tau) {
  auto* w = reinterpret_cast<World*>(h);
  if (target) std::memcpy(target, w->target.data(), w->target.size() * sizeof(double));
  if (counters) std::memcpy(counters, w->counters.data(), w->counters.size() * sizeof(int32_t));
  if (last_tau) std::memcpy(last_tau, w->last_tau.data(), w->last_tau.size() * sizeof(double));
  return STP_OK;
}

int orc_set_task_state(orc_world* h, const double* target, const int32_t* counters, const double* last_tau) {
  auto* w = reinterpret_cast<World*>(h);
  if (target) std::memcpy(w->target.data(), target, w->target.size() * sizeof(double));
  if (counters) std::memcpy(w->counters.data(), counters, w->counters.size() * sizeof(int32_t));
  if (last_tau) std::memcpy(w->last_tau.data(), last_tau, w->last_tau.size() * sizeof(double));
  return STP_OK;
}

// obs of the current state (after set_state / set_task_state), feet flags
// taken from the last physics step.
int orc_observe(orc_world* h, double* obs) {
  auto* w = reinterpret_cast<World*>(h);
  const int od = orc::obs_dim(*w);
  for (int e = 0; e < w->n; ++e) orc::make_obs(*w, e, obs + size_t(e) * od);
  return STP_OK;
}

double orc_terrain_height(const stp_static_box* boxes, int32_t n, double x, double y) {
  return orc::stp_terrain_height_orc(boxes, n, x, y);
}

}  // extern "C"

// Debug/parity hook: restated first Newton linearisation of env e
// (assemble_system, solver.cpp:419-446) as a dense matrix.
extern "C" int orc_first_system(orc_world* h, int e, const double* torques, double* Hd, double* rhs) {
  auto* w = reinterpret_cast<World*>(h);
  using T = double;
  orc::Model<T> m;
  m.load(w->model);
  orc::Cfg<T> cf;
  cf.load(w->cfg);
  const int B = m.nb;
  orc::Body<T> st[STP_MAX_BODIES];
  for (int b = 0; b < B; ++b) {
    const double* s = w->body(e, b);
    st[b].x = {s[0], s[1], s[2]};
    st[b].q = {s[3], s[4], s[5], s[6]};
    st[b].v = {s[7], s[8], s[9]};
    st[b].w = {s[10], s[11], s[12]};
  }
  std::vector<orc::Box<T>> boxes;
  std::vector<orc::Contact<T>> cts;
  orc::detect(m, st, boxes, cf.plane, cf.margin, cts);
  T tau[STP_MAX_JOINTS];
  for (int j = 0; j < m.nj; ++j) tau[j] = std::clamp(torques[j], -m.tmax[j], m.tmax[j]);
  orc::V<T> zero[STP_MAX_BODIES];
  orc::Dyn<T> dyn[STP_MAX_BODIES];
  orc::dynamics(m, st, tau, zero, zero, cf, dyn);
  std::vector<int> joints;
  for (int j = 0; j < m.nj; ++j) joints.push_back(j);
  std::vector<orc::Contact<T>*> cp;
  for (auto& c : cts) cp.push_back(&c);
  std::vector<orc::Row<T>> rows;
  orc::build_rows(m, st, joints, cp, dyn, cf, rows);
  int slot[STP_MAX_BODIES];
  std::vector<int> sb;
  for (int b = 0; b < B; ++b) {
    slot[b] = m.is_static[b] ? -1 : int(sb.size());
    if (!m.is_static[b]) sb.push_back(b);
  }
  T u[6 * STP_MAX_BODIES];
  for (size_t i = 0; i < sb.size(); ++i) {
    const auto& s = st[sb[i]];
    u[6 * i + 0] = s.v.x; u[6 * i + 1] = s.v.y; u[6 * i + 2] = s.v.z;
    u[6 * i + 3] = s.w.x; u[6 * i + 4] = s.w.y; u[6 * i + 5] = s.w.z;
  }
  static orc::BlockSys<T> H;
  orc::assemble(m, dyn, rows, cp, slot, sb, u, cf, H, rhs);
  const int n = 6 * int(sb.size());
  for (int i = 0; i < n * n; ++i) Hd[i] = 0;
  for (int i = 0; i < H.k; ++i)
    for (int j = 0; j < H.k; ++j)
      if (H.present[i][j])
        for (int r = 0; r < 6; ++r)
          for (int c = 0; c < 6; ++c) Hd[(6 * i + r) * n + 6 * j + c] = H.blk[i][j][6 * r + c];
  return int(cts.size());
}
