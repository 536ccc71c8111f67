// Host-side configuration helpers of the C-ABI: bundled Ant / Humanoid
// assets, StepConfig / TaskConfig defaults, model validation, terrain
// generation and the terrain height query.
//
// The reference ships no asset (SPEC.md:182-232 is prose only),
// so the articulations are defined here once, as data, and handed to both
// the GPU path and the CPU oracle through the same stp_model struct.
// Decisions follow SPEC.md:219-223 (capsule humanoid, 40 kg, 21 actuated
// hinges, "28 DoF" = 7 root + 21; ant = torso sphere + 4 two-segment legs)
// and DESIGN.md §A0.  Multi-DoF hips / shoulders / abdomen / ankles are
// chains of hinges through light link bodies because JointDesc is
// hinge-only (types.hpp:58-71): 22 bodies for 21 hinges.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "stampede_sim.h"
#include "stp_error.h"
#include "stp_rng.h"

namespace {

struct V3 {
  double x, y, z;
};
struct Q4 {
  double w, x, y, z;
};

V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 scl(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
V3 crs(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double nrm(V3 a) { return std::sqrt(dot(a, a)); }
V3 unit(V3 a) { return scl(a, 1.0 / nrm(a)); }
Q4 qmul(Q4 a, Q4 b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
Q4 qconj(Q4 q) { return {q.w, -q.x, -q.y, -q.z}; }
V3 qrot(Q4 q, V3 v) {
  const V3 u{q.x, q.y, q.z};
  const V3 t = scl(crs(u, v), 2.0);
  const V3 c = crs(u, t);
  return {v.x + q.w * t.x + c.x, v.y + q.w * t.y + c.y, v.z + q.w * t.z + c.z};
}
V3 qrot_inv(Q4 q, V3 v) { return qrot(qconj(q), v); }
// shortest-arc rotation taking +z onto direction d
Q4 z_to(V3 d) {
  d = unit(d);
  const double c = d.z;
  if (c > 1.0 - 1e-12) return {1, 0, 0, 0};
  if (c < -1.0 + 1e-12) return {0, 1, 0, 0};
  const V3 axis = unit(crs({0, 0, 1}, d));
  const double ang = std::acos(c);
  const double s = std::sin(0.5 * ang);
  return {std::cos(0.5 * ang), axis.x * s, axis.y * s, axis.z * s};
}

constexpr double kDeg = M_PI / 180.0;

struct Builder {
  stp_model* m;
  explicit Builder(stp_model* out, const char* name) : m(out) {
    std::memset(m, 0, sizeof(*m));
    std::snprintf(m->name, sizeof(m->name), "%s", name);
  }
  // Body whose principal frame has local z along `axis_dir` (capsules) so
  // the inertia is diagonal in the body frame (types.hpp:42 "principal").
  int body(int shape, double radius, double half_length, V3 pos, V3 axis_dir, double mass) {
    const int b = m->n_bodies++;
    stp_body& d = m->bodies[b];
    d.shape = shape;
    d.radius = radius;
    d.half_length = half_length;
    d.local_rot[0] = 1;
    d.mass = mass;
    if (shape == STP_SPHERE) {
      const double i = 0.4 * mass * radius * radius;
      d.inertia_diag[0] = d.inertia_diag[1] = d.inertia_diag[2] = i;
    } else {
      // solid capsule approximated as a cylinder of length 2(h + r)
      const double len = 2.0 * (half_length + radius);
      const double ia = 0.5 * mass * radius * radius;
      const double ip = mass * (3.0 * radius * radius + len * len) / 12.0;
      d.inertia_diag[0] = d.inertia_diag[1] = ip;
      d.inertia_diag[2] = ia;
    }
    const Q4 q = shape == STP_SPHERE ? Q4{1, 0, 0, 0} : z_to(axis_dir);
    double* s = m->rest_state[b];
    s[0] = pos.x; s[1] = pos.y; s[2] = pos.z;
    s[3] = q.w; s[4] = q.x; s[5] = q.y; s[6] = q.z;
    return b;
  }
  // Hinge with world anchor / world axis at the rest pose (angle zero).
  void joint(int parent, int child, V3 anchor, V3 axis, double lo_deg, double hi_deg,
             double max_torque) {
    const int j = m->n_joints++;
    stp_joint& d = m->joints[j];
    d.parent = parent;
    d.child = child;
    const double* sp = m->rest_state[parent];
    const double* sc = m->rest_state[child];
    const V3 xp{sp[0], sp[1], sp[2]}, xc{sc[0], sc[1], sc[2]};
    const Q4 qp{sp[3], sp[4], sp[5], sp[6]}, qc{sc[3], sc[4], sc[5], sc[6]};
    const V3 ap = qrot_inv(qp, sub(anchor, xp));
    const V3 ac = qrot_inv(qc, sub(anchor, xc));
    const V3 axp = unit(qrot_inv(qp, unit(axis)));
    const V3 axc = unit(qrot_inv(qc, unit(axis)));
    const Q4 rest = qmul(qconj(qp), qc);
    d.anchor_parent[0] = ap.x; d.anchor_parent[1] = ap.y; d.anchor_parent[2] = ap.z;
    d.anchor_child[0] = ac.x; d.anchor_child[1] = ac.y; d.anchor_child[2] = ac.z;
    d.axis_parent[0] = axp.x; d.axis_parent[1] = axp.y; d.axis_parent[2] = axp.z;
    d.axis_child[0] = axc.x; d.axis_child[1] = axc.y; d.axis_child[2] = axc.z;
    d.rest_relative[0] = rest.w; d.rest_relative[1] = rest.x;
    d.rest_relative[2] = rest.y; d.rest_relative[3] = rest.z;
    d.limit_lo = lo_deg * kDeg;
    d.limit_hi = hi_deg * kDeg;
    d.max_torque = max_torque;
  }
};

// Ant: torso sphere + 4 legs of (upper, lower) capsules, 8 hinges
// ("4 legs and 8 controllable joints").
// Standing pose: torso centre 0.55 m, lower legs reach 5 mm above ground.
void build_ant(stp_model* m) {
  Builder b(m, "ant");
  const double zt = 0.55;
  b.body(STP_SPHERE, 0.25, 0, {0, 0, zt}, {0, 0, 1}, 5.0);
  for (int k = 0; k < 4; ++k) {
    const double phi = (45.0 + 90.0 * k) * kDeg;
    const V3 d{std::cos(phi), std::sin(phi), 0};
    const V3 hip{0.2 * d.x, 0.2 * d.y, zt};
    const V3 knee{0.5 * d.x, 0.5 * d.y, zt};
    const V3 foot{0.72 * d.x, 0.72 * d.y, 0.085};
    const V3 mid_u{0.5 * (hip.x + knee.x), 0.5 * (hip.y + knee.y), zt};
    const int up = b.body(STP_CAPSULE, 0.08, 0.15, mid_u, d, 1.0);
    const V3 seg = sub(foot, knee);
    const V3 mid_l{knee.x + 0.5 * seg.x, knee.y + 0.5 * seg.y, knee.z + 0.5 * seg.z};
    const int lo = b.body(STP_CAPSULE, 0.08, 0.5 * nrm(seg), mid_l, seg, 1.5);
    b.joint(0, up, hip, {0, 0, 1}, -30, 30, 30.0);
    b.joint(up, lo, knee, {-d.y, d.x, 0}, -40, 40, 30.0);
    m->feet[m->n_feet++] = lo;
  }
  m->root = 0;
  m->fall_height = 0.28;
  m->alive_bonus = 0.5;   // PAPER.md App. C
}

// Humanoid: 13 capsule segments + 9 light hinge links = 22 bodies,
// 21 actuated hinges in the DeepMind-control layout (abdomen z/y/x, hips
// x/z/y, knees, ankles y/x, shoulders 1/2, elbows), 40 kg.
// Ranges and gears (tau_max) follow that layout.  Faces +x, stands on z = 0.
void build_humanoid(stp_model* m) {
  Builder b(m, "humanoid");
  const V3 Z{0, 0, 1}, Y{0, 1, 0}, X{1, 0, 0}, NY{0, -1, 0};
  const double link_m = 0.5, link_r = 0.05;
  const int torso = b.body(STP_CAPSULE, 0.11, 0.16, {0, 0, 1.33}, Z, 7.6);
  const int abd = b.body(STP_SPHERE, link_r, 0, {0, 0, 1.10}, Z, link_m);
  const int lwaist = b.body(STP_CAPSULE, 0.09, 0.05, {0, 0, 1.03}, Y, 2.5);
  const int pelvis = b.body(STP_CAPSULE, 0.10, 0.07, {0, 0, 0.90}, Y, 4.8);
  b.joint(torso, abd, {0, 0, 1.10}, Z, -45, 45, 40);
  b.joint(abd, lwaist, {0, 0, 1.10}, Y, -75, 30, 40);
  b.joint(lwaist, pelvis, {0, 0, 0.97}, X, -35, 35, 40);
  for (int side = 0; side < 2; ++side) {  // 0 = right (y < 0), 1 = left
    const double s = side == 0 ? -1.0 : 1.0;
    const double y = 0.1 * s;
    const V3 hip{0, y, 0.86}, knee{0, y, 0.47}, ankle{0, y, 0.10};
    const int hx = b.body(STP_SPHERE, link_r, 0, hip, Z, link_m);
    const int hz = b.body(STP_SPHERE, link_r, 0, hip, Z, link_m);
    const int thigh = b.body(STP_CAPSULE, 0.06, 0.135, {0, y, 0.665}, Z, 4.3);
    const int shin = b.body(STP_CAPSULE, 0.05, 0.13, {0, y, 0.29}, Z, 2.5);
    const int al = b.body(STP_SPHERE, 0.04, 0, ankle, Z, link_m);
    const int foot = b.body(STP_CAPSULE, 0.045, 0.07, {0.03, y, 0.046}, X, 1.0);
    // mirrored ranges: rotations about x and z flip sign on the left side
    if (side == 0) {
      b.joint(pelvis, hx, hip, X, -25, 5, 40);
      b.joint(hx, hz, hip, Z, -60, 35, 40);
    } else {
      b.joint(pelvis, hx, hip, X, -5, 25, 40);
      b.joint(hx, hz, hip, Z, -35, 60, 40);
    }
    b.joint(hz, thigh, hip, Y, -110, 20, 120);
    b.joint(thigh, shin, knee, NY, -150, 5, 80);
    b.joint(shin, al, ankle, Y, -50, 50, 20);
    b.joint(al, foot, ankle, X, -50, 50, 20);
    m->feet[m->n_feet++] = foot;
  }
  for (int side = 0; side < 2; ++side) {
    const double s = side == 0 ? -1.0 : 1.0;
    const double y = 0.19 * s;
    const V3 shoulder{0, y, 1.42}, elbow{0, y, 1.14};
    const int sl = b.body(STP_SPHERE, 0.04, 0, shoulder, Z, link_m);
    const int upper = b.body(STP_CAPSULE, 0.04, 0.10, {0, y, 1.28}, Z, 1.4);
    const int lower = b.body(STP_CAPSULE, 0.035, 0.11, {0, y, 0.99}, Z, 1.1);
    if (side == 0) b.joint(torso, sl, shoulder, X, -85, 60, 20);
    else b.joint(torso, sl, shoulder, X, -60, 85, 20);
    b.joint(sl, upper, shoulder, Y, -85, 60, 20);
    b.joint(upper, lower, elbow, Y, -90, 50, 40);
  }
  m->root = torso;
  m->fall_height = 0.8;
  m->alive_bonus = 2.0;  // PAPER.md App. C
}

bool finite3(const double* v) {
  return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
}
double norm3(const double* v) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

}  // namespace

extern "C" {

int stp_abi_version(void) { return STP_ABI_VERSION; }

const char* stp_last_error(void) { return stp::last_error_cstr(); }

void stp_struct_sizes(int64_t out[7]) {
  out[0] = sizeof(stp_body);
  out[1] = sizeof(stp_joint);
  out[2] = sizeof(stp_model);
  out[3] = sizeof(stp_step_config);
  out[4] = sizeof(stp_static_box);
  out[5] = sizeof(stp_terrain_spec);
  out[6] = sizeof(stp_task);
}

void stp_default_step_config(stp_step_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->dt = 1.0 / 120.0;
  c->newton_iters = 4;
  c->krylov_tol = 1e-6;
  c->krylov_max_iters = 16;
  c->contact_margin = 0.02;
  c->baumgarte = 0.2;
  c->joint_hardness = 3000;
  c->contact_hardness = 300;
  c->limit_hardness = 6000;
  c->friction_smoothing = 1e-3;
  c->limit_activation = 0.05;
  c->gravity[2] = -9.8;
  c->has_ground_plane = 1;
  c->reference_alias_quirk = 1;
}

int stp_builtin_model(const char* name, stp_model* out) {
  if (!name || !out) return stp::fail(STP_EINVAL, "stp_builtin_model: null argument");
  const std::string n(name);
  if (n == "ant") build_ant(out);
  else if (n == "humanoid") build_humanoid(out);
  else return stp::fail(STP_EINVAL, "stp_builtin_model: unknown model '" + n + "'");
  return STP_OK;
}

int stp_validate_model(const stp_model* m) {
  // Scene::validate rules (scene.cpp:36-68) plus the GPU layout rules.
  if (!m) return stp::fail(STP_EINVAL, "model: null");
  const int n = m->n_bodies;
  if (n < 1 || n > STP_MAX_BODIES) return stp::fail(STP_EINVAL, "model: n_bodies must be in [1, 32]");
  if (m->n_joints < 0 || m->n_joints > STP_MAX_JOINTS)
    return stp::fail(STP_EINVAL, "model: n_joints must be in [0, 31]");
  if (m->root < 0 || m->root >= n) return stp::fail(STP_EINVAL, "model: root out of range");
  if (m->n_feet < 0 || m->n_feet > STP_MAX_FEET) return stp::fail(STP_EINVAL, "model: n_feet");
  for (int f = 0; f < m->n_feet; ++f)
    if (m->feet[f] < 0 || m->feet[f] >= n) return stp::fail(STP_EINVAL, "model: foot out of range");
  for (int b = 0; b < n; ++b) {
    const stp_body& d = m->bodies[b];
    if (d.shape < STP_SPHERE || d.shape > STP_BOX) return stp::fail(STP_EINVAL, "model: bad shape type");
    if (!d.is_static && (d.mass <= 0 || d.inertia_diag[0] <= 0 || d.inertia_diag[1] <= 0 ||
                         d.inertia_diag[2] <= 0))
      return stp::fail(STP_EINVAL, "scene: dynamic body with nonpositive mass or inertia");
    for (int k = 0; k < STP_STATE_STRIDE; ++k)
      if (!std::isfinite(m->rest_state[b][k])) return stp::fail(STP_EINVAL, "model: non-finite rest state");
  }
  int parent_joints[STP_MAX_BODIES] = {0};
  for (int j = 0; j < m->n_joints; ++j) {
    const stp_joint& d = m->joints[j];
    if (d.parent < 0 || d.parent >= n || d.child < 0 || d.child >= n || d.parent == d.child)
      return stp::fail(STP_EINVAL, "scene: joint body index out of range");
    if (d.limit_lo >= d.limit_hi) return stp::fail(STP_EINVAL, "scene: joint limits out of order");
    if (std::abs(norm3(d.axis_parent) - 1.0) > 1e-9 || std::abs(norm3(d.axis_child) - 1.0) > 1e-9)
      return stp::fail(STP_EINVAL, "scene: joint axis must be unit length");
    if (d.max_torque <= 0) return stp::fail(STP_EINVAL, "scene: joint max_torque must be positive");
    if (!finite3(d.anchor_parent) || !finite3(d.anchor_child))
      return stp::fail(STP_EINVAL, "model: non-finite joint anchor");
    if (d.child <= d.parent)
      return stp::fail(STP_EINVAL, "model: joints must be topologically ordered (child > parent)");
    if (++parent_joints[d.child] > 1)
      return stp::fail(STP_EINVAL, "model: each body may be the child of at most one joint (tree)");
  }
  return STP_OK;
}

int stp_default_task(int32_t kind, stp_task* t) {
  if (!t) return stp::fail(STP_EINVAL, "stp_default_task: null");
  if (kind < STP_TASK_ANT || kind > STP_TASK_HFH_TERRAIN)
    return stp::fail(STP_EINVAL, "stp_default_task: unknown task kind");
  std::memset(t, 0, sizeof(*t));
  t->kind = kind;
  t->episode_cap = 1000;           // PAPER.md:212 "maximum episode length ... 1000 frames"
  t->perturb_min = 200;            // PAPER.md:219 "every 200 to 300 frames"
  t->perturb_max = 300;
  t->perturb_force_lo = 1.0;       // "a few Newtons" -> SPEC.md:329 default 1-5 N
  t->perturb_force_hi = 5.0;
  t->reset_noise = 0.05;
  t->auto_reset = 1;
  t->target_radius = 100.0;
  t->target_tolerance = 1.0;
  if (kind == STP_TASK_HFH || kind == STP_TASK_HFH_TERRAIN) {
    t->fall_grace = 160;           // PAPER.md:210 "(160 frames)"
    t->target_refresh = 200;
    t->spacing = 2.0;
    t->height_map = kind == STP_TASK_HFH_TERRAIN;
    t->inter_agent_collisions = kind == STP_TASK_HFH || kind == STP_TASK_HFH_TERRAIN;
  } else {
    t->fall_grace = 0;
    t->target_refresh = 0;         // fixed target 1000 m ahead
    t->spacing = 3.0;
  }
  return STP_OK;
}

int stp_generate_terrain(const stp_terrain_spec* spec, stp_static_box* out, int32_t capacity) {
  if (!spec) return stp::fail(STP_EINVAL, "generate_terrain: null spec");
  if (spec->count < 0 || spec->dim_lo <= 0 || spec->dim_hi < spec->dim_lo || spec->x_hi < spec->x_lo ||
      spec->y_hi < spec->y_lo || spec->yaw_hi < spec->yaw_lo)
    return stp::fail(STP_EINVAL, "generate_terrain: degenerate ranges");
  if (spec->count > capacity || (spec->count > 0 && !out))
    return stp::fail(STP_EINVAL, "generate_terrain: output capacity too small");
  for (int i = 0; i < spec->count; ++i) {
    const uint64_t s = stp_derive_seed(spec->seed, STP_TAG_TERRAIN, (uint64_t)i);
    stp_static_box& b = out[i];
    for (int k = 0; k < 3; ++k)
      b.half_extents[k] = 0.5 * (spec->dim_lo + (spec->dim_hi - spec->dim_lo) * stp_uniform(s, k));
    b.center[0] = spec->x_lo + (spec->x_hi - spec->x_lo) * stp_uniform(s, 3);
    b.center[1] = spec->y_lo + (spec->y_hi - spec->y_lo) * stp_uniform(s, 4);
    b.center[2] = b.half_extents[2];  // resting on the plane z = 0
    b.yaw = spec->yaw_lo + (spec->yaw_hi - spec->yaw_lo) * stp_uniform(s, 5);
  }
  return spec->count;
}

double stp_terrain_height(const stp_static_box* boxes, int32_t n, double x, double y) {
  // terrain_height, collide.cpp:348-359
  double h = 0.0;
  for (int i = 0; i < n; ++i) {
    const stp_static_box& b = boxes[i];
    const double c = std::cos(b.yaw), s = std::sin(b.yaw);
    const double dx = x - b.center[0], dy = y - b.center[1];
    const double lx = c * dx + s * dy;
    const double ly = -s * dx + c * dy;
    if (std::abs(lx) <= b.half_extents[0] && std::abs(ly) <= b.half_extents[1]) {
      const double top = b.center[2] + b.half_extents[2];
      if (top > h) h = top;
    }
  }
  return h;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Articulation text format "stampede-model 1":
// line-oriented stanzas, '#' comments, numbers in %.17g so serialize -> load
// is the identity on stp_model.
//
//   stampede-model 1
//   name <text>            alive_bonus <x>        fall_height <x>
//   body <name>            (fields, then 'end'):
//     shape sphere|capsule|box   static 0|1   radius r   half_length h
//     half_extents x y z   local_pos x y z   local_rot w x y z
//     mass m   inertia ix iy iz   rest x y z qw qx qy qz vx vy vz wx wy wz
//   end
//   joint <name>           (fields, then 'end'):
//     parent <body>   child <body>   anchor_parent x y z   anchor_child x y z
//     axis_parent x y z   axis_child x y z   rest_relative w x y z   limit lo hi
//   end
//   actuator <joint> <tau_max>
//   foot <body>
//   root <body>
// ---------------------------------------------------------------------------
namespace {

int parse_fail(int line, const std::string& what) {
  return stp::fail(STP_EINVAL, "load_model: " + (line > 0 ? "line " + std::to_string(line) + ": " : std::string()) + what);
}

bool read_n(std::istringstream& ls, double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!(ls >> v[i])) return false;
  std::string extra;
  return !(ls >> extra);
}

}  // namespace

extern "C" int stp_model_from_text(const char* text, stp_model* out) {
  if (!text || !out) return stp::fail(STP_EINVAL, "load_model: null argument");
  stp_model m;
  std::memset(&m, 0, sizeof(m));
  std::map<std::string, int> body_id, joint_id;
  std::vector<bool> has_tau;
  bool header = false, has_root = false;
  std::string root_name;
  std::vector<std::pair<std::string, std::string>> joint_ends;  // parent, child names per joint
  std::vector<int> joint_line;
  enum { NONE, BODY, JOINT } open = NONE;
  std::istringstream in(text);
  std::string raw;
  int line = 0;
  while (std::getline(in, raw)) {
    ++line;
    const size_t hash = raw.find('#');
    if (hash != std::string::npos) raw.resize(hash);
    std::istringstream ls(raw);
    std::string key;
    if (!(ls >> key)) continue;
    if (!header) {
      int version = 0;
      if (key != "stampede-model" || !(ls >> version)) return parse_fail(line, "expected 'stampede-model 1' header");
      if (version != 1) return parse_fail(line, "unsupported model format version " + std::to_string(version));
      header = true;
      continue;
    }
    auto nums = [&](double* v, int n) {
      return read_n(ls, v, n) ? STP_OK : parse_fail(line, "expected " + std::to_string(n) + " number(s) after '" + key + "'");
    };
    int rc = STP_OK;
    if (open == BODY) {
      stp_body& b = m.bodies[m.n_bodies - 1];
      if (key == "end") open = NONE;
      else if (key == "shape") {
        std::string t;
        ls >> t;
        if (t == "sphere") b.shape = STP_SPHERE;
        else if (t == "capsule") b.shape = STP_CAPSULE;
        else if (t == "box") b.shape = STP_BOX;
        else return parse_fail(line, "unknown shape '" + t + "'");
      } else if (key == "static") {
        double v;
        rc = nums(&v, 1);
        b.is_static = v != 0;
      } else if (key == "radius") rc = nums(&b.radius, 1);
      else if (key == "half_length") rc = nums(&b.half_length, 1);
      else if (key == "half_extents") rc = nums(b.half_extents, 3);
      else if (key == "local_pos") rc = nums(b.local_pos, 3);
      else if (key == "local_rot") rc = nums(b.local_rot, 4);
      else if (key == "mass") rc = nums(&b.mass, 1);
      else if (key == "inertia") rc = nums(b.inertia_diag, 3);
      else if (key == "rest") rc = nums(m.rest_state[m.n_bodies - 1], STP_STATE_STRIDE);
      else return parse_fail(line, "unknown body field '" + key + "'");
    } else if (open == JOINT) {
      stp_joint& j = m.joints[m.n_joints - 1];
      if (key == "end") open = NONE;
      else if (key == "parent") ls >> joint_ends.back().first;
      else if (key == "child") ls >> joint_ends.back().second;
      else if (key == "anchor_parent") rc = nums(j.anchor_parent, 3);
      else if (key == "anchor_child") rc = nums(j.anchor_child, 3);
      else if (key == "axis_parent") rc = nums(j.axis_parent, 3);
      else if (key == "axis_child") rc = nums(j.axis_child, 3);
      else if (key == "rest_relative") rc = nums(j.rest_relative, 4);
      else if (key == "limit") {
        double v[2];
        rc = nums(v, 2);
        j.limit_lo = v[0];
        j.limit_hi = v[1];
      } else return parse_fail(line, "unknown joint field '" + key + "'");
    } else if (key == "name") {
      std::string nm;
      std::getline(ls >> std::ws, nm);
      std::strncpy(m.name, nm.c_str(), sizeof(m.name) - 1);
    } else if (key == "alive_bonus") rc = nums(&m.alive_bonus, 1);
    else if (key == "fall_height") rc = nums(&m.fall_height, 1);
    else if (key == "body") {
      std::string nm;
      if (!(ls >> nm)) return parse_fail(line, "body without a name");
      if (body_id.count(nm)) return parse_fail(line, "duplicate body '" + nm + "'");
      if (m.n_bodies >= STP_MAX_BODIES) return parse_fail(line, "more than 32 bodies");
      body_id[nm] = m.n_bodies;
      stp_body& b = m.bodies[m.n_bodies++];
      b.local_rot[0] = 1.0;
      m.rest_state[m.n_bodies - 1][3] = 1.0;
      open = BODY;
    } else if (key == "joint") {
      std::string nm;
      if (!(ls >> nm)) return parse_fail(line, "joint without a name");
      if (joint_id.count(nm)) return parse_fail(line, "duplicate joint '" + nm + "'");
      if (m.n_joints >= STP_MAX_JOINTS) return parse_fail(line, "more than 31 joints");
      joint_id[nm] = m.n_joints;
      stp_joint& j = m.joints[m.n_joints++];
      j.rest_relative[0] = 1.0;
      joint_ends.emplace_back();
      joint_line.push_back(line);
      has_tau.push_back(false);
      open = JOINT;
    } else if (key == "actuator") {
      std::string jn;
      double tau;
      if (!(ls >> jn >> tau)) return parse_fail(line, "expected 'actuator <joint> <tau_max>'");
      auto it = joint_id.find(jn);
      if (it == joint_id.end()) return parse_fail(line, "actuator of unknown joint '" + jn + "'");
      m.joints[it->second].max_torque = tau;
      has_tau[it->second] = true;
    } else if (key == "foot") {
      std::string bn;
      ls >> bn;
      auto it = body_id.find(bn);
      if (it == body_id.end()) return parse_fail(line, "foot of unknown body '" + bn + "'");
      if (m.n_feet >= STP_MAX_FEET) return parse_fail(line, "more than 4 feet");
      m.feet[m.n_feet++] = it->second;
    } else if (key == "root") {
      if (!(ls >> root_name)) return parse_fail(line, "root without a body name");
      has_root = true;
    } else {
      return parse_fail(line, "unknown keyword '" + key + "'");
    }
    if (rc != STP_OK) return rc;
  }
  if (!header) return parse_fail(0, "empty document (expected 'stampede-model 1')");
  if (open != NONE) return parse_fail(line, "unterminated stanza (missing 'end')");
  if (!has_root) return parse_fail(0, "missing field 'root'");
  auto rb = body_id.find(root_name);
  if (rb == body_id.end()) return parse_fail(0, "root names unknown body '" + root_name + "'");
  m.root = rb->second;
  for (int j = 0; j < m.n_joints; ++j) {
    auto pa = body_id.find(joint_ends[j].first), ch = body_id.find(joint_ends[j].second);
    if (pa == body_id.end() || ch == body_id.end())
      return parse_fail(joint_line[j], "joint needs known 'parent' and 'child' bodies");
    m.joints[j].parent = pa->second;
    m.joints[j].child = ch->second;
    if (!has_tau[j]) return parse_fail(joint_line[j], "joint without an 'actuator' (tau_max)");
  }
  // the joint graph must be a tree: each body has at most one parent and
  // following parents from any body ends at a body without one (no cycle)
  std::vector<int> parent(m.n_bodies, -1);
  for (int j = 0; j < m.n_joints; ++j) {
    const int c = m.joints[j].child;
    if (parent[c] >= 0) return parse_fail(joint_line[j], "body has two parent joints");
    parent[c] = m.joints[j].parent;
  }
  for (int b = 0; b < m.n_bodies; ++b) {
    int x = b;
    for (int steps = 0; x >= 0; ++steps) {
      if (steps > m.n_bodies) return parse_fail(0, "cyclic joint graph");
      x = parent[x];
    }
  }
  for (int b = 0; b < m.n_bodies; ++b)
    if (!m.bodies[b].is_static && !(m.bodies[b].mass > 0))
      return parse_fail(0, "body " + std::to_string(b) + ": nonpositive mass");
  const int rc = stp_validate_model(&m);
  if (rc != STP_OK) return rc;
  *out = m;
  return STP_OK;
}

extern "C" int stp_model_to_text(const stp_model* m, char* buf, int32_t capacity, int32_t* length) {
  if (!m) return stp::fail(STP_EINVAL, "serialize_model: null model");
  std::string o;
  char t[256];
  auto num = [&](double v) {
    std::snprintf(t, sizeof t, " %.17g", v);
    o += t;
  };
  auto vec = [&](const char* k, const double* v, int n) {
    o += "  ";
    o += k;
    for (int i = 0; i < n; ++i) num(v[i]);
    o += "\n";
  };
  o += "stampede-model 1\n";
  o += "name " + std::string(m->name, strnlen(m->name, sizeof(m->name))) + "\n";
  o += "alive_bonus";
  num(m->alive_bonus);
  o += "\nfall_height";
  num(m->fall_height);
  o += "\n";
  static const char* shapes[] = {"sphere", "capsule", "box"};
  for (int b = 0; b < m->n_bodies; ++b) {
    const stp_body& d = m->bodies[b];
    o += "body b" + std::to_string(b) + "\n";
    o += std::string("  shape ") + shapes[d.shape] + "\n";
    o += "  static " + std::to_string(d.is_static) + "\n";
    vec("radius", &d.radius, 1);
    vec("half_length", &d.half_length, 1);
    vec("half_extents", d.half_extents, 3);
    vec("local_pos", d.local_pos, 3);
    vec("local_rot", d.local_rot, 4);
    vec("mass", &d.mass, 1);
    vec("inertia", d.inertia_diag, 3);
    vec("rest", m->rest_state[b], STP_STATE_STRIDE);
    o += "end\n";
  }
  for (int j = 0; j < m->n_joints; ++j) {
    const stp_joint& d = m->joints[j];
    o += "joint j" + std::to_string(j) + "\n";
    o += "  parent b" + std::to_string(d.parent) + "\n";
    o += "  child b" + std::to_string(d.child) + "\n";
    vec("anchor_parent", d.anchor_parent, 3);
    vec("anchor_child", d.anchor_child, 3);
    vec("axis_parent", d.axis_parent, 3);
    vec("axis_child", d.axis_child, 3);
    vec("rest_relative", d.rest_relative, 4);
    const double lim[2] = {d.limit_lo, d.limit_hi};
    vec("limit", lim, 2);
    o += "end\n";
  }
  for (int j = 0; j < m->n_joints; ++j) {
    o += "actuator j" + std::to_string(j);
    num(m->joints[j].max_torque);
    o += "\n";
  }
  for (int f = 0; f < m->n_feet; ++f) o += "foot b" + std::to_string(m->feet[f]) + "\n";
  o += "root b" + std::to_string(m->root) + "\n";
  if (length) *length = int32_t(o.size());
  if (buf && capacity > 0) {
    const size_t n = std::min<size_t>(o.size(), size_t(capacity) - 1);
    std::memcpy(buf, o.data(), n);
    buf[n] = '\0';
  }
  return STP_OK;
}
