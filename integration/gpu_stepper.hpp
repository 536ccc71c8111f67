// GpuStepper — the reference-side glue a `stampede` maintainer would add to
// route physics::step (proj/include/stampede/physics/solver.hpp:52-53) through
// the B200 C-ABI (include/stampede_sim.h, libstampede_b200.so).  Header-only;
// compiled and exercised side by side with the reference's own physics::step
// by integration/test_gpu_stepper.cpp.
//
// Scope: scenes whose agents (Scene::agents, scene.hpp:24-28) share one
// articulation layout — every agent has the same bodies (shapes, inertials)
// and the same joints relative to its first body, its joints listed as one
// contiguous block per agent in agent order.  That is every scene the SPEC env
// layer builds (N copies of the Ant / Humanoid model); other
// scenes are rejected with std::invalid_argument, like Scene::validate.
#pragma once

#include <algorithm>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "stampede/physics/solver.hpp"
#include "stampede_sim.h"

namespace stampede::physics {

namespace gpu_detail {

inline void check(int rc) {
  if (rc != STP_OK) throw std::runtime_error(std::string("libstampede_b200: ") + stp_last_error());
}

inline void put3(double* d, const Vec3& v) {
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
}
inline void put4(double* d, const Quat& q) {
  d[0] = q.w;
  d[1] = q.x;
  d[2] = q.y;
  d[3] = q.z;
}

// Agent `a`'s articulation as the C-ABI model (types.hpp:40-71 -> stp_body /
// stp_joint); body and joint indices relative to the agent's first body.
inline void agent_model(const Scene& scene, int a, int joints_per_agent, stp_model* m) {
  const AgentRange& ag = scene.agents[a];
  std::memset(m, 0, sizeof(*m));
  std::strncpy(m->name, "scene-agent", sizeof(m->name) - 1);
  m->n_bodies = ag.end - ag.begin;
  m->n_joints = joints_per_agent;
  if (m->n_bodies < 1 || m->n_bodies > STP_MAX_BODIES || m->n_joints > STP_MAX_JOINTS)
    throw std::invalid_argument("GpuStepper: agent size outside the device layout (<= 32 bodies)");
  m->root = -1;  // the agent's first dynamic body
  for (int k = 0; k < m->n_bodies && m->root < 0; ++k)
    if (!scene.inertials[ag.begin + k].is_static) m->root = k;
  if (m->root < 0) throw std::invalid_argument("GpuStepper: agent without a dynamic body");
  for (int k = 0; k < m->n_bodies; ++k) {
    const Shape& s = scene.shapes[ag.begin + k];
    const BodyInertial& in = scene.inertials[ag.begin + k];
    stp_body& b = m->bodies[k];
    b.shape = s.type == ShapeType::Sphere ? STP_SPHERE : s.type == ShapeType::Capsule ? STP_CAPSULE : STP_BOX;
    b.is_static = in.is_static ? 1 : 0;
    b.radius = s.radius;
    b.half_length = s.half_length;
    put3(b.half_extents, s.half_extents);
    put3(b.local_pos, s.local_pos);
    put4(b.local_rot, s.local_rot);
    b.mass = in.mass;
    put3(b.inertia_diag, in.inertia_diag);
    const RigidBodyState& st = scene.states[ag.begin + k];  // rest pose = the current one
    put3(m->rest_state[k] + 0, st.position);
    put4(m->rest_state[k] + 3, st.orientation);
  }
  for (int j = 0; j < joints_per_agent; ++j) {
    const JointDesc& d = scene.joints[size_t(a) * joints_per_agent + j];
    stp_joint& o = m->joints[j];
    o.parent = d.parent - ag.begin;
    o.child = d.child - ag.begin;
    if (o.parent < 0 || o.parent >= m->n_bodies || o.child < 0 || o.child >= m->n_bodies)
      throw std::invalid_argument("GpuStepper: joint of another agent in this agent's joint block");
    put3(o.anchor_parent, d.anchor_parent);
    put3(o.anchor_child, d.anchor_child);
    put3(o.axis_parent, d.axis_parent);
    put3(o.axis_child, d.axis_child);
    put4(o.rest_relative, d.rest_relative);
    o.limit_lo = d.limit_lo;
    o.limit_hi = d.limit_hi;
    o.max_torque = d.max_torque;
  }
  m->fall_height = -1e300;  // the env layer is not used through this adapter
}

// structural equality of two agents' models (the rest pose excluded)
inline bool same_layout(stp_model a, stp_model b) {
  std::memset(a.rest_state, 0, sizeof(a.rest_state));
  std::memset(b.rest_state, 0, sizeof(b.rest_state));
  return std::memcmp(&a, &b, sizeof(stp_model)) == 0;
}

}  // namespace gpu_detail

class GpuStepper {
 public:
  // One device handle for the whole scene: agent a = env a (env_offset 0).
  GpuStepper(const Scene& scene, const StepConfig& cfg, int device = 0, int precision = STP_PRECISION_F32) {
    using namespace gpu_detail;
    if (scene.agents.empty()) throw std::invalid_argument("GpuStepper: scene has no agents");
    n_ = static_cast<int>(scene.agents.size());
    if (scene.joints.size() % size_t(n_) != 0)
      throw std::invalid_argument("GpuStepper: agents must share one joint layout");
    joints_ = static_cast<int>(scene.joints.size() / size_t(n_));
    agent_model(scene, 0, joints_, &model_);
    bodies_ = model_.n_bodies;
    for (int a = 0; a < n_; ++a) {
      if (scene.agents[a].begin != a * bodies_ || scene.agents[a].end != (a + 1) * bodies_)
        throw std::invalid_argument("GpuStepper: agents must be contiguous, equal-size body ranges");
      stp_model m{};
      agent_model(scene, a, joints_, &m);
      if (!same_layout(m, model_)) throw std::invalid_argument("GpuStepper: agents must share one articulation");
    }
    stp_step_config c;
    stp_default_step_config(&c);  // reference_alias_quirk = 1: the reference's assemble, bit for bit in f64
    c.dt = cfg.dt;
    c.newton_iters = cfg.newton_iters;
    c.krylov_tol = cfg.krylov_tol;
    c.krylov_max_iters = cfg.krylov_max_iters;
    c.contact_margin = cfg.contact_margin;
    c.baumgarte = cfg.baumgarte;
    c.joint_hardness = cfg.joint_hardness;
    c.contact_hardness = cfg.contact_hardness;
    c.limit_hardness = cfg.limit_hardness;
    c.friction_smoothing = cfg.friction_smoothing;
    c.limit_activation = cfg.limit_activation;
    put3(c.gravity, scene.gravity);
    c.has_ground_plane = scene.has_ground_plane ? 1 : 0;
    stp_task t;
    stp_default_task(STP_TASK_HUMANOID, &t);
    t.reset_noise = 0;
    t.auto_reset = 0;
    t.perturb_min = t.perturb_max = 0;
    t.inter_agent_collisions = scene.inter_agent_collisions ? 1 : 0;
    h_ = stp_create(&model_, &t, &c, n_, device, /*seed=*/0, precision, /*env_offset=*/0);
    if (!h_) throw std::invalid_argument(std::string("GpuStepper: ") + stp_last_error());
    std::vector<stp_static_box> boxes;  // Scene::static_boxes (types.hpp:86-90)
    for (const StaticBox& b : scene.static_boxes) {
      stp_static_box o{};
      put3(o.center, b.center);
      put3(o.half_extents, b.half_extents);
      o.yaw = b.yaw;
      boxes.push_back(o);
    }
    if (!boxes.empty()) check(stp_set_terrain(h_, boxes.data(), static_cast<int32_t>(boxes.size())));
    cap_ = stp_contact_capacity(h_);
  }
  ~GpuStepper() { stp_destroy(h_); }
  GpuStepper(const GpuStepper&) = delete;
  GpuStepper& operator=(const GpuStepper&) = delete;

  // Drop-in for physics::step(scene, torques, cfg): same inputs, the same
  // in-place Scene update, the same StepReport (contacts in detect_contacts
  // order, totals of Newton / Krylov iterations, failed agents).
  StepReport step(Scene& scene, std::span<const double> torques) {
    using namespace gpu_detail;
    if (torques.size() != scene.joints.size())  // clamp_torques, solver.cpp:397-398
      throw std::invalid_argument("clamp_torques: torque count must equal joint count");
    if (scene.body_count() != n_ * bodies_) throw std::invalid_argument("GpuStepper: scene changed shape");
    static_assert(sizeof(RigidBodyState) == STP_STATE_STRIDE * sizeof(double), "RigidBodyState layout");
    check(stp_set_state(h_, reinterpret_cast<const double*>(scene.states.data())));
    if (!scene.external_force.empty() || !scene.external_torque.empty()) {
      std::vector<double> loads(size_t(n_) * bodies_ * 6, 0.0);
      for (size_t b = 0; b < scene.external_force.size() && b < size_t(n_) * bodies_; ++b)
        put3(&loads[6 * b], scene.external_force[b]);
      for (size_t b = 0; b < scene.external_torque.size() && b < size_t(n_) * bodies_; ++b)
        put3(&loads[6 * b + 3], scene.external_torque[b]);
      check(stp_set_external_loads(h_, loads.data()));
    }
    check(stp_physics_step_host(h_, torques.data()));
    check(stp_get_state(h_, reinterpret_cast<double*>(scene.states.data())));
    scene.clear_external_loads();  // scene.cpp:75-78
    return report();
  }

 private:
  StepReport report() {
    using namespace gpu_detail;
    const size_t N = size_t(n_), C = size_t(cap_);
    std::vector<int32_t> count(N), ba(N * C), bb(N * C), newton(N), krylov(N);
    std::vector<double> pt(N * C * 3), nr(N * C * 3), sep(N * C), pn(N * C), ptan(N * C * 3);
    std::vector<uint8_t> failed(N), overflow(N);
    check(stp_get_contacts(h_, count.data(), ba.data(), bb.data(), pt.data(), nr.data(), sep.data(), pn.data(),
                           ptan.data()));
    check(stp_get_report(h_, newton.data(), krylov.data(), failed.data(), overflow.data()));
    StepReport rep;
    std::vector<std::tuple<int, int, SolvedContact>> inter;  // (a, b) order after the static ones
    for (size_t e = 0; e < N; ++e) {
      if (overflow[e]) throw std::runtime_error("GpuStepper: device contact capacity exceeded");
      for (int k = 0; k < count[e] && size_t(k) < C; ++k) {
        const size_t i = e * C + k;
        SolvedContact sc;
        sc.geom.body_a = int(e) * bodies_ + ba[i];
        sc.geom.body_b = bb[i] < 0 ? kStaticBody : bb[i];  // inter-agent: the partner's global index
        sc.geom.point = {pt[3 * i], pt[3 * i + 1], pt[3 * i + 2]};
        sc.geom.normal = {nr[3 * i], nr[3 * i + 1], nr[3 * i + 2]};
        sc.geom.separation = sep[i];
        sc.normal_impulse = pn[i];
        sc.tangential_impulse = {ptan[3 * i], ptan[3 * i + 1], ptan[3 * i + 2]};
        if (sc.geom.body_b == kStaticBody) rep.contacts.push_back(sc);
        else inter.emplace_back(sc.geom.body_a, sc.geom.body_b, sc);
      }
      // the reference sums its islands' iteration counts (solver.cpp:581-582);
      // an island is one env here (a contact-merged island reports its
      // iterations in each of its envs)
      rep.newton_iterations += newton[e];
      rep.krylov_iterations += krylov[e];
      if (failed[e]) rep.failed_agents.push_back(int(e));
    }
    std::stable_sort(inter.begin(), inter.end(), [](const auto& x, const auto& y) {
      return std::tie(std::get<0>(x), std::get<1>(x)) < std::tie(std::get<0>(y), std::get<1>(y));
    });
    for (auto& c : inter) rep.contacts.push_back(std::get<2>(c));
    return rep;
  }

  stp_sim* h_ = nullptr;
  stp_model model_{};
  int n_ = 0, bodies_ = 0, joints_ = 0, cap_ = 0;
};

}  // namespace stampede::physics
