// ORACLE — TEST INFRASTRUCTURE ONLY.  Compiled (by oracle/Makefile) together
// with the UNMODIFIED reference sources under /root/reference/proj/src into
// oracle/_ref/libstampede_ref.so.  It drives the reference's own
// stampede::physics::step (solver.cpp:448-597) exactly as the reference's
// batching architecture intends: all N agents in ONE Scene, islands solved
// on the reference util::ThreadPool (threading.hpp:32-126).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "env_oracle.hpp"
#include "stampede/physics/scene.hpp"
#include "stampede/physics/solver.hpp"
#include "stampede/util/threading.hpp"

namespace orc {
namespace {

namespace ph = stampede::physics;
namespace la = stampede::linalg;

struct ReferencePhysics : PhysicsBackend {
  ph::Scene scene;
  ph::StepConfig cfg;
  std::unique_ptr<stampede::util::ThreadPool> pool;
  int built_n = -1;
  size_t built_boxes = size_t(-1);

  const char* name() const override { return "reference"; }

  void build(const World& w) {
    const stp_model& m = w.model;
    const int B = m.n_bodies;
    scene = ph::Scene{};
    scene.has_ground_plane = w.cfg.has_ground_plane != 0;
    scene.gravity = {w.cfg.gravity[0], w.cfg.gravity[1], w.cfg.gravity[2]};
    scene.inter_agent_collisions = w.task.inter_agent_collisions != 0;  // HFH
    for (int e = 0; e < w.n; ++e) {
      for (int b = 0; b < B; ++b) {
        const stp_body& d = m.bodies[b];
        ph::Shape s;
        s.type = d.shape == STP_SPHERE ? ph::ShapeType::Sphere
                 : d.shape == STP_CAPSULE ? ph::ShapeType::Capsule
                                          : ph::ShapeType::Box;
        s.radius = d.radius;
        s.half_length = d.half_length;
        s.half_extents = {d.half_extents[0], d.half_extents[1], d.half_extents[2]};
        s.local_pos = {d.local_pos[0], d.local_pos[1], d.local_pos[2]};
        s.local_rot = {d.local_rot[0], d.local_rot[1], d.local_rot[2], d.local_rot[3]};
        scene.shapes.push_back(s);
        scene.inertials.push_back(
            ph::BodyInertial{d.mass, {d.inertia_diag[0], d.inertia_diag[1], d.inertia_diag[2]}, d.is_static != 0});
        scene.states.push_back(ph::RigidBodyState{});
      }
      for (int j = 0; j < m.n_joints; ++j) {
        const stp_joint& d = m.joints[j];
        ph::JointDesc jd;
        jd.parent = e * B + d.parent;
        jd.child = e * B + d.child;
        jd.anchor_parent = {d.anchor_parent[0], d.anchor_parent[1], d.anchor_parent[2]};
        jd.anchor_child = {d.anchor_child[0], d.anchor_child[1], d.anchor_child[2]};
        jd.axis_parent = {d.axis_parent[0], d.axis_parent[1], d.axis_parent[2]};
        jd.axis_child = {d.axis_child[0], d.axis_child[1], d.axis_child[2]};
        jd.rest_relative = {d.rest_relative[0], d.rest_relative[1], d.rest_relative[2], d.rest_relative[3]};
        jd.limit_lo = d.limit_lo;
        jd.limit_hi = d.limit_hi;
        jd.max_torque = d.max_torque;
        scene.joints.push_back(jd);
      }
      scene.agents.push_back({e * B, (e + 1) * B});
    }
    for (const auto& b : w.boxes)
      scene.static_boxes.push_back(ph::StaticBox{{b.center[0], b.center[1], b.center[2]},
                                                 {b.half_extents[0], b.half_extents[1], b.half_extents[2]},
                                                 b.yaw});
    scene.validate();
    const stp_step_config& c = w.cfg;
    cfg.dt = c.dt;
    cfg.newton_iters = c.newton_iters;
    cfg.krylov_tol = c.krylov_tol;
    cfg.krylov_max_iters = c.krylov_max_iters;
    cfg.contact_margin = c.contact_margin;
    cfg.baumgarte = c.baumgarte;
    cfg.joint_hardness = c.joint_hardness;
    cfg.contact_hardness = c.contact_hardness;
    cfg.limit_hardness = c.limit_hardness;
    cfg.friction_smoothing = c.friction_smoothing;
    cfg.limit_activation = c.limit_activation;
    if (w.nthreads > 1 && !pool) pool = std::make_unique<stampede::util::ThreadPool>(w.nthreads);
    built_n = w.n;
    built_boxes = w.boxes.size();
  }

  void step(World& w, const double* torques) override {
    if (built_n != w.n || built_boxes != w.boxes.size()) build(w);
    const int B = w.nb();
    const int NB = w.n * B;
    scene.ensure_load_buffers();
    for (int i = 0; i < NB; ++i) {
      const double* s = w.state.data() + size_t(i) * STP_STATE_STRIDE;
      ph::RigidBodyState& rs = scene.states[i];
      rs.position = {s[0], s[1], s[2]};
      rs.orientation = {s[3], s[4], s[5], s[6]};
      rs.linear_velocity = {s[7], s[8], s[9]};
      rs.angular_velocity = {s[10], s[11], s[12]};
      const double* l = w.loads.data() + size_t(i) * 6;
      scene.external_force[i] = {l[0], l[1], l[2]};
      scene.external_torque[i] = {l[3], l[4], l[5]};
    }
    std::vector<double> tq(torques, torques + size_t(w.n) * w.nj());
    const ph::StepReport rep = ph::step(scene, tq, cfg, pool.get());
    for (int i = 0; i < NB; ++i) {
      double* s = w.state.data() + size_t(i) * STP_STATE_STRIDE;
      const ph::RigidBodyState& rs = scene.states[i];
      s[0] = rs.position.x; s[1] = rs.position.y; s[2] = rs.position.z;
      s[3] = rs.orientation.w; s[4] = rs.orientation.x; s[5] = rs.orientation.y; s[6] = rs.orientation.z;
      s[7] = rs.linear_velocity.x; s[8] = rs.linear_velocity.y; s[9] = rs.linear_velocity.z;
      s[10] = rs.angular_velocity.x; s[11] = rs.angular_velocity.y; s[12] = rs.angular_velocity.z;
    }
    for (auto& c : w.contacts) c.clear();
    for (const auto& sc : rep.contacts) {
      const int e = sc.geom.body_a / B;
      ContactRec r{};
      r.a = sc.geom.body_a - e * B;
      // static -1; a body of another agent (inter-agent contact, listed with
      // body_a's env) as its global index env * B + body (always >= B)
      r.b = sc.geom.body_b < 0 ? -1 : (sc.geom.body_b / B == e ? sc.geom.body_b - e * B : sc.geom.body_b);
      r.p[0] = sc.geom.point.x; r.p[1] = sc.geom.point.y; r.p[2] = sc.geom.point.z;
      r.n[0] = sc.geom.normal.x; r.n[1] = sc.geom.normal.y; r.n[2] = sc.geom.normal.z;
      r.sep = sc.geom.separation;
      r.pn = sc.normal_impulse;
      r.pt[0] = sc.tangential_impulse.x; r.pt[1] = sc.tangential_impulse.y; r.pt[2] = sc.tangential_impulse.z;
      w.contacts[e].push_back(r);
    }
    // StepReport only carries scene totals (types.hpp:115-120): per-env
    // iteration counts are unavailable from the reference.
    std::fill(w.newton.begin(), w.newton.end(), -1);
    std::fill(w.krylov.begin(), w.krylov.end(), -1);
    if (!w.newton.empty()) {
      w.newton[0] = rep.newton_iterations;
      w.krylov[0] = rep.krylov_iterations;
    }
    std::fill(w.failed.begin(), w.failed.end(), 0);
    for (int a : rep.failed_agents) w.failed[a] = 1;
    std::fill(w.loads.begin(), w.loads.end(), 0.0);
  }
};

}  // namespace

std::unique_ptr<PhysicsBackend> make_reference_backend() { return std::make_unique<ReferencePhysics>(); }

}  // namespace orc

// Debug/parity hook: the reference's first Newton linearisation
// (assemble_system, solver.cpp:419-446) of env e as a dense matrix.
extern "C" int orc_ref_first_system(void* h, int e, const double* torques, double* H, double* rhs) {
  using namespace stampede;
  auto* w = reinterpret_cast<orc::World*>(h);
  const stp_model& m = w->model;
  const int B = m.n_bodies;
  physics::Scene sc;
  sc.has_ground_plane = w->cfg.has_ground_plane != 0;
  for (int b = 0; b < B; ++b) {
    const stp_body& d = m.bodies[b];
    physics::Shape s;
    s.type = d.shape == STP_SPHERE ? physics::ShapeType::Sphere
             : d.shape == STP_CAPSULE ? physics::ShapeType::Capsule : physics::ShapeType::Box;
    s.radius = d.radius; s.half_length = d.half_length;
    s.half_extents = {d.half_extents[0], d.half_extents[1], d.half_extents[2]};
    sc.shapes.push_back(s);
    sc.inertials.push_back(physics::BodyInertial{d.mass, {d.inertia_diag[0], d.inertia_diag[1], d.inertia_diag[2]}, d.is_static != 0});
    const double* s0 = w->body(e, b);
    sc.states.push_back(physics::RigidBodyState{{s0[0], s0[1], s0[2]}, {s0[3], s0[4], s0[5], s0[6]}, {s0[7], s0[8], s0[9]}, {s0[10], s0[11], s0[12]}});
  }
  for (int j = 0; j < m.n_joints; ++j) {
    const stp_joint& d = m.joints[j];
    physics::JointDesc jd;
    jd.parent = d.parent; jd.child = d.child;
    jd.anchor_parent = {d.anchor_parent[0], d.anchor_parent[1], d.anchor_parent[2]};
    jd.anchor_child = {d.anchor_child[0], d.anchor_child[1], d.anchor_child[2]};
    jd.axis_parent = {d.axis_parent[0], d.axis_parent[1], d.axis_parent[2]};
    jd.axis_child = {d.axis_child[0], d.axis_child[1], d.axis_child[2]};
    jd.rest_relative = {d.rest_relative[0], d.rest_relative[1], d.rest_relative[2], d.rest_relative[3]};
    jd.limit_lo = d.limit_lo; jd.limit_hi = d.limit_hi; jd.max_torque = d.max_torque;
    sc.joints.push_back(jd);
  }
  sc.agents.push_back({0, B});
  physics::StepConfig cfg;
  auto contacts = physics::detect_contacts(sc, cfg.contact_margin);
  std::vector<double> tq(torques, torques + m.n_joints);
  auto sys = physics::assemble_system(sc, contacts, tq, cfg);
  auto dense = sys.matrix.to_dense();
  std::copy(dense.begin(), dense.end(), H);
  std::copy(sys.rhs.begin(), sys.rhs.end(), rhs);
  return int(contacts.size());
}

// Parity hook for inter-agent contacts: the reference's detect_contacts
// (collide.cpp:270-346) with Scene::inter_agent_collisions = true on the
// world's current state.  Global body indices (env * B + body), the
// reference's list order; returns the total count (entries beyond capacity
// are not written).
extern "C" int orc_ref_detect(void* h, int capacity, int32_t* body_a, int32_t* body_b, double* point,
                              double* normal, double* separation) {
  auto* w = reinterpret_cast<orc::World*>(h);
  orc::ReferencePhysics rp;
  rp.build(*w);
  rp.scene.inter_agent_collisions = true;
  const int NB = w->n * w->nb();
  for (int i = 0; i < NB; ++i) {
    const double* s = w->state.data() + size_t(i) * STP_STATE_STRIDE;
    stampede::physics::RigidBodyState& rs = rp.scene.states[i];
    rs.position = {s[0], s[1], s[2]};
    rs.orientation = {s[3], s[4], s[5], s[6]};
    rs.linear_velocity = {s[7], s[8], s[9]};
    rs.angular_velocity = {s[10], s[11], s[12]};
  }
  const auto cs = stampede::physics::detect_contacts(rp.scene, w->cfg.contact_margin);
  const int n = int(cs.size());
  for (int i = 0; i < n && i < capacity; ++i) {
    body_a[i] = cs[i].body_a;
    body_b[i] = cs[i].body_b;
    point[3 * i] = cs[i].point.x; point[3 * i + 1] = cs[i].point.y; point[3 * i + 2] = cs[i].point.z;
    normal[3 * i] = cs[i].normal.x; normal[3 * i + 1] = cs[i].normal.y; normal[3 * i + 2] = cs[i].normal.z;
    separation[i] = cs[i].separation;
  }
  return n;
}

// Snapshot hooks (Scene::save_snapshot / load_snapshot, scene.cpp:80-104) on a
// reference scene built from the world: the checker of the GPU's SSNP bytes.
extern "C" int64_t orc_ref_save_snapshot(void* h, uint8_t* buf, int64_t cap) {
  auto* w = reinterpret_cast<orc::World*>(h);
  orc::ReferencePhysics rp;
  rp.build(*w);
  const int NB = w->n * w->nb();
  for (int i = 0; i < NB; ++i) {
    const double* s = w->state.data() + size_t(i) * STP_STATE_STRIDE;
    auto& rs = rp.scene.states[i];
    rs.position = {s[0], s[1], s[2]};
    rs.orientation = {s[3], s[4], s[5], s[6]};
    rs.linear_velocity = {s[7], s[8], s[9]};
    rs.angular_velocity = {s[10], s[11], s[12]};
  }
  std::stringstream ss;
  rp.scene.save_snapshot(ss);
  const std::string b = ss.str();
  if (int64_t(b.size()) <= cap) std::memcpy(buf, b.data(), b.size());
  return int64_t(b.size());
}

extern "C" int orc_ref_load_snapshot(void* h, const uint8_t* buf, int64_t size) {
  auto* w = reinterpret_cast<orc::World*>(h);
  orc::ReferencePhysics rp;
  rp.build(*w);
  std::stringstream ss(std::string(reinterpret_cast<const char*>(buf), size_t(size)));
  try {
    rp.scene.load_snapshot(ss);
  } catch (const std::exception& ex) {
    return orc::set_error(std::string(ex.what()));
  }
  const int NB = w->n * w->nb();
  for (int i = 0; i < NB; ++i) {
    double* s = w->state.data() + size_t(i) * STP_STATE_STRIDE;
    const auto& rs = rp.scene.states[i];
    s[0] = rs.position.x; s[1] = rs.position.y; s[2] = rs.position.z;
    s[3] = rs.orientation.w; s[4] = rs.orientation.x; s[5] = rs.orientation.y; s[6] = rs.orientation.z;
    s[7] = rs.linear_velocity.x; s[8] = rs.linear_velocity.y; s[9] = rs.linear_velocity.z;
    s[10] = rs.angular_velocity.x; s[11] = rs.angular_velocity.y; s[12] = rs.angular_velocity.z;
  }
  return 0;
}
