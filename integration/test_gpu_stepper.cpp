// Side-by-side check of the INTEGRATION.md adapter (integration/gpu_stepper.hpp):
// one reference Scene of N Humanoid agents stepped by the unmodified
// reference physics::step (solver.hpp:52-53, compiled from /root/reference
// into oracle/_ref/libstampede_ref.so) and by GpuStepper::step
// (libstampede_b200.so), teacher-forced: both start every step from the same
// Scene.  Compares states, the ordered contact lists (SolvedContact,
// types.hpp:109-113), iteration totals and failed_agents (types.hpp:115-120).
//
//   usage: test_gpu_stepper [f64|f32] [agents] [steps]    (exit status 0 = pass)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "gpu_stepper.hpp"

using namespace stampede;
using namespace stampede::physics;

static Scene humanoid_scene(int n, int precision) {
  stp_model m{};
  if (stp_builtin_model("humanoid", &m) != STP_OK) throw std::runtime_error(stp_last_error());
  // initial poses: the C-ABI reset (grid placement + noise)
  stp_task t;
  stp_default_task(STP_TASK_HUMANOID, &t);
  stp_step_config c;
  stp_default_step_config(&c);
  stp_sim* h = stp_create(&m, &t, &c, n, 0, 7, precision, 0);
  if (!h) throw std::runtime_error(stp_last_error());
  std::vector<double> st(size_t(n) * m.n_bodies * 13);
  gpu_detail::check(stp_get_state(h, st.data()));
  stp_destroy(h);
  Scene s;
  for (int a = 0; a < n; ++a) {
    const int b0 = a * m.n_bodies;
    for (int b = 0; b < m.n_bodies; ++b) {
      const stp_body& d = m.bodies[b];
      Shape sh;
      sh.type = d.shape == STP_SPHERE ? ShapeType::Sphere : d.shape == STP_CAPSULE ? ShapeType::Capsule : ShapeType::Box;
      sh.radius = d.radius;
      sh.half_length = d.half_length;
      sh.half_extents = {d.half_extents[0], d.half_extents[1], d.half_extents[2]};
      sh.local_pos = {d.local_pos[0], d.local_pos[1], d.local_pos[2]};
      sh.local_rot = {d.local_rot[0], d.local_rot[1], d.local_rot[2], d.local_rot[3]};
      s.shapes.push_back(sh);
      s.inertials.push_back({d.mass, {d.inertia_diag[0], d.inertia_diag[1], d.inertia_diag[2]}, d.is_static != 0});
      const double* x = &st[(size_t(b0) + b) * 13];
      s.states.push_back({{x[0], x[1], x[2]}, {x[3], x[4], x[5], x[6]}, {x[7], x[8], x[9]}, {x[10], x[11], x[12]}});
    }
    for (int j = 0; j < m.n_joints; ++j) {
      const stp_joint& d = m.joints[j];
      JointDesc jd;
      jd.parent = b0 + d.parent;
      jd.child = b0 + d.child;
      jd.anchor_parent = {d.anchor_parent[0], d.anchor_parent[1], d.anchor_parent[2]};
      jd.anchor_child = {d.anchor_child[0], d.anchor_child[1], d.anchor_child[2]};
      jd.axis_parent = {d.axis_parent[0], d.axis_parent[1], d.axis_parent[2]};
      jd.axis_child = {d.axis_child[0], d.axis_child[1], d.axis_child[2]};
      jd.rest_relative = {d.rest_relative[0], d.rest_relative[1], d.rest_relative[2], d.rest_relative[3]};
      jd.limit_lo = d.limit_lo;
      jd.limit_hi = d.limit_hi;
      jd.max_torque = d.max_torque;
      s.joints.push_back(jd);
    }
    s.agents.push_back({b0, b0 + m.n_bodies});
  }
  return s;
}

int main(int argc, char** argv) {
  const std::string prec = argc > 1 ? argv[1] : "f64";
  const int n = argc > 2 ? std::atoi(argv[2]) : 16;
  const int steps = argc > 3 ? std::atoi(argv[3]) : 40;
  const int precision = prec == "f32" ? STP_PRECISION_F32 : STP_PRECISION_F64;
  const double tol_x = precision == STP_PRECISION_F64 ? 1e-7 : 5e-3;
  Scene ref = humanoid_scene(n, precision);
  StepConfig cfg;  // types.hpp:92-107 defaults
  GpuStepper gpu(ref, cfg, 0, precision);
  std::mt19937_64 eng(2026);
  std::uniform_real_distribution<double> u(-1, 1);
  double worst = 0;
  int contacts = 0, mism = 0, boundary = 0, iter_mism = 0;
  for (int t = 0; t < steps; ++t) {
    std::vector<double> tq(ref.joints.size());
    for (size_t j = 0; j < tq.size(); ++j) tq[j] = u(eng) * ref.joints[j].max_torque * 1.3;  // some beyond tau_max
    if (t == 7) {  // a perturbation load on agent 1's root (Scene::external_force, scene.hpp:45-46)
      ref.ensure_load_buffers();
      ref.external_force[ref.agents[1 % n].begin] = {40.0, -25.0, 0.0};
    }
    Scene g = ref;  // teacher-forced: the same Scene into both steppers
    const StepReport rr = step(ref, tq, cfg);
    const StepReport rg = gpu.step(g, tq);
    for (size_t b = 0; b < ref.states.size(); ++b) {
      const Vec3 d = ref.states[b].position - g.states[b].position;
      worst = std::max(worst, std::max({std::abs(d.x), std::abs(d.y), std::abs(d.z)}));
    }
    contacts += int(rr.contacts.size());
    if (rr.failed_agents != rg.failed_agents) ++mism;
    if (precision == STP_PRECISION_F64 &&
        (rr.newton_iterations != rg.newton_iterations || rr.krylov_iterations != rg.krylov_iterations))
      ++iter_mism;
    bool same = rr.contacts.size() == rg.contacts.size();
    if (!same) std::printf("  step %d: contact count %zu vs %zu\n", t, rr.contacts.size(), rg.contacts.size());
    for (size_t k = 0; same && k < rr.contacts.size(); ++k) {
      const ContactPoint &a = rr.contacts[k].geom, &b = rg.contacts[k].geom;
      const double pa = rr.contacts[k].normal_impulse, pb = rg.contacts[k].normal_impulse;
      same = a.body_a == b.body_a && a.body_b == b.body_b &&
             std::abs(a.separation - b.separation) <= (precision == STP_PRECISION_F64 ? 1e-9 : 1e-4) &&
             std::abs(pa - pb) <= (precision == STP_PRECISION_F64 ? 1e-5 : 5e-2) * std::max(1.0, std::abs(pa));
      if (!same)
        std::printf("  step %d contact %zu: bodies (%d,%d) vs (%d,%d), sep %.12g vs %.12g, pn %.9g vs %.9g\n", t, k,
                    a.body_a, a.body_b, b.body_a, b.body_b, a.separation, b.separation, pa, pb);
    }
    if (!same) {
      // fp32: a contact within 1e-5 m of the speculative margin may flip (reported, not hidden)
      bool near = false;
      for (const auto& c : rr.contacts) near = near || std::abs(c.geom.separation - cfg.contact_margin) < 1e-5;
      if (precision == STP_PRECISION_F32 && near) ++boundary;
      else ++mism;
    }
  }
  std::printf("GpuStepper vs physics::step (%s, %d Humanoid agents, %d teacher-forced steps): max |dx| %.3e m "
              "(tol %.0e); %d reference contacts; contact-list / failed-agent mismatches %d (boundary %d); "
              "iteration-total mismatches %d\n",
              prec.c_str(), n, steps, worst, tol_x, contacts, mism, boundary, iter_mism);
  // wrong torque count: the reference's invalid_argument (solver.cpp:397-398)
  bool threw = false;
  try {
    std::vector<double> bad(ref.joints.size() - 1);
    Scene g = ref;
    gpu.step(g, bad);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  const bool ok = worst <= tol_x && mism == 0 && iter_mism == 0 && contacts > 0 && threw;
  std::printf("%s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}
