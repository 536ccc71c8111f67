// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
//
// Batched env layer restated from SPEC.md:234-359 and PAPER.md App. B/C
// (the reference has no env code), on top of a pluggable
// physics backend:
//   * orc::RestatedPhysics  — oracle/phys_oracle.hpp (double or float)
//   * orc::ReferencePhysics — the compiled reference stampede::physics::step
//                             (oracle/ref_backend.cpp, built into oracle/_ref)
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "stampede_sim.h"

namespace orc {

struct ContactRec {
  int a, b;
  double p[3], n[3], sep, pn, pt[3];
};

struct World;

struct PhysicsBackend {
  virtual ~PhysicsBackend() = default;
  virtual const char* name() const = 0;
  // Steps every env: consumes w.state / w.loads (cleared afterwards),
  // fills w.contacts, w.newton, w.krylov, w.failed.
  virtual void step(World& w, const double* torques) = 0;
};

struct World {
  stp_model model{};
  stp_task task{};
  stp_step_config cfg{};
  int n = 0;
  uint64_t seed = 0;
  int64_t env_offset = 0;
  int nthreads = 1;
  int precision = 1;  // 1 = double, 0 = float (restated backend only)
  std::vector<stp_static_box> boxes;
  std::vector<double> state;  // n * B * 13
  std::vector<double> loads;  // n * B * 6
  std::vector<std::vector<ContactRec>> contacts;
  std::vector<int32_t> newton, krylov;
  std::vector<uint8_t> failed;
  std::vector<double> target;      // n * 2
  std::vector<int32_t> counters;   // n * 8
  std::vector<double> last_tau;    // n * J
  std::vector<uint8_t> feet;       // n * STP_MAX_FEET (last step's flags)
  std::unique_ptr<PhysicsBackend> physics;

  int nb() const { return model.n_bodies; }
  int nj() const { return model.n_joints; }
  double* body(int e, int b) { return state.data() + (size_t(e) * nb() + b) * STP_STATE_STRIDE; }
};

std::unique_ptr<PhysicsBackend> make_restated_backend();
std::unique_ptr<PhysicsBackend> make_reference_backend();  // only in oracle/_ref

// last-error setter for the C API (returns STP_EINVAL)
int set_error(const std::string& message);

}  // namespace orc
