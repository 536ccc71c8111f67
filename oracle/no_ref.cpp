// ORACLE — TEST INFRASTRUCTURE ONLY.  liboracle.so carries only the
// restated physics; the compiled reference backend lives in oracle/_ref.
#include "env_oracle.hpp"

namespace orc {
std::unique_ptr<PhysicsBackend> make_reference_backend() { return nullptr; }
}  // namespace orc
