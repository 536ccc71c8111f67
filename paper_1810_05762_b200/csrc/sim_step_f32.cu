#include "sim_step.cuh"

namespace stp {
template cudaError_t launch_env_step<float>(const KArgs<float>&, int, int, cudaStream_t);
}  // namespace stp
