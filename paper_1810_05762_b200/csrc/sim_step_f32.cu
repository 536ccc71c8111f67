#include "sim_step.cuh"

namespace stp {
template cudaError_t launch_env_step<float>(const KArgs<float>&, int, int, cudaStream_t, const IslandStreams*);
template int island_launch_budget<float>(int);
}  // namespace stp
