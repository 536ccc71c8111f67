#include "sim_step.cuh"

namespace stp {
template cudaError_t launch_env_step<double>(const KArgs<double>&, int, int, cudaStream_t, const IslandStreams*);
template int island_launch_budget<double>(int);
}  // namespace stp
