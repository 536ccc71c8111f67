// Host-visible launch entry of the fused step kernel (sim_step.cu).
#pragma once
#include <cuda_runtime.h>

#include "sim_kernels.cuh"

namespace stp {
// Global scratch rows per lane of every env (sim_step.cuh: G_QH, G_HD, G_LC,
// then 12 overflow contact slots of 11 rows for the terrain instantiation,
// whose 4 first slots per body live in shared memory).
constexpr int kSpillSlots = 12;
constexpr int kScratchRows = 55 + 11 * kSpillSlots;
// lanes = W (8/16/32 lanes per env), cpb = shared-memory contact slots per body
// (2: plane only; 4 + kSpillSlots overflow rows: terrain boxes, dynamic boxes).
template <class T>
cudaError_t launch_env_step(const KArgs<T>& a, int lanes, int cpb, cudaStream_t s);
}  // namespace stp
