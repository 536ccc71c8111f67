// Host-visible launch entry of the fused step kernel (sim_step.cu).
#pragma once
#include <cuda_runtime.h>

#include "sim_kernels.cuh"

namespace stp {
// Global scratch rows per lane of every env (sim_step.cuh: G_QH, G_HD, G_LC,
// then 8 overflow contact slots of 11 rows for the terrain instantiation).
constexpr int kSpillSlots = 8;
constexpr int kScratchRows = 55 + 11 * kSpillSlots;
// lanes = W (8/16/32 lanes per env), cpb = contact slots per body.
template <class T>
cudaError_t launch_env_step(const KArgs<T>& a, int lanes, int cpb, cudaStream_t s);
}  // namespace stp
