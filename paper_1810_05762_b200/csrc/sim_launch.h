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

// Inter-agent contact detection (sim_pairs.cu): the reference's dynamic-pair
// contacts of every env of a sim, global body indices, reference order.
struct PairScratch;
void pair_scratch_free(PairScratch* p);
template <class T>
cudaError_t detect_pairs(PairScratch*& scratch, const DevModel<T>* model, int B, const T* state, const double* origin,
                         int n, int W, double margin, int cap_out, int* count, int32_t* body_a, int32_t* body_b,
                         double* point, double* normal, double* separation, bool* overflow, cudaStream_t st);
}  // namespace stp
