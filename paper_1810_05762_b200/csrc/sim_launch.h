// Host-visible launch entry of the fused step kernel (sim_step.cu).
#pragma once
#include <cuda_runtime.h>

#include "sim_kernels.cuh"

namespace stp {
// Global scratch rows per lane of every env (sim_step.cuh: G_QH, G_HD, G_LC,
// then 12 overflow contact slots of 11 rows for the terrain instantiation,
// whose 4 first slots per body live in shared memory, then the island mode's
// cross-contact slots).
constexpr int kSpillSlots = 12;
// island mode: per cross-contact slot 19 geometry / weight rows, the 36-entry
// transformed coupling block and the partner's global index (sim_step.cuh G_XS)
constexpr int kXSlotRows = 19 + 36 + 1;
constexpr int kScratchRows = 55 + 11 * kSpillSlots + kXSlotRows * kXSlots;
// lanes = W (8/16/32 lanes per env), cpb = shared-memory contact slots per body
// (2: plane only; 4 + kSpillSlots overflow rows: terrain boxes, dynamic boxes).
template <class T>
cudaError_t launch_env_step(const KArgs<T>& a, int lanes, int cpb, cudaStream_t s);

struct PairScratch;
// Device view of the step's inter-agent coupling (prepare_islands).
struct IslandView {
  const uint8_t* merged;
  const int* isl_members;
  const int* isl_count;
  int* err;  // bit 1: more than kXSlots cross contacts on a body, 2: island larger than kIslandMax
  const XSlot* xslots;
  const int* xcount;
};
template <class T>
cudaError_t prepare_islands(PairScratch*& scratch, const DevModel<T>* model, int B, const T* state,
                            const double* origin, int n, int W, double margin, IslandView* view, cudaStream_t st);

// Inter-agent contact detection (sim_pairs.cu): the reference's dynamic-pair
// contacts of every env of a sim, global body indices, reference order.
void pair_scratch_free(PairScratch* p);
template <class T>
cudaError_t detect_pairs(PairScratch*& scratch, const DevModel<T>* model, int B, const T* state, const double* origin,
                         int n, int W, double margin, int cap_out, int* count, int32_t* body_a, int32_t* body_b,
                         double* point, double* normal, double* separation, bool* overflow, cudaStream_t st);
}  // namespace stp
