// Host-visible launch entry of the fused step kernel (sim_step.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "sim_kernels.cuh"

namespace stp {
// Runs an entry point on its handle's device and restores the caller's
// current device afterwards (handles on several GPUs in one process).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != device && cudaSetDevice(device) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
// per-device one-time kernel attribute setup (cudaFuncSetAttribute is per device)
inline bool first_on_device(bool (&done)[64]) {
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) return true;
  if (done[d]) return false;
  done[d] = true;
  return true;
}

// Programmatic dependent launch along a stream's chain of dependent kernels
// (the inter-agent pre-step kernels, the step kernel, K4): a kernel launched
// with launch_pdl may be scheduled while its predecessor drains; it runs
// pdl_wait() before touching anything the predecessor writes, and
// pdl_trigger() so its own successor can be scheduled early.  Both are no-ops
// for a plain launch.  STP_PDL=0 launches plainly (A/B timing).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("STP_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
#endif

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
// side stream + fork / join events of a handle with inter-agent collisions:
// the island launches run concurrently with the main step launch
struct IslandStreams {
  cudaStream_t side;  // highest stream priority: island CTAs get SMs before the main launch
  cudaEvent_t fork, join;
  // pinned host copy of the previous step's island count (written by an async
  // copy on `side`, read without a sync): sizes the persistent island grid.
  // Only a hint: the grid loops over however many islands there are.
  int* h_count;
};
template <class T>
cudaError_t launch_env_step(const KArgs<T>& a, int lanes, int cpb, cudaStream_t s,
                            const IslandStreams* isl = nullptr);

// CTAs of the island launch that are co-resident on the current device (the
// budget of big-island parts per step, sim_step.cuh big_island_ctas).
template <class T>
int island_launch_budget(int cpb);

struct PairScratch;
// Device view of the step's inter-agent coupling (prepare_islands).
struct IslandView {
  const uint8_t* merged;  // 1: stepped by an island launch, 2: island over budget (stepped alone, flagged)
  const int* isl_members;
  const int* isl_count;
  const int* isl_order;  // two-env islands first, then the rest
  const int* isl_npair;
  int* err;  // bit 1: more than kXSlots cross contacts on a body, 4: contact edges dropped,
             // 8: candidate env pairs dropped (pair capacity)
  const XSlot* xslots;
  const int* xcount;
  // islands larger than `cap` envs (multi-CTA launch)
  const int* big_count;
  const int* big_off;
  const int* big_size;
  const int* big_members;
  int* big_bar;
  void* big_xch;
};
// cap = envs per one-CTA island (island_cap<T>), max_parts = island_launch_budget
template <class T>
cudaError_t prepare_islands(PairScratch*& scratch, const DevModel<T>* model, int B, const T* state,
                            const double* origin, int n, int W, double margin, int cap, int max_parts,
                            IslandView* view, cudaStream_t st);

// Inter-agent contact detection (sim_pairs.cu): the reference's dynamic-pair
// contacts of every env of a sim, global body indices, reference order.
void pair_scratch_free(PairScratch* p);
template <class T>
cudaError_t detect_pairs(PairScratch*& scratch, const DevModel<T>* model, int B, const T* state, const double* origin,
                         int n, int W, double margin, int cap_out, int* count, int32_t* body_a, int32_t* body_b,
                         double* point, double* normal, double* separation, bool* overflow, cudaStream_t st);
}  // namespace stp
