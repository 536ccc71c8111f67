// Host side of the C-ABI (include/stampede_sim.h): handle lifecycle,
// device buffers, model upload, state import/export and kernel launches.
//
// This replaces the reference's in-process entry points
//   stampede::physics::step            (solver.hpp:52-53)  -> stp_physics_step
//   Scene state access / snapshot      (scene.hpp:31-63)   -> stp_set_state/get_state
//   StepReport                         (types.hpp:115-120) -> stp_get_report/get_contacts
// and the SPEC-only env API -> stp_reset / stp_step.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "sim_launch.h"
#include "stampede_sim.h"
#include "stp_error.h"

struct stp_sim {
  int device = 0;
  cudaStream_t stream = nullptr;
  // Launches may run on any stream (a caller's: torch's current stream, the
  // legacy default stream; NULL: the handle's own non-blocking stream) and the
  // accessors run on the handle's stream.  A handle is one sequential object
  // (the reference's Scene): every launch is recorded in ev_last and the next
  // launch or accessor on another stream waits on it (order_after_last), so
  // work on one handle executes in call order whatever streams are mixed.
  cudaEvent_t ev_caller = nullptr;  // ev_last
  cudaStream_t last_stream = nullptr;
  bool caller_pending = false;      // ev_last holds an unfinished launch
  int precision = STP_PRECISION_F32;
  int W = 32, cpb = 2, cap = 64;
  stp_model model{};
  stp_task task{};
  stp_step_config cfg{};
  int n = 0, B = 0, J = 0, obs_dim = 0;
  uint64_t seed = 0;
  int64_t env_offset = 0;
  size_t tsize = 4;  // sizeof(T)
  void* d_model = nullptr;
  void* d_state = nullptr;
  double* d_origin = nullptr;
  void* d_loads = nullptr;
  bool loads_pending = false;
  int32_t* d_counters = nullptr;
  void* d_target = nullptr;
  void* d_last_tau = nullptr;
  uint32_t* d_feet = nullptr;
  int32_t* d_newton = nullptr;
  int32_t* d_krylov = nullptr;
  uint8_t* d_failed = nullptr;
  uint8_t* d_overflow = nullptr;
  int32_t* d_ccount = nullptr;
  int32_t* d_cbody = nullptr;
  double* d_cdata = nullptr;
  bool record = false;  // record contacts on the next physics step(s)
  double* d_boxes = nullptr;
  int n_boxes = 0;
  void* d_scratch = nullptr;
  void* d_dbg = nullptr;  // assemble_system hook capture (stp_debug_first_system)
  stp::IslandStreams isl{};  // inter-agent handles: island launches beside the main launch
  int dbg_env = -1;
  // terrain broadphase grid
  int grid_nx = 0, grid_ny = 0;
  double grid_x0 = 0, grid_y0 = 0, grid_inv = 0;
  int* d_cell_start = nullptr;
  int* d_cell_list = nullptr;
  int4* d_box_cells = nullptr;
  // staging for the host-buffer entry points
  float* d_act = nullptr;
  float* d_obs = nullptr;
  float* d_rew = nullptr;
  uint8_t* d_done = nullptr;
  // host-buffer pipelining: env chunks on their own streams so one chunk's
  // copies overlap the other chunks' kernels (created on first use)
#ifndef STP_HOST_CHUNKS
#define STP_HOST_CHUNKS 4
#endif
  static constexpr int kChunks = STP_HOST_CHUNKS;
  cudaStream_t cs[kChunks] = {};
  cudaEvent_t ev_in = nullptr, ev_out[kChunks] = {};
  // stp_step_host, inter-agent handles: the actions' upload runs on cs[0]
  // beside the pre-step chain (which reads only the state); the step launch
  // waits for it (act_wait, consumed by launch())
  cudaEvent_t ev_act = nullptr, act_wait = nullptr;
  stp::PairScratch* pairs = nullptr;  // inter-agent detection scratch (created on first use)
  std::vector<void*> allocations;
};

namespace {

using stp::fail;

int cuda_fail(cudaError_t e, const char* what) {
  return fail(STP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                   \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

template <class P>
int dalloc(stp_sim* s, P** p, size_t bytes) {
  void* raw = nullptr;
  cudaError_t e = cudaMalloc(&raw, std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  CK(cudaMemsetAsync(raw, 0, std::max<size_t>(bytes, 16), s->stream));
  s->allocations.push_back(raw);
  *p = reinterpret_cast<P*>(raw);
  return STP_OK;
}

// Island rule of the GPU path: an env's dynamic bodies must form ONE
// joint-connected component (solver.cpp:458-502 then yields one island per
// env) unless the env is a single free body.
bool single_island(const stp_model& m) {
  int par[STP_MAX_BODIES];
  for (int b = 0; b < m.n_bodies; ++b) par[b] = b;
  auto find = [&](int x) {
    while (par[x] != x) x = par[x] = par[par[x]];
    return x;
  };
  for (int j = 0; j < m.n_joints; ++j) {
    const stp_joint& d = m.joints[j];
    if (!m.bodies[d.parent].is_static && !m.bodies[d.child].is_static) par[find(d.parent)] = find(d.child);
  }
  int root = -1;
  for (int b = 0; b < m.n_bodies; ++b) {
    if (m.bodies[b].is_static) continue;
    const int r = find(b);
    if (root < 0) root = r;
    else if (r != root) return false;
  }
  return true;
}

// Child -> parent summation schedule for the PCR matvec.  Every round each
// lane pulls one value (one shuffle); a parent needs the sum of its
// children's contributions, so a parent with m children needs m rounds unless
// siblings are pre-added: with R rounds, children are paired (head, tail), the
// head adds the tail's value into its own contribution in round 0 and the
// parent reads the head in a later round.  R is the smallest count that fits
// (2 for the Humanoid: torso and pelvis; 3 for the Ant's 4-legged torso).
template <class T>
void gather_schedule(const stp_model& m, stp::DevModel<T>& d) {
  const int n = m.n_bodies;
  std::vector<std::vector<int>> kids(n);
  for (int j = 0; j < m.n_joints; ++j) kids[m.joints[j].parent].push_back(m.joints[j].child);
  for (int R = 1; R <= 4; ++R) {
    int slot_src[4][32], slot_kind[4][32];  // kind 0 none, 1 Y, 2 T
    for (int r = 0; r < 4; ++r)
      for (int b = 0; b < 32; ++b) {
        slot_src[r][b] = b;
        slot_kind[r][b] = 0;
      }
    bool ok = true;
    std::vector<std::vector<int>> sources(n);  // what each parent reads (Y)
    std::vector<int> min_round(32, 0);
    for (int p = 0; p < n && ok; ++p) {
      const auto& k = kids[p];
      if (int(k.size()) <= R) {
        sources[p] = k;
        continue;
      }
      for (size_t i = 0; i < k.size(); i += 2) {
        sources[p].push_back(k[i]);
        if (i + 1 < k.size()) {
          if (slot_kind[0][k[i]] != 0) ok = false;
          slot_src[0][k[i]] = k[i + 1];
          slot_kind[0][k[i]] = 2;
          min_round[k[i]] = 1;
        }
      }
      if (int(sources[p].size()) > R) ok = false;
    }
    for (int p = 0; p < n && ok; ++p) {
      for (int s : sources[p]) {
        int r = min_round[s];
        while (r < R && slot_kind[r][p] != 0) ++r;
        if (r >= R) {
          ok = false;
          break;
        }
        slot_src[r][p] = s;
        slot_kind[r][p] = 1;
      }
    }
    if (!ok) continue;
    d.gather_rounds = R;
    for (int r = 0; r < 4; ++r) {
      d.gather_has_t[r] = 0;
      for (int b = 0; b < 32; ++b) {
        d.gather_src[r][b] = slot_src[r][b];
        d.gather_wy[r][b] = T(slot_kind[r][b] == 1 ? 1 : 0);
        d.gather_wt[r][b] = T(slot_kind[r][b] == 2 ? 1 : 0);
        if (slot_kind[r][b] == 2) d.gather_has_t[r] = 1;
      }
    }
    return;
  }
}

template <class T>
void build_dev_model(const stp_model& m, const stp_step_config& cfg, stp::DevModel<T>& d) {
  std::memset(&d, 0, sizeof(d));
  d.nb = m.n_bodies;
  d.nj = m.n_joints;
  d.root = m.root;
  d.n_feet = m.n_feet;
  for (int f = 0; f < m.n_feet; ++f) {
    d.feet[f] = m.feet[f];
    d.feet_mask |= 1 << m.feet[f];
  }
  d.fall_height = T(m.fall_height);
  d.alive_bonus = T(m.alive_bonus);
  for (int b = 0; b < 32; ++b) {
    d.parent[b] = -1;
    d.joint[b] = -1;
    d.lrot[0][b] = T(1);
  }
  for (int b = 0; b < m.n_bodies; ++b) {
    const stp_body& s = m.bodies[b];
    d.shape[b] = s.shape;
    d.is_static[b] = s.is_static;
    d.radius[b] = T(s.radius);
    d.half_len[b] = T(s.half_length);
    for (int k = 0; k < 3; ++k) {
      d.hext[k][b] = T(s.half_extents[k]);
      d.lpos[k][b] = T(s.local_pos[k]);
      d.inertia[k][b] = T(s.inertia_diag[k]);
      d.inv_inertia[k][b] = s.is_static ? T(0) : T(1.0 / s.inertia_diag[k]);
    }
    for (int k = 0; k < 4; ++k) d.lrot[k][b] = T(s.local_rot[k]);
    d.mass[b] = T(s.mass);
    d.inv_mass[b] = s.is_static ? T(0) : T(1.0 / s.mass);
    for (int k = 0; k < 13; ++k) d.rest_state[k][b] = T(m.rest_state[b][k]);
  }
  int n_dyn = 0;
  for (int b = 0; b < m.n_bodies; ++b) n_dyn += m.bodies[b].is_static ? 0 : 1;
  int pair_index = 0;
  for (int j = 0; j < m.n_joints; ++j) {
    const stp_joint& s = m.joints[j];
    const int c = s.child;
    d.parent[c] = s.parent;
    d.joint[c] = j;
    d.lane_of_joint[j] = c;
    d.child_mask[s.parent] |= 1 << c;
    for (int k = 0; k < 3; ++k) {
      d.anc_p[k][c] = T(s.anchor_parent[k]);
      d.anc_c[k][c] = T(s.anchor_child[k]);
      d.ax_p[k][c] = T(s.axis_parent[k]);
      d.ax_c[k][c] = T(s.axis_child[k]);
    }
    for (int k = 0; k < 4; ++k) d.rest[k][c] = T(s.rest_relative[k]);
    d.lim_lo[c] = T(s.limit_lo);
    d.lim_hi[c] = T(s.limit_hi);
    d.tmax[c] = T(s.max_torque);
    // Reference aliasing quirk (solver.cpp:350-351, block_sparse.cpp:33-37):
    // with n_dyn diagonal blocks created first and two blocks per coupled
    // pair in row order, creating (child, parent) reallocates the block pool
    // exactly when the count before it is a power of two.
    if (!m.bodies[s.parent].is_static && !m.bodies[c].is_static) {
      const int nblk = n_dyn + 2 * pair_index + 1;  // blocks once (parent, child) exists
      if (cfg.reference_alias_quirk && (nblk & (nblk - 1)) == 0) d.quirk[c] = 1;
      ++pair_index;
    }
  }
  for (int k = 0; k < 4; ++k)
    for (int b = 0; b < 32; ++b) d.child_list[k][b] = -1;
  d.max_children = 0;
  for (int b = 0; b < m.n_bodies; ++b) {
    int n = 0;
    for (int c = 0; c < m.n_bodies; ++c)
      if ((d.child_mask[b] >> c) & 1) d.child_list[n++ < 4 ? n - 1 : 3][b] = c;
    d.max_children = std::max(d.max_children, n);
  }
  gather_schedule(m, d);
  int maxd = 0;
  for (int b = 0; b < m.n_bodies; ++b) {  // topological order: parent < child
    d.depth[b] = d.parent[b] < 0 ? 0 : d.depth[d.parent[b]] + 1;
    maxd = std::max(maxd, d.depth[b]);
  }
  d.max_depth = maxd;
}

template <class T>
stp::DevCfg<T> dev_cfg(const stp_step_config& c) {
  stp::DevCfg<T> d;
  d.dt = T(c.dt);
  d.tol = T(c.krylov_tol);
  d.margin = T(c.contact_margin);
  d.beta = T(c.baumgarte);
  d.kj = T(c.joint_hardness);
  d.kc = T(c.contact_hardness);
  d.kl = T(c.limit_hardness);
  d.epsf = T(c.friction_smoothing);
  d.lim_act = T(c.limit_activation);
  d.gx = T(c.gravity[0]);
  d.gy = T(c.gravity[1]);
  d.gz = T(c.gravity[2]);
  d.newton = c.newton_iters;
  d.kmax = c.krylov_max_iters;
  d.plane = c.has_ground_plane;
  return d;
}

stp::DevTask dev_task(const stp_task& t) {
  stp::DevTask d;
  d.kind = t.kind;
  d.episode_cap = t.episode_cap;
  d.fall_grace = t.fall_grace;
  d.target_refresh = t.target_refresh;
  d.target_radius = t.target_radius;
  d.target_tolerance = t.target_tolerance;
  d.spacing = t.spacing;
  d.perturb_min = t.perturb_min;
  d.perturb_max = t.perturb_max;
  d.force_lo = t.perturb_force_lo;
  d.force_hi = t.perturb_force_hi;
  d.reset_noise = t.reset_noise;
  d.auto_reset = t.auto_reset;
  d.height_map = t.height_map;
  return d;
}

template <class T>
stp::KArgs<T> make_args(stp_sim* s, int mode) {
  stp::KArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.model = reinterpret_cast<const stp::DevModel<T>*>(s->d_model);
  a.cfg = dev_cfg<T>(s->cfg);
  a.task = dev_task(s->task);
  a.n = s->n;
  a.mode = mode;
  a.seed = s->seed;
  a.env_offset = s->env_offset;
  a.state = reinterpret_cast<T*>(s->d_state);
  a.origin = s->d_origin;
  a.loads = s->loads_pending ? reinterpret_cast<T*>(s->d_loads) : nullptr;
  a.obs_dim = s->obs_dim;
  a.counters = s->d_counters;
  a.target = reinterpret_cast<T*>(s->d_target);
  a.last_tau = reinterpret_cast<T*>(s->d_last_tau);
  a.feet = s->d_feet;
  a.newton_out = s->d_newton;
  a.krylov_out = s->d_krylov;
  a.failed_out = s->d_failed;
  a.overflow_out = s->d_overflow;
  a.record = s->record ? 1 : 0;
  a.cap = s->cap;
  a.c_count = s->d_ccount;
  a.c_body = s->d_cbody;
  a.c_data = s->d_cdata;
  a.n_boxes = s->n_boxes;
  a.boxes = s->d_boxes;
  a.scratch = reinterpret_cast<T*>(s->d_scratch);
  a.dbg = s->dbg_env >= 0 ? reinterpret_cast<T*>(s->d_dbg) : nullptr;
  a.dbg_env = s->dbg_env;
  a.grid_nx = s->grid_nx;
  a.grid_ny = s->grid_ny;
  a.grid_x0 = s->grid_x0;
  a.grid_y0 = s->grid_y0;
  a.grid_inv = s->grid_inv;
  a.cell_start = s->d_cell_start;
  a.cell_list = s->d_cell_list;
  a.box_cells = s->d_box_cells;
  return a;
}

template <class T>
int launch_t(stp_sim* s, int mode, const float* torques, const float* actions, float* obs, float* reward,
             uint8_t* done, const uint8_t* mask, cudaStream_t st, int e_begin, int e_end) {
  auto a = make_args<T>(s, mode);
  a.e_begin = e_begin;
  if (e_end >= 0) a.n = e_end;
  a.torques = torques;
  a.actions = actions;
  a.obs = obs;
  a.reward = reward;
  a.done = done;
  a.reset_mask = mask;
  if (mode != 2 && s->task.inter_agent_collisions && s->n > 1) {
    // Scene::inter_agent_collisions (HFH): contacts between
    // agents of the pre-step state (collide.cpp:300-343) merge envs into
    // islands solved together (solver.cpp:458-502); all on the device
    stp::IslandView v{};
    const int cap = sizeof(T) == 4 ? stp::kIslandMax : stp::kIslandMax / 2;  // island_cap<T>
    cudaError_t e = stp::prepare_islands<T>(s->pairs, reinterpret_cast<const stp::DevModel<T>*>(s->d_model), s->B,
                                            reinterpret_cast<const T*>(s->d_state), s->d_origin, s->n, s->W,
                                            s->cfg.contact_margin, cap, stp::island_launch_budget<T>(s->cpb), &v,
                                            st);
    if (e != cudaSuccess) return cuda_fail(e, "inter-agent island preparation");
    a.merged = v.merged;
    a.isl_members = v.isl_members;
    a.isl_count = v.isl_count;
    a.isl_order = v.isl_order;
    a.isl_npair = v.isl_npair;
    a.isl_err = v.err;
    a.xslots = v.xslots;
    a.xcount = v.xcount;
    a.big_count = v.big_count;
    a.big_off = v.big_off;
    a.big_size = v.big_size;
    a.big_members = v.big_members;
    a.big_bar = v.big_bar;
    a.big_xch = reinterpret_cast<T*>(v.big_xch);
  }
  if (s->act_wait) {  // the actions' upload (stp_step_host) overlapped the pre-step chain
    CK(cudaStreamWaitEvent(st, s->act_wait, 0));
    s->act_wait = nullptr;
  }
  if (a.merged && !s->isl.side) {
    // the highest stream priority: island CTAs (long, latency-bound chains of a
    // few warps) get SMs before the main launch fills the machine instead of
    // waiting for its last wave to drain (crowded HFH rollout: 0.380 -> 0.361
    // ms per step; uncrowded steps unchanged)
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&s->isl.side, cudaStreamNonBlocking, hi));
    CK(cudaMallocHost(&s->isl.h_count, sizeof(int)));
    s->isl.h_count[0] = a.n;  // first step: no hint (grid min(n / 2, SMs))
    CK(cudaEventCreateWithFlags(&s->isl.fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->isl.join, cudaEventDisableTiming));
  }
  static const bool side = [] {  // STP_ISL_SIDE=0: island launches in order on the caller's stream (A/B)
    const char* v = getenv("STP_ISL_SIDE");
    return !(v && v[0] == '0');
  }();
  const cudaError_t e = stp::launch_env_step<T>(a, s->W, s->cpb, st, a.merged && side ? &s->isl : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "k_env_step launch");
  return STP_OK;
}

// order stream `st` after the handle's last launch when that was made on
// another stream
int order_after_last(stp_sim* s, cudaStream_t st) {
  if (s->caller_pending && s->last_stream != st) CK(cudaStreamWaitEvent(st, s->ev_caller, 0));
  return STP_OK;
}
// record a launch made on `st` as the handle's last one
int mark_last(stp_sim* s, cudaStream_t st) {
  CK(cudaEventRecord(s->ev_caller, st));
  s->last_stream = st;
  s->caller_pending = true;
  return STP_OK;
}
// the accessors (handle's stream, synchronous): after every earlier launch
int join_caller(stp_sim* s) { return order_after_last(s, s->stream); }

bool is_chunk_stream(const stp_sim* s, cudaStream_t st) {
  for (int c = 0; c < stp_sim::kChunks; ++c)
    if (st == s->cs[c]) return true;
  return false;
}

int launch(stp_sim* s, int mode, const float* torques, const float* actions, float* obs, float* reward,
           uint8_t* done, const uint8_t* mask, cudaStream_t st, int e_begin = 0, int e_end = -1) {
  // stp_step_host's chunk streams are ordered by that call itself (ev_in /
  // ev_out), so its chunks overlap one another
  const bool chunk = is_chunk_stream(s, st);
  if (!chunk)
    if (const int rc = order_after_last(s, st)) return rc;
  const int rc = s->precision == STP_PRECISION_F64
                     ? launch_t<double>(s, mode, torques, actions, obs, reward, done, mask, st, e_begin, e_end)
                     : launch_t<float>(s, mode, torques, actions, obs, reward, done, mask, st, e_begin, e_end);
  if (rc) return rc;
  if (mode != 2) s->loads_pending = false;
  if (!chunk) return mark_last(s, st);
  return STP_OK;
}

cudaStream_t pick(stp_sim* s, void* stream) { return stream ? reinterpret_cast<cudaStream_t>(stream) : s->stream; }

int validate_cfg(const stp_step_config& c) {
  if (!(c.dt > 0)) return fail(STP_EINVAL, "step config: dt must be > 0");
  if (c.newton_iters < 1) return fail(STP_EINVAL, "step config: newton_iters must be >= 1");
  if (!(c.krylov_tol > 0) || c.krylov_max_iters < 1)
    return fail(STP_EINVAL, "solve_krylov: tol must be > 0 and max_iters >= 1");
  if (c.contact_margin < 0) return fail(STP_EINVAL, "detect_contacts: margin must be >= 0");
  const double g = std::sqrt(c.gravity[0] * c.gravity[0] + c.gravity[1] * c.gravity[1] + c.gravity[2] * c.gravity[2]);
  if (std::abs(g - 9.8) > 1e-9) return fail(STP_EINVAL, "scene: gravity magnitude must be 9.8");
  return STP_OK;
}

}  // namespace

namespace stp {
int sim_dims(const stp_sim* s, int* n, int* J, uint64_t* seed, long long* off, void** stream) {
  if (!s) return STP_EINVAL;
  *n = s->n;
  *J = s->J;
  *seed = s->seed;
  *off = s->env_offset;
  *stream = reinterpret_cast<void*>(s->stream);
  return STP_OK;
}
int sim_device(const stp_sim* s) { return s ? s->device : 0; }
// call-order sequencing of launches made outside this file (sim_aux.cu)
int sim_order(stp_sim* s, void* st) { return order_after_last(s, reinterpret_cast<cudaStream_t>(st)); }
int sim_mark(stp_sim* s, void* st) { return mark_last(s, reinterpret_cast<cudaStream_t>(st)); }
}  // namespace stp

extern "C" {

stp_sim* stp_create(const stp_model* model, const stp_task* task, const stp_step_config* cfg, int32_t n_envs,
                    int32_t device, uint64_t seed, int32_t precision, int64_t env_offset) {
  if (!model || !task || !cfg) {
    fail(STP_EINVAL, "stp_create: null argument");
    return nullptr;
  }
  if (n_envs <= 0) {
    fail(STP_EINVAL, "reset: N must be > 0");
    return nullptr;
  }
  if (stp_validate_model(model) != STP_OK) return nullptr;
  if (validate_cfg(*cfg) != STP_OK) return nullptr;
  for (int b = 0; b < model->n_bodies; ++b) {
    int kids = 0;
    for (int j = 0; j < model->n_joints; ++j) kids += model->joints[j].parent == b;
    if (kids > 4) {
      fail(STP_EINVAL, "model: the GPU path supports at most 4 child joints per body");
      return nullptr;
    }
  }
  if (!single_island(*model)) {
    fail(STP_EINVAL, "model: the GPU path needs every env's dynamic bodies joint-connected (one island per env)");
    return nullptr;
  }
  if (precision != STP_PRECISION_F32 && precision != STP_PRECISION_F64) {
    fail(STP_EINVAL, "stp_create: precision must be STP_PRECISION_F32 or STP_PRECISION_F64");
    return nullptr;
  }
  auto* s = new stp_sim();
  s->device = device;
  s->precision = precision;
  s->model = *model;
  s->task = *task;
  s->cfg = *cfg;
  s->n = n_envs;
  s->B = model->n_bodies;
  s->J = model->n_joints;
  s->seed = seed;
  s->env_offset = env_offset;
  s->W = s->B <= 8 ? 8 : (s->B <= 16 ? 16 : 32);
  if (precision == STP_PRECISION_F32 && s->W < 32) {
    // Several envs per warp only pay when that is what fits the launch into
    // one wave of resident warps (3 blocks x 4 warps per SM): their lane
    // groups diverge, so a shared warp runs ~1.25x longer than a full-warp
    // env (measured, Ant: 64 envs 0.091 -> 0.056 ms, 1776: 0.097 -> 0.078,
    // 4096: 0.205 -> 0.202 with W = 32; 2048: 0.098 with W = 16, 0.130 with 32).
    int dev_sms = 0;
    if (cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
      cudaGetLastError();
      dev_sms = 148;
    }
    const long long resident = 12LL * dev_sms;
    const long long narrow = (n_envs * (long long)s->W + 31) / 32;
    if (!(n_envs > resident && narrow <= resident)) s->W = 32;
  }
  bool boxes_shape = false;
  for (int b = 0; b < s->B; ++b) boxes_shape = boxes_shape || model->bodies[b].shape == STP_BOX;
  s->cpb = boxes_shape || task->kind == STP_TASK_HFH_TERRAIN ? 4 : 2;
  s->cap = s->B * (s->cpb > 2 ? s->cpb + stp::kSpillSlots : s->cpb);  // slots per body incl. overflow rows
  s->obs_dim = 11 + 3 * s->J + model->n_feet + (task->height_map ? 165 : 0);
  s->tsize = precision == STP_PRECISION_F64 ? 8 : 4;
  auto bail = [&](int) -> stp_sim* {
    stp_destroy(s);
    return nullptr;
  };
  int dev_count = 0;
  cudaError_t e = cudaGetDeviceCount(&dev_count);
  if (e == cudaSuccess && (device < 0 || device >= dev_count)) e = cudaErrorInvalidDevice;
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaSetDevice");
    delete s;
    return nullptr;
  }
  const stp::DeviceGuard dg_(device);  // the caller's current device is restored on return
  e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_caller, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaStreamCreate");
    delete s;
    return nullptr;
  }
  const size_t N = size_t(n_envs);
  const size_t ts = s->tsize;
  int rc = STP_OK;
  if (precision == STP_PRECISION_F64) rc = dalloc(s, &s->d_model, sizeof(stp::DevModel<double>));
  else rc = dalloc(s, &s->d_model, sizeof(stp::DevModel<float>));
  if (rc || (rc = dalloc(s, &s->d_state, N * stp::kStateFields * s->W * ts)) ||
      (rc = dalloc(s, &s->d_origin, N * 2 * sizeof(double))) || (rc = dalloc(s, &s->d_loads, N * 6 * s->W * ts)) ||
      (rc = dalloc(s, &s->d_counters, N * 8 * sizeof(int32_t))) || (rc = dalloc(s, &s->d_target, N * 2 * ts)) ||
      (rc = dalloc(s, &s->d_last_tau, N * std::max(1, s->J) * ts)) || (rc = dalloc(s, &s->d_feet, N * 4)) ||
      (rc = dalloc(s, &s->d_newton, N * 4)) || (rc = dalloc(s, &s->d_krylov, N * 4)) ||
      (rc = dalloc(s, &s->d_failed, N)) || (rc = dalloc(s, &s->d_overflow, N)) ||
      (rc = dalloc(s, &s->d_ccount, N * 4)) || (rc = dalloc(s, &s->d_cbody, N * s->cap * 4)) ||
      (rc = dalloc(s, &s->d_cdata, N * s->cap * stp::kCData * sizeof(double))) ||
      (rc = dalloc(s, &s->d_act, N * std::max(1, s->J) * 4)) || (rc = dalloc(s, &s->d_obs, N * s->obs_dim * 4)) ||
      (rc = dalloc(s, &s->d_rew, N * 4)) || (rc = dalloc(s, &s->d_done, N)) ||
      (rc = dalloc(s, &s->d_scratch, N * size_t(stp::kScratchRows) * s->W * ts)))
    return bail(rc);
  if (precision == STP_PRECISION_F64) {
    stp::DevModel<double> dm;
    build_dev_model(*model, *cfg, dm);
    e = cudaMemcpyAsync(s->d_model, &dm, sizeof(dm), cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  } else {
    stp::DevModel<float> dm;
    build_dev_model(*model, *cfg, dm);
    e = cudaMemcpyAsync(s->d_model, &dm, sizeof(dm), cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  }
  if (e != cudaSuccess) {
    cuda_fail(e, "model upload");
    return bail(STP_ECUDA);
  }
  // initial reset of every env
  if (stp_reset(s, nullptr, nullptr, nullptr) != STP_OK) return bail(STP_ECUDA);
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) {
    cuda_fail(e, "initial reset");
    return bail(STP_ECUDA);
  }
  return s;
}

void stp_destroy(stp_sim* s) {
  if (!s) return;
  const stp::DeviceGuard dg_(s->device);
  if (s->ev_caller) cudaEventSynchronize(s->ev_caller);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (int c = 0; c < stp_sim::kChunks; ++c) {
    if (s->cs[c]) {
      cudaStreamSynchronize(s->cs[c]);
      cudaStreamDestroy(s->cs[c]);
    }
    if (s->ev_out[c]) cudaEventDestroy(s->ev_out[c]);
  }
  if (s->ev_in) cudaEventDestroy(s->ev_in);
  if (s->ev_act) cudaEventDestroy(s->ev_act);
  if (s->isl.side) {
    cudaStreamSynchronize(s->isl.side);
    if (s->isl.h_count) cudaFreeHost(s->isl.h_count);
    cudaStreamDestroy(s->isl.side);
    cudaEventDestroy(s->isl.fork);
    cudaEventDestroy(s->isl.join);
  }
  if (s->ev_caller) cudaEventDestroy(s->ev_caller);
  stp::pair_scratch_free(s->pairs);
  for (void* p : s->allocations) cudaFree(p);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

int stp_set_terrain(stp_sim* s, const stp_static_box* boxes, int32_t n) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || n < 0 || (n > 0 && !boxes)) return fail(STP_EINVAL, "stp_set_terrain: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  std::vector<double> h(size_t(std::max(n, 1)) * 8);
  for (int i = 0; i < n; ++i) {
    const stp_static_box& b = boxes[i];
    double* o = h.data() + 8 * i;
    o[0] = b.center[0];
    o[1] = b.center[1];
    o[2] = b.center[2];
    o[3] = b.half_extents[0];
    o[4] = b.half_extents[1];
    o[5] = b.half_extents[2];
    o[6] = std::cos(b.yaw);  // obb_frame, collide.cpp:131
    o[7] = std::sin(b.yaw);
  }
  CK(cudaStreamSynchronize(s->stream));
  if (s->d_boxes) {
    CK(cudaFree(s->d_boxes));
    s->allocations.erase(std::remove(s->allocations.begin(), s->allocations.end(), (void*)s->d_boxes),
                         s->allocations.end());
    s->d_boxes = nullptr;
  }
  int rc = dalloc(s, &s->d_boxes, h.size() * sizeof(double));
  if (rc) return rc;
  CK(cudaMemcpyAsync(s->d_boxes, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  s->n_boxes = n;
  // Uniform xy grid over the boxes' loose footprints (the reference's box
  // broadphase box, collide.cpp:289-290: centre +- (hx+hy, hx+hy)); each box
  // is listed, in index order, in every cell its footprint overlaps.
  for (void* p : {(void*)s->d_cell_start, (void*)s->d_cell_list, (void*)s->d_box_cells}) {
    if (!p) continue;
    CK(cudaFree(p));
    s->allocations.erase(std::remove(s->allocations.begin(), s->allocations.end(), p), s->allocations.end());
  }
  s->d_cell_start = nullptr;
  s->d_cell_list = nullptr;
  s->d_box_cells = nullptr;
  s->grid_nx = s->grid_ny = 0;
  if (n > 0) {
    const double cell = 2.0;
    double x0 = 1e300, y0 = 1e300, x1 = -1e300, y1 = -1e300;
    for (int i = 0; i < n; ++i) {
      const double ex = boxes[i].half_extents[0] + boxes[i].half_extents[1];
      x0 = std::min(x0, boxes[i].center[0] - ex);
      x1 = std::max(x1, boxes[i].center[0] + ex);
      y0 = std::min(y0, boxes[i].center[1] - ex);
      y1 = std::max(y1, boxes[i].center[1] + ex);
    }
    const int nx = std::max(1, int(std::ceil((x1 - x0) / cell)) + 1);
    const int ny = std::max(1, int(std::ceil((y1 - y0) / cell)) + 1);
    if (double(nx) * ny > 16e6) return fail(STP_EINVAL, "set_terrain: terrain extent too large for the grid");
    const double inv = 1.0 / cell;
    auto cl = [](int c, int m) { return c < 0 ? 0 : (c >= m ? m - 1 : c); };
    std::vector<int4> bc(n);
    std::vector<int> count(size_t(nx) * ny + 1, 0);
    for (int i = 0; i < n; ++i) {
      const double ex = boxes[i].half_extents[0] + boxes[i].half_extents[1];
      bc[i].x = cl(int(std::floor((boxes[i].center[0] - ex - x0) * inv)), nx);
      bc[i].y = cl(int(std::floor((boxes[i].center[1] - ex - y0) * inv)), ny);
      bc[i].z = cl(int(std::floor((boxes[i].center[0] + ex - x0) * inv)), nx);
      bc[i].w = cl(int(std::floor((boxes[i].center[1] + ex - y0) * inv)), ny);
      for (int cy = bc[i].y; cy <= bc[i].w; ++cy)
        for (int cx = bc[i].x; cx <= bc[i].z; ++cx) ++count[size_t(cy) * nx + cx + 1];
    }
    for (size_t c = 1; c < count.size(); ++c) count[c] += count[c - 1];
    std::vector<int> fill(count.begin(), count.end() - 1), list(count.back());
    for (int i = 0; i < n; ++i)
      for (int cy = bc[i].y; cy <= bc[i].w; ++cy)
        for (int cx = bc[i].x; cx <= bc[i].z; ++cx) list[fill[size_t(cy) * nx + cx]++] = i;
    if ((rc = dalloc(s, &s->d_cell_start, count.size() * sizeof(int))) ||
        (rc = dalloc(s, &s->d_cell_list, std::max<size_t>(1, list.size()) * sizeof(int))) ||
        (rc = dalloc(s, &s->d_box_cells, bc.size() * sizeof(int4))))
      return rc;
    CK(cudaMemcpyAsync(s->d_cell_start, count.data(), count.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    if (!list.empty())
      CK(cudaMemcpyAsync(s->d_cell_list, list.data(), list.size() * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->d_box_cells, bc.data(), bc.size() * sizeof(int4), cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    s->grid_nx = nx;
    s->grid_ny = ny;
    s->grid_x0 = x0;
    s->grid_y0 = y0;
    s->grid_inv = inv;
  }
  if (n > 0 && s->cpb < 4) {
    // terrain contacts need more slots per body: grow the recorded list too
    s->cpb = 4;
    s->cap = s->B * (s->cpb > 2 ? s->cpb + stp::kSpillSlots : s->cpb);  // slots per body incl. overflow rows
    const size_t N = size_t(s->n);
    for (void* p : {(void*)s->d_cbody, (void*)s->d_cdata}) {
      CK(cudaFree(p));
      s->allocations.erase(std::remove(s->allocations.begin(), s->allocations.end(), p), s->allocations.end());
    }
    if ((rc = dalloc(s, &s->d_cbody, N * s->cap * 4)) ||
        (rc = dalloc(s, &s->d_cdata, N * s->cap * stp::kCData * sizeof(double))))
      return rc;
  }
  return STP_OK;
}

int32_t stp_num_envs(const stp_sim* s) { return s ? s->n : 0; }
int32_t stp_obs_dim(const stp_sim* s) { return s ? s->obs_dim : 0; }
int32_t stp_action_dim(const stp_sim* s) { return s ? s->J : 0; }
int32_t stp_contact_capacity(const stp_sim* s) { return s ? s->cap : 0; }

namespace {
constexpr uint32_t kSnapshotMagic = 0x504e5353;  // "SSNP", scene.cpp:25-26
constexpr uint32_t kSnapshotVersion = 1;
}  // namespace

int64_t stp_snapshot_size(const stp_sim* s) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  return s ? int64_t(16) + int64_t(s->n) * s->B * STP_STATE_STRIDE * 8 : 0;
}

int stp_save_snapshot(stp_sim* s, uint8_t* buf, int64_t capacity) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || !buf) return fail(STP_EINVAL, "stp_save_snapshot: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  const int64_t need = stp_snapshot_size(s);
  if (capacity < need) return fail(STP_EINVAL, "stp_save_snapshot: buffer too small");
  const uint64_t nb = uint64_t(s->n) * s->B;
  std::memcpy(buf, &kSnapshotMagic, 4);
  std::memcpy(buf + 4, &kSnapshotVersion, 4);
  std::memcpy(buf + 8, &nb, 8);
  return stp_get_state(s, reinterpret_cast<double*>(buf + 16));  // RigidBodyState order (types.hpp:28-32)
}

int stp_load_snapshot(stp_sim* s, const uint8_t* buf, int64_t size) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || !buf || size < 16) return fail(STP_EINVAL, "stp_load_snapshot: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  uint32_t magic, version;
  uint64_t nb;
  std::memcpy(&magic, buf, 4);
  std::memcpy(&version, buf + 4, 4);
  std::memcpy(&nb, buf + 8, 8);
  if (magic != kSnapshotMagic) return fail(STP_EINVAL, "scene snapshot: bad magic");
  if (version != kSnapshotVersion) return fail(STP_EINVAL, "scene snapshot: unsupported version");
  if (nb != uint64_t(s->n) * s->B) return fail(STP_EINVAL, "scene snapshot: body count mismatch");
  if (size < stp_snapshot_size(s)) return fail(STP_EINVAL, "scene snapshot: truncated");
  std::vector<double> st(size_t(nb) * STP_STATE_STRIDE);
  std::memcpy(st.data(), buf + 16, st.size() * 8);  // unaligned-safe
  return stp_set_state(s, st.data());
}

int stp_detect_inter_agent(stp_sim* s, int32_t capacity, int32_t* count, int32_t* body_a, int32_t* body_b,
                           double* point, double* normal, double* separation) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || !count || capacity < 0) return fail(STP_EINVAL, "stp_detect_inter_agent: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  bool overflow = false;
  int n = 0;
  cudaError_t e;
  if (s->precision == STP_PRECISION_F64)
    e = stp::detect_pairs<double>(s->pairs, reinterpret_cast<const stp::DevModel<double>*>(s->d_model), s->B,
                                  reinterpret_cast<const double*>(s->d_state), s->d_origin, s->n, s->W,
                                  s->cfg.contact_margin, capacity, &n, body_a, body_b, point, normal, separation,
                                  &overflow, s->stream);
  else
    e = stp::detect_pairs<float>(s->pairs, reinterpret_cast<const stp::DevModel<float>*>(s->d_model), s->B,
                                 reinterpret_cast<const float*>(s->d_state), s->d_origin, s->n, s->W,
                                 s->cfg.contact_margin, capacity, &n, body_a, body_b, point, normal, separation,
                                 &overflow, s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "stp_detect_inter_agent");
  if (overflow) return fail(STP_EINVAL, "stp_detect_inter_agent: candidate buffer overflow");
  *count = n;
  return STP_OK;
}
void* stp_stream(const stp_sim* s) { return s ? reinterpret_cast<void*>(s->stream) : nullptr; }

int stp_reset(stp_sim* s, const uint8_t* mask, float* obs, void* stream) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_reset: null handle");
  return launch(s, 2, nullptr, nullptr, obs, nullptr, nullptr, mask, pick(s, stream));
}

int stp_step(stp_sim* s, const float* actions, float* obs, float* reward, uint8_t* done, void* stream) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_step: null handle");
  if (s->J > 0 && !actions) return fail(STP_EINVAL, "env_step: actions required");
  return launch(s, 1, nullptr, actions, obs, reward, done, nullptr, pick(s, stream));
}

#ifndef STP_HOST_MIN_CHUNK
#define STP_HOST_MIN_CHUNK 1024
#endif
constexpr size_t kMinChunk = STP_HOST_MIN_CHUNK;

// Device view of a page-locked host buffer (UVA), or null for pageable memory.
static void* pinned_view(void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

int stp_step_host(stp_sim* s, const float* actions, float* obs, float* reward, uint8_t* done) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || (s->J > 0 && !actions)) return fail(STP_EINVAL, "stp_step_host: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n);
  // reward / done (5 bytes per env) go straight from the kernel into
  // page-locked host buffers, saving two small downloads (~5 us of fixed
  // latency each) at the end of the call; pageable buffers are copied.
  float* rew_z = static_cast<float*>(pinned_view(reward));
  uint8_t* done_z = static_cast<uint8_t*>(pinned_view(done));
  float* rew_k = reward ? (rew_z ? rew_z : s->d_rew) : nullptr;
  uint8_t* done_k = done ? (done_z ? done_z : s->d_done) : nullptr;
  // up to 4 chunks of >= 1024 envs (measured on B200 at 4096 envs: 4 chunks
  // 0.234 ms, 8 chunks 0.243 ms, one launch 0.259 ms per call)
  // (envs coupled by inter-agent contacts are stepped as one launch)
  const int C = s->task.inter_agent_collisions
                    ? 1
                    : int(std::min<size_t>(stp_sim::kChunks, std::max<size_t>(1, N / kMinChunk)));
  if (C == 1) {
    if (s->task.inter_agent_collisions && s->J) {
      // upload beside the pre-step chain (detection reads the state only)
      if (!s->ev_in) {
        CK(cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming));
        for (int c = 0; c < stp_sim::kChunks; ++c) {
          CK(cudaStreamCreateWithFlags(&s->cs[c], cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&s->ev_out[c], cudaEventDisableTiming));
        }
      }
      if (!s->ev_act) CK(cudaEventCreateWithFlags(&s->ev_act, cudaEventDisableTiming));
      CK(cudaEventRecord(s->ev_in, s->stream));  // after the work already queued (readers of d_act)
      CK(cudaStreamWaitEvent(s->cs[0], s->ev_in, 0));
      CK(cudaMemcpyAsync(s->d_act, actions, N * s->J * sizeof(float), cudaMemcpyHostToDevice, s->cs[0]));
      CK(cudaEventRecord(s->ev_act, s->cs[0]));
      s->act_wait = s->ev_act;
    } else {
      CK(cudaMemcpyAsync(s->d_act, actions, N * s->J * sizeof(float), cudaMemcpyHostToDevice, s->stream));
    }
    // one launch: nothing overlaps a download at the end, so page-locked obs
    // buffers are written by the kernels directly (the PCIe stores spread over
    // the step) instead of one exposed copy
    float* obs_z = obs ? static_cast<float*>(pinned_view(obs)) : nullptr;
    int rc = launch(s, 1, nullptr, s->d_act, obs ? (obs_z ? obs_z : s->d_obs) : nullptr, rew_k, done_k, nullptr,
                    s->stream);
    s->act_wait = nullptr;
    if (rc) return rc;
    if (obs && !obs_z)
      CK(cudaMemcpyAsync(obs, s->d_obs, N * s->obs_dim * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
    if (reward && !rew_z) CK(cudaMemcpyAsync(reward, s->d_rew, N * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
    if (done && !done_z) CK(cudaMemcpyAsync(done, s->d_done, N, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return STP_OK;
  }
  if (!s->ev_in) {
    CK(cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming));
    for (int c = 0; c < stp_sim::kChunks; ++c) {
      CK(cudaStreamCreateWithFlags(&s->cs[c], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&s->ev_out[c], cudaEventDisableTiming));
    }
  }
  // every chunk starts after the work already queued on the handle's stream
  CK(cudaEventRecord(s->ev_in, s->stream));
  const size_t O = size_t(s->obs_dim), J = size_t(s->J);
  // page-locked obs are written by the chunk kernels directly (the last
  // chunk's download was exposed at the end of the call; measured 4096 envs:
  // e2e 22.6 -> 24.6 M env-steps/s)
  float* obs_z = obs ? static_cast<float*>(pinned_view(obs)) : nullptr;
  const bool loads = s->loads_pending;  // pending external loads apply to every chunk
  for (int c = 0; c < C; ++c) {
    const size_t e0 = N * c / C, e1 = N * (c + 1) / C, n = e1 - e0;
    cudaStream_t st = s->cs[c];
    s->loads_pending = loads;
    CK(cudaStreamWaitEvent(st, s->ev_in, 0));
    if (J) CK(cudaMemcpyAsync(s->d_act + e0 * J, actions + e0 * J, n * J * sizeof(float), cudaMemcpyHostToDevice, st));
    int rc = launch(s, 1, nullptr, s->d_act, obs ? (obs_z ? obs_z : s->d_obs) : nullptr, rew_k, done_k, nullptr, st,
                    int(e0), int(e1));
    if (rc) return rc;
    if (obs && !obs_z)
      CK(cudaMemcpyAsync(obs + e0 * O, s->d_obs + e0 * O, n * O * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (reward && !rew_z)
      CK(cudaMemcpyAsync(reward + e0, s->d_rew + e0, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (done && !done_z) CK(cudaMemcpyAsync(done + e0, s->d_done + e0, n, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s->ev_out[c], st));
  }
  // later work on the handle's stream is ordered after every chunk
  for (int c = 0; c < C; ++c) CK(cudaStreamWaitEvent(s->stream, s->ev_out[c], 0));
  CK(cudaStreamSynchronize(s->stream));
  return mark_last(s, s->stream);
}

int stp_physics_step(stp_sim* s, const float* torques, void* stream) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_physics_step: null handle");
  if (s->J > 0 && !torques) return fail(STP_EINVAL, "clamp_torques: torque count must equal joint count");
  return launch(s, 0, torques, nullptr, nullptr, nullptr, nullptr, nullptr, pick(s, stream));
}

int stp_physics_step_host(stp_sim* s, const double* torques) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_physics_step_host: null handle");
  if (const int rc_ = join_caller(s)) return rc_;
  if (s->J > 0 && !torques) return fail(STP_EINVAL, "clamp_torques: torque count must equal joint count");
  const size_t N = size_t(s->n);
  std::vector<float> t(N * s->J);
  for (size_t i = 0; i < t.size(); ++i) t[i] = float(torques[i]);
  if (!t.empty()) CK(cudaMemcpyAsync(s->d_act, t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  s->record = true;
  int rc = launch(s, 0, s->d_act, nullptr, nullptr, nullptr, nullptr, nullptr, s->stream);
  s->record = false;
  if (rc) return rc;
  CK(cudaStreamSynchronize(s->stream));
  return STP_OK;
}


int stp_set_state(stp_sim* s, const double* state) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || !state) return fail(STP_EINVAL, "stp_set_state: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n);
  const int W = s->W, B = s->B, R = s->model.root;
  std::vector<double> origin(N * 2);
  std::vector<unsigned char> buf(N * stp::kStateFields * W * s->tsize, 0);
  for (size_t e = 0; e < N; ++e) {
    const double* root = state + (e * B + R) * STP_STATE_STRIDE;
    const double ox = std::rint(root[0]), oy = std::rint(root[1]);
    origin[2 * e] = ox;
    origin[2 * e + 1] = oy;
    for (int b = 0; b < B; ++b) {
      const double* st = state + (e * B + b) * STP_STATE_STRIDE;
      for (int f = 0; f < STP_STATE_STRIDE; ++f) {
        double v = st[f];
        if (f == 0) v -= ox;
        if (f == 1) v -= oy;
        const size_t idx = (e * stp::kStateFields + f) * W + b;
        if (s->precision == STP_PRECISION_F64) reinterpret_cast<double*>(buf.data())[idx] = v;
        else reinterpret_cast<float*>(buf.data())[idx] = float(v);
      }
    }
  }
  // targets are stored relative to the origin: shift them with it
  std::vector<double> tgt(N * 2);
  std::vector<double> old(N * 2);
  std::vector<unsigned char> traw(N * 2 * s->tsize);
  CK(cudaMemcpyAsync(old.data(), s->d_origin, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(traw.data(), s->d_target, traw.size(), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  for (size_t i = 0; i < N * 2; ++i) {
    const double t = s->precision == STP_PRECISION_F64 ? reinterpret_cast<double*>(traw.data())[i]
                                                       : double(reinterpret_cast<float*>(traw.data())[i]);
    const double tw = old[i] + t;
    const double tl = tw - origin[i];
    if (s->precision == STP_PRECISION_F64) reinterpret_cast<double*>(traw.data())[i] = tl;
    else reinterpret_cast<float*>(traw.data())[i] = float(tl);
  }
  CK(cudaMemcpyAsync(s->d_state, buf.data(), buf.size(), cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(s->d_origin, origin.data(), origin.size() * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(s->d_target, traw.data(), traw.size(), cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return STP_OK;
}

int stp_get_state(stp_sim* s, double* state) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || !state) return fail(STP_EINVAL, "stp_get_state: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n);
  const int W = s->W, B = s->B;
  std::vector<unsigned char> buf(N * stp::kStateFields * W * s->tsize);
  std::vector<double> origin(N * 2);
  CK(cudaMemcpyAsync(buf.data(), s->d_state, buf.size(), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(origin.data(), s->d_origin, origin.size() * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  for (size_t e = 0; e < N; ++e)
    for (int b = 0; b < B; ++b)
      for (int f = 0; f < STP_STATE_STRIDE; ++f) {
        const size_t idx = (e * stp::kStateFields + f) * W + b;
        double v = s->precision == STP_PRECISION_F64 ? reinterpret_cast<double*>(buf.data())[idx]
                                                     : double(reinterpret_cast<float*>(buf.data())[idx]);
        if (f == 0) v += origin[2 * e];
        if (f == 1) v += origin[2 * e + 1];
        state[(e * B + b) * STP_STATE_STRIDE + f] = v;
      }
  return STP_OK;
}

int stp_set_external_loads(stp_sim* s, const double* loads) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || !loads) return fail(STP_EINVAL, "stp_set_external_loads: bad arguments");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n);
  const int W = s->W, B = s->B;
  std::vector<unsigned char> buf(N * 6 * W * s->tsize, 0);
  for (size_t e = 0; e < N; ++e)
    for (int b = 0; b < B; ++b)
      for (int k = 0; k < 6; ++k) {
        const double v = loads[(e * B + b) * 6 + k];
        const size_t idx = (e * 6 + k) * W + b;
        if (s->precision == STP_PRECISION_F64) reinterpret_cast<double*>(buf.data())[idx] = v;
        else reinterpret_cast<float*>(buf.data())[idx] = float(v);
      }
  CK(cudaMemcpyAsync(s->d_loads, buf.data(), buf.size(), cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  s->loads_pending = true;
  return STP_OK;
}

int stp_get_contacts(stp_sim* s, int32_t* count, int32_t* body_a, int32_t* body_b, double* point, double* normal,
                     double* separation, double* normal_impulse, double* tangential_impulse) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_get_contacts: null handle");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n), C = size_t(s->cap);
  std::vector<int32_t> cnt(N), body(N * C);
  std::vector<double> data(N * C * stp::kCData);
  CK(cudaMemcpyAsync(cnt.data(), s->d_ccount, N * 4, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(body.data(), s->d_cbody, N * C * 4, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(data.data(), s->d_cdata, data.size() * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  for (size_t e = 0; e < N; ++e) {
    if (count) count[e] = cnt[e];
    const int m = std::min<int>(cnt[e], int(C));
    for (int i = 0; i < m; ++i) {
      const size_t k = e * C + i;
      const double* d = data.data() + k * stp::kCData;
      if (body_a) body_a[k] = body[k] & 0xff;
      if (body_b) body_b[k] = (body[k] >> 8) - 1;  // -1 static; inter-agent: partner's global index
      for (int c = 0; c < 3; ++c) {
        if (point) point[3 * k + c] = d[c];
        if (normal) normal[3 * k + c] = d[3 + c];
        if (tangential_impulse) tangential_impulse[3 * k + c] = d[8 + c];
      }
      if (separation) separation[k] = d[6];
      if (normal_impulse) normal_impulse[k] = d[7];
    }
  }
  return STP_OK;
}

int stp_get_report(stp_sim* s, int32_t* newton, int32_t* krylov, uint8_t* failed, uint8_t* overflow) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_get_report: null handle");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n);
  if (newton) CK(cudaMemcpyAsync(newton, s->d_newton, N * 4, cudaMemcpyDeviceToHost, s->stream));
  if (krylov) CK(cudaMemcpyAsync(krylov, s->d_krylov, N * 4, cudaMemcpyDeviceToHost, s->stream));
  if (failed) CK(cudaMemcpyAsync(failed, s->d_failed, N, cudaMemcpyDeviceToHost, s->stream));
  if (overflow) CK(cudaMemcpyAsync(overflow, s->d_overflow, N, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return STP_OK;
}

int stp_get_task_state(stp_sim* s, double* target, int32_t* counters, double* last_tau) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_get_task_state: null handle");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n), J = size_t(s->J);
  std::vector<double> origin(N * 2);
  std::vector<unsigned char> traw(N * 2 * s->tsize), lraw(N * std::max<size_t>(J, 1) * s->tsize);
  CK(cudaMemcpyAsync(origin.data(), s->d_origin, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(traw.data(), s->d_target, traw.size(), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(lraw.data(), s->d_last_tau, lraw.size(), cudaMemcpyDeviceToHost, s->stream));
  if (counters) CK(cudaMemcpyAsync(counters, s->d_counters, N * 8 * 4, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  auto rd = [&](const std::vector<unsigned char>& v, size_t i) {
    return s->precision == STP_PRECISION_F64 ? reinterpret_cast<const double*>(v.data())[i]
                                             : double(reinterpret_cast<const float*>(v.data())[i]);
  };
  if (target)
    for (size_t i = 0; i < N * 2; ++i) target[i] = origin[i] + rd(traw, i);
  if (last_tau)
    for (size_t i = 0; i < N * J; ++i) last_tau[i] = rd(lraw, i);
  return STP_OK;
}

int stp_set_task_state(stp_sim* s, const double* target, const int32_t* counters, const double* last_tau) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s) return fail(STP_EINVAL, "stp_set_task_state: null handle");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n), J = size_t(s->J);
  std::vector<double> origin(N * 2);
  CK(cudaMemcpyAsync(origin.data(), s->d_origin, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  auto put = [&](std::vector<unsigned char>& v, size_t i, double x) {
    if (s->precision == STP_PRECISION_F64) reinterpret_cast<double*>(v.data())[i] = x;
    else reinterpret_cast<float*>(v.data())[i] = float(x);
  };
  if (target) {
    std::vector<unsigned char> traw(N * 2 * s->tsize);
    for (size_t i = 0; i < N * 2; ++i) put(traw, i, target[i] - origin[i]);
    CK(cudaMemcpyAsync(s->d_target, traw.data(), traw.size(), cudaMemcpyHostToDevice, s->stream));
  }
  if (last_tau && J > 0) {
    std::vector<unsigned char> lraw(N * J * s->tsize);
    for (size_t i = 0; i < N * J; ++i) put(lraw, i, last_tau[i]);
    CK(cudaMemcpyAsync(s->d_last_tau, lraw.data(), lraw.size(), cudaMemcpyHostToDevice, s->stream));
  }
  if (counters) CK(cudaMemcpyAsync(s->d_counters, counters, N * 8 * 4, cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return STP_OK;
}

// assemble_system (solver.hpp:41-44, solver.cpp:419-446) on the device path:
// the first Newton linearisation of env `env` as the step kernel builds it
// (H over the dynamic bodies' slots, dense row-major [6S][6S], with the
// reference's block-pointer aliasing applied to block (parent, child); rhs
// [6S]) and the Krylov iterations of each Newton iteration.  The state is
// restored afterwards; pending external loads apply (and are kept).
int stp_debug_first_system(stp_sim* s, int32_t env, const double* torques, double* H, double* rhs,
                           int32_t* krylov, int32_t* n_slots) {
  const stp::DeviceGuard dg_(s ? s->device : 0);
  if (!s || env < 0 || env >= s->n || (s->J > 0 && !torques))
    return fail(STP_EINVAL, "stp_debug_first_system: bad arguments");
  if (s->task.inter_agent_collisions) return fail(STP_EINVAL, "stp_debug_first_system: single-env islands only");
  if (const int rc_ = join_caller(s)) return rc_;
  const size_t N = size_t(s->n), ts = s->tsize, W = size_t(s->W), B = size_t(s->B);
  const size_t dbg_elems = 32 * stp::kDbgStride + stp::kDbgNewton;
  if (!s->d_dbg)
    if (const int rc = dalloc(s, &s->d_dbg, dbg_elems * 8)) return rc;
  // save what a physics step changes
  void *st = nullptr, *org = nullptr, *ld = nullptr;
  const size_t st_bytes = N * stp::kStateFields * W * ts, org_bytes = N * 2 * sizeof(double),
               ld_bytes = N * 6 * W * ts;
  CK(cudaMalloc(&st, st_bytes));
  CK(cudaMalloc(&org, org_bytes));
  CK(cudaMalloc(&ld, ld_bytes));
  const bool loads = s->loads_pending;
  CK(cudaMemcpyAsync(st, s->d_state, st_bytes, cudaMemcpyDeviceToDevice, s->stream));
  CK(cudaMemcpyAsync(org, s->d_origin, org_bytes, cudaMemcpyDeviceToDevice, s->stream));
  CK(cudaMemcpyAsync(ld, s->d_loads, ld_bytes, cudaMemcpyDeviceToDevice, s->stream));
  CK(cudaMemsetAsync(s->d_dbg, 0, dbg_elems * ts, s->stream));
  std::vector<float> t(N * s->J);
  for (size_t i = 0; i < t.size(); ++i) t[i] = float(torques[i]);
  if (!t.empty()) CK(cudaMemcpyAsync(s->d_act, t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  s->dbg_env = env;
  int rc = launch(s, 0, s->d_act, nullptr, nullptr, nullptr, nullptr, nullptr, s->stream);
  s->dbg_env = -1;
  std::vector<unsigned char> raw(dbg_elems * ts);
  if (!rc) {
    CK(cudaMemcpyAsync(raw.data(), s->d_dbg, raw.size(), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaMemcpyAsync(s->d_state, st, st_bytes, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->d_origin, org, org_bytes, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->d_loads, ld, ld_bytes, cudaMemcpyDeviceToDevice, s->stream));
    s->loads_pending = loads;
  }
  CK(cudaStreamSynchronize(s->stream));
  cudaFree(st);
  cudaFree(org);
  cudaFree(ld);
  if (rc) return rc;
  auto val = [&](size_t i) -> double {
    if (ts == 8) return reinterpret_cast<const double*>(raw.data())[i];
    return double(reinterpret_cast<const float*>(raw.data())[i]);
  };
  // slots: dynamic bodies in body order (assemble_system's body_to_slot)
  int slot[STP_MAX_BODIES];
  int S = 0;
  for (size_t b = 0; b < B; ++b) slot[b] = s->model.bodies[b].is_static ? -1 : S++;
  const size_t n6 = size_t(6) * S;
  if (n_slots) *n_slots = S;
  auto sidx = [](int r, int c) { return r >= c ? r * (r + 1) / 2 + c : c * (c + 1) / 2 + r; };
  if (H) std::fill(H, H + n6 * n6, 0.0);
  for (size_t b = 0; b < B; ++b) {
    if (slot[b] < 0) continue;
    const size_t o = b * stp::kDbgStride, i0 = size_t(6) * slot[b];
    if (H)
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) H[(i0 + r) * n6 + i0 + c] = val(o + sidx(r, c));
    if (rhs)
      for (int r = 0; r < 6; ++r) rhs[i0 + r] = val(o + 21 + r);
  }
  for (int j = 0; H && j < s->J; ++j) {
    const stp_joint& jd = s->model.joints[j];
    const int c = jd.child, p = jd.parent;
    if (slot[c] < 0 || slot[p] < 0) continue;
    const size_t o = size_t(c) * stp::kDbgStride, ci = size_t(6) * slot[c], pi = size_t(6) * slot[p];
    double hcp[36];
    for (int k = 0; k < 36; ++k) hcp[k] = val(o + 27 + k);
    const double d0 = val(o + 63);
    const double ja0[6] = {-1, 0, 0, val(o + 64), val(o + 65), val(o + 66)};
    const double jb0[6] = {1, 0, 0, val(o + 67), val(o + 68), val(o + 69)};
    for (int r = 0; r < 6; ++r)
      for (int k = 0; k < 6; ++k) {
        H[(ci + r) * n6 + pi + k] = hcp[r * 6 + k];                             // H(child, parent)
        H[(pi + k) * n6 + ci + r] = hcp[r * 6 + k] - d0 * ja0[k] * jb0[r];      // H(parent, child)
      }
  }
  if (krylov)
    for (int it = 0; it < s->cfg.newton_iters && it < stp::kDbgNewton; ++it)
      krylov[it] = int32_t(val(32 * stp::kDbgStride + it));
  return STP_OK;
}

}  // extern "C"
