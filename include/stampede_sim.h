/*
 * stampede_sim.h — C-ABI of the B200-native batched locomotion simulator.
 *
 * This is the drop-in boundary for the data-parallel hot path of the
 * reference (`stampede`, /root/reference/proj): stepping N independent
 * Ant/Humanoid environments.  Every entry point names the reference
 * interface it replaces (file:line under /root/reference/proj or SPEC.md).
 *
 * Conventions
 *  - Plain C types only; no torch or C++ types cross this boundary.
 *  - Functions return STP_OK (0) or a negative/positive status code; the
 *    human-readable reason is available from stp_last_error() (thread-local).
 *    No C++ exception ever crosses the ABI (the reference throws
 *    std::invalid_argument at the same preconditions, see each entry).
 *  - "device" pointers are CUDA device pointers on the handle's device;
 *    "host" pointers are ordinary (preferably pinned) host memory.
 *  - All calls on one handle are asynchronous on the given CUDA stream
 *    (NULL = the handle's own stream) unless documented as synchronous.
 *    The synchronous accessors (state, loads, contacts, report, task state,
 *    snapshots, terrain, the host-buffer steps) order themselves after the
 *    most recent launch made on a caller's stream, so e.g. stp_get_state
 *    right after an asynchronous stp_step sees that step.
 *    A handle is not reentrant (reference Scene is not either,
 *    solver.hpp:46-53); use one handle per GPU / per process.
 *  - Per-body state layout in host buffers is the reference's
 *    RigidBodyState order (types.hpp:28-32; identical to the snapshot
 *    layout scene.cpp:85-90): position xyz, orientation wxyz,
 *    linear velocity xyz, angular velocity xyz = 13 doubles per body.
 */
#ifndef STAMPEDE_SIM_H
#define STAMPEDE_SIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STP_ABI_VERSION 2
#define STP_MAX_BODIES 32
#define STP_MAX_JOINTS 31
#define STP_MAX_FEET 4
#define STP_STATE_STRIDE 13

/* status codes */
#define STP_OK 0
#define STP_EINVAL 22  /* invalid argument (reference: std::invalid_argument) */
#define STP_ENOMEM 12  /* device/host allocation failed                      */
#define STP_ECUDA 100  /* CUDA runtime error                                 */
#define STP_ESTATE 101 /* call not valid in the handle's current state       */

/* ShapeType, types.hpp:47 */
#define STP_SPHERE 0
#define STP_CAPSULE 1
#define STP_BOX 2

/* task kinds, SPEC.md:240 (TaskConfig.kind) */
#define STP_TASK_ANT 0
#define STP_TASK_HUMANOID 1
#define STP_TASK_HFH 2
#define STP_TASK_HFH_TERRAIN 3

/* arithmetic of the device kernels */
#define STP_PRECISION_F32 0
#define STP_PRECISION_F64 1 /* parity instrument: same kernels instantiated in double */

/* One rigid body: Shape (types.hpp:49-56) + BodyInertial (types.hpp:40-44). */
typedef struct stp_body {
  int32_t shape; /* STP_SPHERE / STP_CAPSULE / STP_BOX; capsule axis = local z */
  int32_t is_static;
  double radius;
  double half_length;     /* capsule cylinder half length */
  double half_extents[3]; /* box */
  double local_pos[3];
  double local_rot[4]; /* w x y z */
  double mass;
  double inertia_diag[3]; /* principal body frame */
} stp_body;

/* Hinge joint, JointDesc types.hpp:60-71. */
typedef struct stp_joint {
  int32_t parent, child;
  double anchor_parent[3], anchor_child[3];
  double axis_parent[3], axis_child[3];
  double rest_relative[4]; /* parent->child orientation at angle zero (w x y z) */
  double limit_lo, limit_hi, max_torque;
} stp_joint;

/* Articulation model (SPEC.md:187-190 ArticulationModel).  Joint j must
 * have child > parent (tree in topological order); the GPU path maps one
 * body to one lane of a warp, so n_bodies <= 32. */
typedef struct stp_model {
  char name[32];
  int32_t n_bodies, n_joints;
  int32_t root;
  int32_t n_feet;
  int32_t feet[STP_MAX_FEET];
  stp_body bodies[STP_MAX_BODIES];
  stp_joint joints[STP_MAX_JOINTS];
  double rest_state[STP_MAX_BODIES][STP_STATE_STRIDE]; /* rest pose, root at xy = 0 */
  double fall_height; /* SPEC.md:342 fall thresholds */
  double alive_bonus; /* PAPER.md App. C: 0.5 ant, 2 humanoid */
} stp_model;

/* StepConfig (types.hpp:92-107) + the Scene-level gravity and ground flag
 * (scene.hpp:37-39). */
typedef struct stp_step_config {
  double dt;
  int32_t newton_iters;
  double krylov_tol;
  int32_t krylov_max_iters;
  double contact_margin;
  double baumgarte;
  double joint_hardness;
  double contact_hardness;
  double limit_hardness;
  double friction_smoothing;
  double limit_activation;
  double gravity[3];
  int32_t has_ground_plane;
  /* 1 (default) = reproduce the reference's block-pointer aliasing in
   * assemble (solver.cpp:350-351 + block_sparse.cpp:33-37): when creating
   * block (b,a) reallocates the block pool, the first row's contribution
   * to block (a,b) is lost.  0 = the symmetric system the reference
   * intends.  See DESIGN.md §"Reference quirks". */
  int32_t reference_alias_quirk;
} stp_step_config;

/* StaticBox, types.hpp:86-90 (terrain obstacle resting in world space). */
typedef struct stp_static_box {
  double center[3];
  double half_extents[3];
  double yaw;
} stp_static_box;

/* TerrainSpec. Boxes rest on z = 0. */
typedef struct stp_terrain_spec {
  int32_t count;
  double dim_lo, dim_hi;  /* full edge length range (m) */
  double x_lo, x_hi, y_lo, y_hi;
  double yaw_lo, yaw_hi;
  uint64_t seed;
} stp_terrain_spec;

/* TaskConfig plus the design decisions recorded in
 * DESIGN.md §"env layer". */
typedef struct stp_task {
  int32_t kind;
  int32_t episode_cap;    /* 1000 frames */
  int32_t fall_grace;     /* 0 (Ant/Humanoid) or 160 (HFH) consecutive frames */
  int32_t target_refresh; /* 200 frames (HFH) */
  double target_radius;   /* 100 m */
  double target_tolerance;/* 1 m */
  double spacing;         /* initial grid spacing, 3 m (2 m HFH) */
  int32_t perturb_min, perturb_max; /* next perturbation in U{min..max} frames */
  double perturb_force_lo, perturb_force_hi; /* N, horizontal, root body */
  double reset_noise;     /* +-0.05 uniform on every initial DoF */
  int32_t auto_reset;     /* reset done envs inside stp_step */
  int32_t height_map;     /* append the 15x11 height map (HFH terrain) */
  int32_t inter_agent_collisions; /* Scene::inter_agent_collisions (scene.hpp), set for the
                                     HFH tasks by reset: contacts between
                                     agents merge their envs into one island */
} stp_task;

typedef struct stp_sim stp_sim;

/* --- configuration helpers (host, synchronous) --------------------------- */
int stp_abi_version(void);
const char* stp_last_error(void);
/* StepConfig defaults, types.hpp:92-107; gravity (0,0,-9.8) scene.hpp:39. */
void stp_default_step_config(stp_step_config* cfg);
/* Bundled assets ("ant", "humanoid"), SPEC.md:199-201 load_model examples. */
int stp_builtin_model(const char* name, stp_model* out);
/* Validation with the reference's rules, Scene::validate scene.cpp:36-68. */
int stp_validate_model(const stp_model* model);
int stp_default_task(int32_t kind, stp_task* out);
/* load_model / serialize: the line-oriented
 * articulation text format "stampede-model 1" (grammar in csrc/models.cpp and
 * DESIGN.md §5).  Parse errors name the line and field (STP_EINVAL); the
 * result is checked with stp_validate_model.  to_text writes at most
 * capacity-1 bytes + NUL and reports the full length; load(to_text(m)) == m. */
int stp_model_from_text(const char* text, stp_model* out);
int stp_model_to_text(const stp_model* model, char* buffer, int32_t capacity, int32_t* length);
/* generate_terrain, SPEC.md:206-214 (counter-based RNG: deterministic). */
int stp_generate_terrain(const stp_terrain_spec* spec, stp_static_box* out, int32_t capacity);
/* terrain_height, collide.cpp:348-359 (host, double; used by tests). */
double stp_terrain_height(const stp_static_box* boxes, int32_t n, double x, double y);

/* sizeof every ABI struct, for binding layout checks: stp_body, stp_joint,
 * stp_model, stp_step_config, stp_static_box, stp_terrain_spec, stp_task. */
void stp_struct_sizes(int64_t out[7]);

/* --- handle lifecycle ------------------------------------------------------ */
/* Creates n_envs environments of `model` on CUDA device `device`.
 * env_offset = global index of this handle's first env (rank * n_envs for a
 * sharded multi-GPU run): every random draw is keyed by the global index, so a
 * G-GPU run is the 1-GPU run partitioned.
 * Returns NULL on failure (see stp_last_error). */
stp_sim* stp_create(const stp_model* model, const stp_task* task, const stp_step_config* cfg,
                    int32_t n_envs, int32_t device, uint64_t seed, int32_t precision,
                    int64_t env_offset);
void stp_destroy(stp_sim* sim);
/* Replace the static terrain boxes (Scene::static_boxes, scene.hpp:38). */
int stp_set_terrain(stp_sim* sim, const stp_static_box* boxes, int32_t n);

int32_t stp_num_envs(const stp_sim* sim);
int32_t stp_obs_dim(const stp_sim* sim);    /* 76 / 241 / 39 */
int32_t stp_action_dim(const stp_sim* sim); /* actuated joints */
int32_t stp_contact_capacity(const stp_sim* sim); /* contact slots per env */
void* stp_stream(const stp_sim* sim);       /* the handle's cudaStream_t */

/* --- the hot path ---------------------------------------------------------- */
/* reset: env_mask is a device uint8[N] (1 = reset) or NULL
 * for all envs.  obs (device float[N*obs_dim]) may be NULL. */
int stp_reset(stp_sim* sim, const uint8_t* env_mask, float* obs, void* stream);

/* env_step: device buffers. actions float[N*A] in [-1,1]
 * (scaled by tau_max), obs float[N*O], reward float[N],
 * done uint8[N].  Any of obs/reward/done may be NULL. */
int stp_step(stp_sim* sim, const float* actions, float* obs, float* reward, uint8_t* done,
             void* stream);

/* Same call with HOST buffers: copies actions H->D, steps, copies
 * obs/reward/done D->H and synchronises the stream (end-to-end path). */
int stp_step_host(stp_sim* sim, const float* actions, float* obs, float* reward, uint8_t* done);

/* physics::step (solver.hpp:52-53, solver.cpp:448-597) on every env:
 * torques device float[N*J] in N*m (clamped like clamp_torques,
 * solver.cpp:395-403).  External loads set by stp_set_external_loads are
 * consumed and cleared (scene.cpp:75-78). */
int stp_physics_step(stp_sim* sim, const float* torques, void* stream);
/* Host-buffer variant (double torques), synchronous; used by parity tests. */
int stp_physics_step_host(stp_sim* sim, const double* torques);

/* Fill device float[N*A] with i.i.d. U[-1,1] actions keyed by
 * derive_seed(seed, TAG_ACTION, env<<32 | step) (rng.hpp:35-37). */
int stp_random_actions(stp_sim* sim, float* actions, uint64_t step, void* stream);

/* --- state / report access (host buffers, synchronous) --------------------- */
int stp_set_state(stp_sim* sim, const double* state);  /* N*B*13 */
int stp_get_state(stp_sim* sim, double* state);        /* N*B*13 */
/* Scene::external_force/torque (scene.hpp:45-46) for the next physics step:
 * host double[N*B*6] = force xyz, torque xyz per body. */
int stp_set_external_loads(stp_sim* sim, const double* loads);
/* Ordered contact list of the last physics step per env (detect_contacts
 * order, collide.cpp:283-299) with the solved impulses (SolvedContact,
 * types.hpp:109-113).  count int32[N]; per slot (N*capacity): body_a,
 * body_b (-1 static; an inter-agent contact is listed with body_a's env after
 * its static contacts, body_b = the partner's global index env * B + body),
 * point[3], normal[3], separation, normal impulse, tangential impulse[3].
 * Any output pointer may be NULL. */
int stp_get_contacts(stp_sim* sim, int32_t* count, int32_t* body_a, int32_t* body_b,
                     double* point, double* normal, double* separation,
                     double* normal_impulse, double* tangential_impulse);
/* Scene snapshot "SSNP" v1 (Scene::save_snapshot / load_snapshot,
 * scene.cpp:80-104): u32 magic 0x504e5353, u32 version 1, u64 body count, then
 * per body (env-major = scene body order) 13 little-endian f64: position,
 * orientation (w x y z), linear velocity, angular velocity.  Byte-compatible
 * with the reference; load rejects a bad magic / version / body count with the
 * reference's messages (STP_EINVAL). */
int64_t stp_snapshot_size(const stp_sim* sim);
int stp_save_snapshot(stp_sim* sim, uint8_t* buffer, int64_t capacity);
int stp_load_snapshot(stp_sim* sim, const uint8_t* buffer, int64_t size);
/* Inter-agent contacts of the current state: the pairs
 * detect_contacts (collide.cpp:300-343) appends when
 * Scene::inter_agent_collisions is set — dynamic sphere/capsule bodies of
 * different envs whose AABBs overlap within the margin, one segment-segment
 * contact each (:219-266), in (body_a, body_b) order.  Body indices are global
 * within the sim (env * B + body).  count = total pairs; at most capacity
 * entries are written; any array may be NULL.  Detection only: the step does
 * not yet solve contact-merged islands. */
int stp_detect_inter_agent(stp_sim* sim, int32_t capacity, int32_t* count, int32_t* body_a, int32_t* body_b,
                           double* point, double* normal, double* separation);
/* StepReport (types.hpp:115-120) of the last physics step, per env:
 * newton iterations, krylov iterations, failed (rolled back) flag,
 * contact overflow flag (more contacts than slots; should stay 0). */
int stp_get_report(stp_sim* sim, int32_t* newton_iters, int32_t* krylov_iters, uint8_t* failed,
                   uint8_t* overflow);
/* Task state per env (host): target xy [N*2] (double), counters [N*8]
 * (frame, flag_frames, fall_frames, next_perturb, episode, flag_draws,
 * perturb_draws, reserved), last normalised torques [N*A] (double).
 * Any pointer may be NULL. */
int stp_get_task_state(stp_sim* sim, double* target, int32_t* counters, double* last_torque);
int stp_set_task_state(stp_sim* sim, const double* target, const int32_t* counters,
                       const double* last_torque);

/* --- K4: rollout policy forward on tcgen05 tensor cores ---------------------
 * SPEC.md:366-409 (SELU MLP, Gaussian policy) and :446-454 (whitening):
 *   x = clip((obs - mean) / std, +-10);  mean = MLP_pi(x);  value = MLP_v(x);
 *   action = mean + exp(log_std) * eps (eps ~ N(0,1), counter-based,
 *   derive_seed(seed, 6, env<<32 | step)); logp = log N(action; mean, std).
 * dims_* = {in, h1, h2, h3, out} (widths <= 256); w_*[l] = packed bf16
 * weights of layer l, K-major core-matrix layout [ceil16(in)/8][ceil16(out)][8]
 * (paper_1810_05762_b200/policy.py pack_linear); b_*[l] = fp32 bias padded to
 * ceil16(out); weights and biases 16-byte aligned.  All pointers are device
 * pointers; asynchronous on `stream`.
 * action_out / logp_out / value_out may be NULL. */
int stp_policy_forward(const float* obs, int32_t n_envs, int32_t obs_dim, const float* obs_mean,
                       const float* obs_std, const int32_t* dims_pi, const void* const* w_pi,
                       const float* const* b_pi, const int32_t* dims_v, const void* const* w_v,
                       const float* const* b_v, const float* log_std, uint64_t seed, uint64_t step,
                       int64_t env_offset, float* mean_out, float* action_out, float* logp_out,
                       float* value_out, void* stream);

/* --- PPO learner data path (config C5) ----------------
 * compute_gae over the rollout buffer, all device pointers
 * of [T][N] (time-major) fp32 rewards / values, uint8 dones, fp32 bootstrap
 * values [N]:  delta_t = r_t + gamma V_{t+1} (1 - done_t) - V_t,
 * A_t = delta_t + gamma lambda (1 - done_t) A_{t+1}, returns = A + V.
 * stats (device double[3], may be NULL) accumulates count, sum(A), sum(A^2)
 * for the (global) advantage normalisation; the caller
 * zeroes it.  Asynchronous on `stream`. */
int stp_gae(const float* rewards, const float* values, const uint8_t* dones, const float* last_value, int32_t T,
            int32_t N, float gamma, float lam, float* advantages, float* returns, double* stats, void* stream);

/* ppo_update's minibatch loss (clipped surrogate on the
 * globally normalised advantages + vf_coef x value MSE) and its gradient with
 * respect to the networks' outputs, for the PPO learner of config C5.
 * mu [B][A] (policy means) and value [B] are the networks' outputs on the
 * minibatch's samples in minibatch order; actions [*][A], old_logp, advantages
 * and returns [*] are the rollout columns, read at row idx[i] for sample i
 * (idx = NULL: row i) — the minibatch gather.  adv_stats = the advantages'
 * (count, sum, sum of squares), already summed over ranks (NULL: advantages
 * used as given).  Writes d_mu [B][A], d_value [B], d_log_std [A] (dL/d of
 * each; the policy's log-std enters only through the log-prob), the output
 * layers' bias gradients d_mu_bias [A] = sum_i d_mu[i] and d_value_bias [1]
 * (either may be NULL), loss[3] = (total, surrogate, value error) and sets
 * *bad = 1 when the total is not finite (bad may be NULL).
 * scratch: double[ceil(B / 128) * (2A + 3)].
 * Deterministic (fixed-order reductions); asynchronous on `stream`.
 * 1 <= A <= 32. */
int stp_ppo_surrogate(const float* mu, const float* log_std, const float* value, const float* actions,
                      const float* old_logp, const float* advantages, const float* returns, const int64_t* idx,
                      int32_t B, int32_t A, const double* adv_stats, float clip, float vf_coef, float* d_mu,
                      float* d_value, float* d_log_std, float* d_mu_bias, float* d_value_bias, float* loss,
                      float* bad, double* scratch, void* stream);

/* KL(old || new) of the diagonal Gaussian policies (kl_diag_gaussian,
 * SPEC.md:428-436) averaged over B states: mu_old / mu_new [B][A], log-stds
 * [A]; *kl_mean (device float) = mean_i sum_j (ls1 - ls0 + (s0^2 + (mu0 -
 * mu1)^2) / (2 s1^2) - 1/2), the input of the learning-rate rule (:468-475).
 * scratch: double[ceil(B / 256)].  Deterministic; asynchronous on `stream`. */
int stp_ppo_kl(const float* mu_old, const float* log_std_old, const float* mu_new, const float* log_std_new,
               int32_t B, int32_t A, float* kl_mean, double* scratch, void* stream);

/* Backward of a hidden layer's SELU in the PPO learner: grad [rows][H]
 * (dL/d the layer's output, overwritten with dL/d its pre-activation, using
 * the output `out` [rows][H]: selu'(z) = lambda for out > 0, else
 * out + lambda alpha) and d_bias [H] = the column sums of the result (the
 * layer's bias gradient), reduced in a fixed order (deterministic).
 * H % 4 == 0, H <= 1024, 16-byte aligned rows; scratch: float[592 * H].
 * Asynchronous on `stream`. */
int stp_selu_backward_bias(float* grad, const float* out, int64_t rows, int32_t H, float* d_bias, float* scratch,
                           void* stream);

/* Forward epilogue of a learner layer: z [rows][H] += bias [H], then SELU
 * (lambda z for z > 0, lambda alpha (e^z - 1) else; selu = 0: bias only), in
 * place.  H % 4 == 0, 16-byte aligned.  Asynchronous on `stream`. */
int stp_bias_selu(float* z, const float* bias, int64_t rows, int32_t H, int32_t selu, void* stream);

/* assemble_system (solver.hpp:41-44, solver.cpp:419-446) on the device path:
 * the first Newton linearisation of env `env` for host torques [N*J] (N*m)
 * exactly as the step kernel assembles it — H dense row-major [6S x 6S] over
 * the S dynamic bodies in body order (AssembledSystem::body_to_slot), the
 * reference's block-pointer aliasing applied to block (parent, child) when
 * stp_step_config.reference_alias_quirk is set; rhs [6S] — and the Krylov
 * iterations of each Newton iteration (krylov[newton_iters]).  The handle's
 * state is left unchanged.  Envs without inter-agent coupling only.  Any
 * output may be NULL; n_slots receives S. */
int stp_debug_first_system(stp_sim* sim, int32_t env, const double* torques, double* H, double* rhs,
                           int32_t* krylov, int32_t* n_slots);

/* --- diagnostics (tests only; not part of the reference interface) ---------
 * The fp32 step kernel's own elementary functions on device arrays, so their
 * accuracy is tested directly: fn 0 = sincos (Cody-Waite +
 * Cephes) of x -> (out0 = sin, out1 = cos); fn 1 = the unit-vector bearing
 * (sin, cos) of atan2(x, y) used by the heading terms.  Asynchronous. */
int stp_debug_math(int32_t fn, const float* x, const float* y, float* out0, float* out1, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STAMPEDE_SIM_H */
