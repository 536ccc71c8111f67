"""Python host mirror of the reference's batched env / physics interface.

Names and argument meaning follow the reference:
  * ``VecEnv.reset`` / ``VecEnv.step``       — SPEC.md:261-278 (reset, env_step)
  * ``VecEnv.physics_step``                  — stampede::physics::step
                                               (solver.hpp:52-53; torques in N*m)
  * ``VecEnv.get_state`` / ``set_state``     — Scene::states in RigidBodyState order
                                               (types.hpp:28-32), shape [N, B, 13]
  * ``VecEnv.contacts`` / ``report``         — StepReport (types.hpp:109-120)
Errors raise ``ValueError`` where the reference throws std::invalid_argument
and ``RuntimeError`` for CUDA failures.  Everything runs through the C-ABI in
``libstampede_b200.so``; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi

TASKS = {"ant": abi.TASK_ANT, "humanoid": abi.TASK_HUMANOID, "hfh": abi.TASK_HFH,
         "hfh_terrain": abi.TASK_HFH_TERRAIN}
MODEL_OF_TASK = {"ant": "ant", "humanoid": "humanoid", "hfh": "humanoid", "hfh_terrain": "humanoid"}


def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "arrays passed to the C-ABI must be contiguous"
        return C.c_void_p(a.ctypes.data)
    # torch tensor
    assert a.is_contiguous(), "tensors passed to the C-ABI must be contiguous"
    return C.c_void_p(a.data_ptr())


def _raise(rc: int, what: str):
    if rc == abi.STP_OK:
        return
    msg = abi.last_error()
    if rc == abi.STP_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (status {rc}): {msg}")


@dataclass
class Contact:
    body_a: int
    body_b: int
    point: np.ndarray
    normal: np.ndarray
    separation: float
    normal_impulse: float
    tangential_impulse: np.ndarray


class VecEnv:
    """N independent environments stepped by the fused sm_100a kernel."""

    def __init__(self, task: str = "humanoid", n_envs: int = 1024, device: int = 0, seed: int = 1234,
                 precision: str = "f32", env_offset: int = 0, model: abi.Model | None = None,
                 step_config: abi.StepConfig | None = None, task_config: abi.Task | None = None,
                 terrain: list | None = None):
        self.lib = abi.load()
        self.task_name = task
        self.model = model if model is not None else abi.builtin_model(MODEL_OF_TASK[task])
        self.cfg = step_config if step_config is not None else abi.default_step_config()
        self.task = task_config if task_config is not None else abi.default_task(TASKS[task])
        self.n_envs = int(n_envs)
        self.device = int(device)
        self.precision = abi.PRECISION_F64 if precision == "f64" else abi.PRECISION_F32
        h = self.lib.stp_create(C.byref(self.model), C.byref(self.task), C.byref(self.cfg), self.n_envs,
                                self.device, C.c_uint64(seed), self.precision, C.c_int64(env_offset))
        if not h:
            msg = abi.last_error()
            if "cuda" in msg.lower() and "invalid" not in msg.lower():
                raise RuntimeError(f"stp_create failed: {msg}")
            raise ValueError(f"stp_create: {msg}")
        self._h = C.c_void_p(h)
        self.obs_dim = int(self.lib.stp_obs_dim(self._h))
        self.action_dim = int(self.lib.stp_action_dim(self._h))
        self.n_bodies = int(self.model.n_bodies)
        self.contact_capacity = int(self.lib.stp_contact_capacity(self._h))
        if terrain is not None:
            self.set_terrain(terrain)

    # ------------------------------------------------------------------ life
    def close(self):
        if getattr(self, "_h", None):
            self.lib.stp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def stream(self) -> int:
        return int(self.lib.stp_stream(self._h) or 0)

    @staticmethod
    def _torch_stream():
        """torch's current stream; its legacy default stream (handle 0) is passed
        as cudaStreamLegacy (0x1) because NULL means "the handle's own stream"."""
        import torch
        h = torch.cuda.current_stream().cuda_stream
        return C.c_void_p(h if h else 1)

    def set_terrain(self, boxes):
        arr = (abi.StaticBox * max(1, len(boxes)))()
        for i, b in enumerate(boxes):
            arr[i] = b
        _raise(self.lib.stp_set_terrain(self._h, arr, len(boxes)), "set_terrain")
        self.contact_capacity = int(self.lib.stp_contact_capacity(self._h))

    # ------------------------------------------------------------ env API
    def reset(self, mask=None):
        """SPEC reset: returns device obs [N, obs_dim] (torch)."""
        import torch
        obs = torch.empty((self.n_envs, self.obs_dim), dtype=torch.float32, device=f"cuda:{self.device}")
        m = None
        if mask is not None:
            m = torch.as_tensor(mask, dtype=torch.uint8, device=obs.device).contiguous()
        _raise(self.lib.stp_reset(self._h, _ptr(m), _ptr(obs), self._torch_stream()), "reset")
        return obs

    def step(self, actions, obs=None, reward=None, done=None):
        """SPEC env_step on device tensors; async on torch's current stream.
        A numpy array routes through the host-buffer entry (stp_step_host)."""
        if isinstance(actions, np.ndarray):
            return self.step_host(actions, obs, reward, done)
        import torch
        dev = f"cuda:{self.device}"
        if actions.shape != (self.n_envs, self.action_dim):
            raise ValueError(f"env_step: actions must have shape {(self.n_envs, self.action_dim)}")
        actions = actions.to(device=dev, dtype=torch.float32).contiguous()
        if obs is None:
            obs = torch.empty((self.n_envs, self.obs_dim), dtype=torch.float32, device=dev)
        if reward is None:
            reward = torch.empty((self.n_envs,), dtype=torch.float32, device=dev)
        if done is None:
            done = torch.empty((self.n_envs,), dtype=torch.uint8, device=dev)
        _raise(self.lib.stp_step(self._h, _ptr(actions), _ptr(obs), _ptr(reward), _ptr(done),
                                 self._torch_stream()), "env_step")
        return obs, reward, done

    def step_host(self, actions: np.ndarray, obs=None, reward=None, done=None):
        """env_step through host buffers (H2D + kernel + D2H, synchronous)."""
        actions = np.ascontiguousarray(actions, dtype=np.float32)
        if actions.shape != (self.n_envs, self.action_dim):
            raise ValueError(f"env_step: actions must have shape {(self.n_envs, self.action_dim)}")
        obs = np.empty((self.n_envs, self.obs_dim), np.float32) if obs is None else obs
        reward = np.empty((self.n_envs,), np.float32) if reward is None else reward
        done = np.empty((self.n_envs,), np.uint8) if done is None else done
        _raise(self.lib.stp_step_host(self._h, _ptr(actions), _ptr(obs), _ptr(reward), _ptr(done)), "env_step")
        return obs, reward, done

    def random_actions(self, step: int, out=None):
        import torch
        if out is None:
            out = torch.empty((self.n_envs, self.action_dim), dtype=torch.float32, device=f"cuda:{self.device}")
        _raise(self.lib.stp_random_actions(self._h, _ptr(out), C.c_uint64(step), self._torch_stream()),
               "random_actions")
        return out

    # -------------------------------------------------------- physics API
    def physics_step(self, torques: np.ndarray):
        """physics::step on every env with host torques [N, J] (N*m); synchronous."""
        t = np.ascontiguousarray(torques, dtype=np.float64)
        if t.size != self.n_envs * self.action_dim:
            raise ValueError("clamp_torques: torque count must equal joint count")
        _raise(self.lib.stp_physics_step_host(self._h, _ptr(t)), "physics_step")

    def physics_step_device(self, torques):
        _raise(self.lib.stp_physics_step(self._h, _ptr(torques), self._torch_stream()), "physics_step")

    def get_state(self) -> np.ndarray:
        s = np.empty((self.n_envs, self.n_bodies, 13), np.float64)
        _raise(self.lib.stp_get_state(self._h, _ptr(s)), "get_state")
        return s

    def set_state(self, state: np.ndarray):
        s = np.ascontiguousarray(state, dtype=np.float64).reshape(self.n_envs, self.n_bodies, 13)
        _raise(self.lib.stp_set_state(self._h, _ptr(s)), "set_state")

    def set_external_loads(self, loads: np.ndarray):
        l = np.ascontiguousarray(loads, dtype=np.float64).reshape(self.n_envs, self.n_bodies, 6)
        _raise(self.lib.stp_set_external_loads(self._h, _ptr(l)), "set_external_loads")

    def contact_arrays(self):
        N, C_ = self.n_envs, self.contact_capacity
        out = dict(count=np.zeros(N, np.int32), body_a=np.full((N, C_), -1, np.int32),
                   body_b=np.full((N, C_), -1, np.int32), point=np.zeros((N, C_, 3)), normal=np.zeros((N, C_, 3)),
                   separation=np.zeros((N, C_)), normal_impulse=np.zeros((N, C_)),
                   tangential_impulse=np.zeros((N, C_, 3)))
        _raise(self.lib.stp_get_contacts(self._h, _ptr(out["count"]), _ptr(out["body_a"]), _ptr(out["body_b"]),
                                         _ptr(out["point"]), _ptr(out["normal"]), _ptr(out["separation"]),
                                         _ptr(out["normal_impulse"]), _ptr(out["tangential_impulse"])),
               "get_contacts")
        return out

    def save_snapshot(self) -> bytes:
        """Scene snapshot "SSNP" v1 (scene.cpp:80-104), byte-compatible with the reference."""
        buf = np.zeros(int(self.lib.stp_snapshot_size(self._h)), np.uint8)
        _raise(self.lib.stp_save_snapshot(self._h, _ptr(buf), buf.size), "save_snapshot")
        return buf.tobytes()

    def load_snapshot(self, data: bytes):
        buf = np.frombuffer(data, np.uint8).copy()
        _raise(self.lib.stp_load_snapshot(self._h, _ptr(buf), buf.size), "load_snapshot")

    def detect_inter_agent(self, capacity: int | None = None):
        """Inter-agent contacts of the current state (row A7, detect_contacts
        with inter_agent_collisions, collide.cpp:300-343): global body indices
        env * B + body, the reference's (a, b) order."""
        cap = capacity if capacity is not None else 4 * self.n_envs * self.n_bodies
        out = dict(body_a=np.zeros(cap, np.int32), body_b=np.zeros(cap, np.int32), point=np.zeros((cap, 3)),
                   normal=np.zeros((cap, 3)), separation=np.zeros(cap))
        n = np.zeros(1, np.int32)
        _raise(self.lib.stp_detect_inter_agent(self._h, cap, _ptr(n), _ptr(out["body_a"]), _ptr(out["body_b"]),
                                               _ptr(out["point"]), _ptr(out["normal"]), _ptr(out["separation"])),
               "detect_inter_agent")
        k = min(int(n[0]), cap)
        return {key: v[:k] for key, v in out.items()}

    def contacts(self, env: int) -> list[Contact]:
        a = self.contact_arrays()
        n = min(int(a["count"][env]), self.contact_capacity)
        return [Contact(int(a["body_a"][env, i]), int(a["body_b"][env, i]), a["point"][env, i],
                        a["normal"][env, i], float(a["separation"][env, i]), float(a["normal_impulse"][env, i]),
                        a["tangential_impulse"][env, i]) for i in range(n)]

    def report(self):
        N = self.n_envs
        newton, krylov = np.zeros(N, np.int32), np.zeros(N, np.int32)
        failed, overflow = np.zeros(N, np.uint8), np.zeros(N, np.uint8)
        _raise(self.lib.stp_get_report(self._h, _ptr(newton), _ptr(krylov), _ptr(failed), _ptr(overflow)),
               "get_report")
        return dict(newton_iterations=newton, krylov_iterations=krylov, failed=failed, overflow=overflow)

    def first_system(self, env: int, torques):
        """assemble_system (solver.hpp:41-44) of env `env` as the CUDA step
        builds it: (H [6S, 6S], rhs [6S], krylov iterations per Newton
        iteration, S); the state is left unchanged."""
        t = np.ascontiguousarray(torques, dtype=np.float64).reshape(self.n_envs, self.action_dim)
        S = sum(1 for b in range(self.n_bodies) if not self.model.bodies[b].is_static)
        H, rhs = np.zeros((6 * S, 6 * S)), np.zeros(6 * S)
        kry = np.zeros(max(1, self.cfg.newton_iters), np.int32)
        ns = np.zeros(1, np.int32)
        _raise(self.lib.stp_debug_first_system(self._h, int(env), _ptr(t), _ptr(H), _ptr(rhs), _ptr(kry), _ptr(ns)),
               "first_system")
        return H, rhs, kry[:self.cfg.newton_iters], int(ns[0])

    def task_state(self):
        N, J = self.n_envs, self.action_dim
        target, counters, last = np.zeros((N, 2)), np.zeros((N, 8), np.int32), np.zeros((N, max(J, 1)))
        _raise(self.lib.stp_get_task_state(self._h, _ptr(target), _ptr(counters), _ptr(last)), "get_task_state")
        return dict(target=target, counters=counters, last_tau=last[:, :J])

    def set_task_state(self, target=None, counters=None, last_tau=None):
        t = None if target is None else np.ascontiguousarray(target, np.float64)
        c = None if counters is None else np.ascontiguousarray(counters, np.int32)
        l = None if last_tau is None else np.ascontiguousarray(last_tau, np.float64)
        _raise(self.lib.stp_set_task_state(self._h, _ptr(t), _ptr(c), _ptr(l)), "set_task_state")
