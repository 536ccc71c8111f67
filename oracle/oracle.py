"""ORACLE — TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py
CPU baseline / reference arm).  Never imported by the product package.

ctypes wrapper over the `orc_*` C API of
  * oracle/liboracle.so                  — restated reference physics
                                           (phys_oracle.hpp, double or float)
  * oracle/_ref/libstampede_ref.so       — the compiled, unmodified reference
                                           stampede::physics::step (parity build)
  * oracle/_ref/libstampede_ref_fast.so  — same, reference Release flags (timing)
with the same method names as paper_1810_05762_b200.sim.VecEnv.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libstampede_ref.so"),
    "reference_fast": os.path.join(HERE, "_ref", "libstampede_ref_fast.so"),
}


def build(reference: bool = True) -> None:
    """Compile the oracle (and, when /root/reference exists, oracle/_ref)."""
    targets = ["liboracle.so"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-j4"] + targets, cwd=HERE, check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


_cache: dict[str, C.CDLL] = {}


def _lib(kind: str) -> C.CDLL:
    if kind in _cache:
        return _cache[kind]
    path = LIBS[kind]
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle library {path} not built (run oracle.build())")
    from paper_1810_05762_b200 import abi  # struct layouts only (the shared boundary header)
    L = C.CDLL(path)
    P = C.c_void_p
    L.orc_create.restype = P
    L.orc_create.argtypes = [C.POINTER(abi.Model), C.POINTER(abi.Task), C.POINTER(abi.StepConfig), C.c_int32,
                             C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32]
    L.orc_destroy.argtypes = [P]
    L.orc_last_error.restype = C.c_char_p
    L.orc_backend.restype = C.c_char_p
    L.orc_backend.argtypes = [P]
    L.orc_obs_dim.argtypes = [P]
    for name in ["orc_set_state", "orc_get_state", "orc_set_external_loads", "orc_physics_step", "orc_observe"]:
        getattr(L, name).argtypes = [P, P]
    L.orc_set_terrain.argtypes = [P, P, C.c_int32]
    L.orc_reset.argtypes = [P, P, P]
    L.orc_step.argtypes = [P, P, P, P, P]
    L.orc_random_actions.argtypes = [P, P, C.c_uint64]
    L.orc_get_contacts.argtypes = [P, C.c_int32] + [P] * 8
    if hasattr(L, "orc_ref_detect"):  # reference builds only
        L.orc_ref_detect.argtypes = [P, C.c_int32] + [P] * 5
        L.orc_ref_detect.restype = C.c_int32
        L.orc_ref_save_snapshot.argtypes = [P, P, C.c_int64]
        L.orc_ref_save_snapshot.restype = C.c_int64
        L.orc_ref_load_snapshot.argtypes = [P, P, C.c_int64]
        L.orc_ref_load_snapshot.restype = C.c_int32
    L.orc_get_report.argtypes = [P, P, P, P]
    L.orc_get_task_state.argtypes = [P, P, P, P]
    L.orc_set_task_state.argtypes = [P, P, P, P]
    L.orc_first_system.argtypes = [P, C.c_int, P, P, P]
    L.orc_terrain_height.restype = C.c_double
    L.orc_terrain_height.argtypes = [P, C.c_int32, C.c_double, C.c_double]
    if hasattr(L, "orc_ref_first_system"):
        L.orc_ref_first_system.argtypes = [P, C.c_int, P, P, P]
    _cache[kind] = L
    return L


def _p(a):
    return C.c_void_p(0) if a is None else C.c_void_p(a.ctypes.data)


class OracleEnv:
    """CPU oracle with the VecEnv method names (host numpy arrays, double)."""

    def __init__(self, model, task, cfg, n_envs: int, seed: int = 1234, env_offset: int = 0, nthreads: int = 1,
                 kind: str = "restatement", precision: str = "f64", terrain=None):
        self.kind = kind
        self.L = _lib(kind)
        self.model, self.task, self.cfg = model, task, cfg
        self.n_envs = n_envs
        self.n_bodies = model.n_bodies
        self.action_dim = model.n_joints
        use_ref = 1 if kind.startswith("reference") else 0
        h = self.L.orc_create(C.byref(model), C.byref(task), C.byref(cfg), n_envs, C.c_uint64(seed),
                              C.c_int64(env_offset), nthreads, 0 if precision == "f32" else 1, use_ref)
        if not h:
            raise RuntimeError(f"orc_create failed: {self.L.orc_last_error().decode()}")
        self.h = C.c_void_p(h)
        self.obs_dim = int(self.L.orc_obs_dim(self.h))
        if terrain:
            self.set_terrain(terrain)

    def close(self):
        if self.h:
            self.L.orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def backend(self) -> str:
        return self.L.orc_backend(self.h).decode()

    def set_terrain(self, boxes):
        from paper_1810_05762_b200 import abi
        arr = (abi.StaticBox * max(1, len(boxes)))()
        for i, b in enumerate(boxes):
            arr[i] = b
        self.L.orc_set_terrain(self.h, C.cast(arr, C.c_void_p), len(boxes))

    def reset(self, mask=None):
        obs = np.zeros((self.n_envs, self.obs_dim))
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.L.orc_reset(self.h, _p(m), _p(obs))
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(actions, np.float64)
        obs = np.zeros((self.n_envs, self.obs_dim))
        rew = np.zeros(self.n_envs)
        done = np.zeros(self.n_envs, np.uint8)
        rc = self.L.orc_step(self.h, _p(a), _p(obs), _p(rew), _p(done))
        if rc:
            raise RuntimeError(self.L.orc_last_error().decode())
        return obs, rew, done

    def observe(self):
        obs = np.zeros((self.n_envs, self.obs_dim))
        self.L.orc_observe(self.h, _p(obs))
        return obs

    def physics_step(self, torques):
        t = np.ascontiguousarray(torques, np.float64)
        rc = self.L.orc_physics_step(self.h, _p(t))
        if rc:
            raise RuntimeError(self.L.orc_last_error().decode())

    def random_actions(self, step: int):
        a = np.zeros((self.n_envs, self.action_dim))
        self.L.orc_random_actions(self.h, _p(a), step)
        return a

    def get_state(self):
        s = np.zeros((self.n_envs, self.n_bodies, 13))
        self.L.orc_get_state(self.h, _p(s))
        return s

    def set_state(self, s):
        s = np.ascontiguousarray(s, np.float64)
        self.L.orc_set_state(self.h, _p(s))

    def set_external_loads(self, loads):
        l = np.ascontiguousarray(loads, np.float64)
        self.L.orc_set_external_loads(self.h, _p(l))

    def contact_arrays(self, capacity: int = 256):
        N = self.n_envs
        out = dict(count=np.zeros(N, np.int32), body_a=np.full((N, capacity), -1, np.int32),
                   body_b=np.full((N, capacity), -1, np.int32), point=np.zeros((N, capacity, 3)),
                   normal=np.zeros((N, capacity, 3)), separation=np.zeros((N, capacity)),
                   normal_impulse=np.zeros((N, capacity)), tangential_impulse=np.zeros((N, capacity, 3)))
        self.L.orc_get_contacts(self.h, capacity, _p(out["count"]), _p(out["body_a"]), _p(out["body_b"]),
                                _p(out["point"]), _p(out["normal"]), _p(out["separation"]),
                                _p(out["normal_impulse"]), _p(out["tangential_impulse"]))
        return out

    def ref_detect_contacts(self, capacity: int = 1 << 16):
        """The compiled reference's detect_contacts with inter_agent_collisions
        on, for the current state: every contact (global body indices), the
        reference's order.  Reference builds only."""
        if not hasattr(self.L, "orc_ref_detect"):
            raise RuntimeError("ref_detect_contacts needs the compiled reference (kind='reference')")
        out = dict(body_a=np.zeros(capacity, np.int32), body_b=np.zeros(capacity, np.int32),
                   point=np.zeros((capacity, 3)), normal=np.zeros((capacity, 3)), separation=np.zeros(capacity))
        n = self.L.orc_ref_detect(self.h, capacity, _p(out["body_a"]), _p(out["body_b"]), _p(out["point"]),
                                  _p(out["normal"]), _p(out["separation"]))
        k = min(n, capacity)
        return {key: v[:k] for key, v in out.items()}

    def ref_save_snapshot(self) -> bytes:
        """Scene::save_snapshot of the compiled reference for the current state."""
        n = self.L.orc_ref_save_snapshot(self.h, None, 0)
        buf = np.zeros(n, np.uint8)
        self.L.orc_ref_save_snapshot(self.h, _p(buf), n)
        return buf.tobytes()

    def ref_load_snapshot(self, data: bytes):
        buf = np.frombuffer(data, np.uint8).copy()
        if self.L.orc_ref_load_snapshot(self.h, _p(buf), buf.size) != 0:
            raise RuntimeError(self.L.orc_last_error().decode())

    def report(self):
        N = self.n_envs
        newton, krylov, failed = np.zeros(N, np.int32), np.zeros(N, np.int32), np.zeros(N, np.uint8)
        self.L.orc_get_report(self.h, _p(newton), _p(krylov), _p(failed))
        return dict(newton_iterations=newton, krylov_iterations=krylov, failed=failed)

    def task_state(self):
        N, J = self.n_envs, self.action_dim
        target, counters, last = np.zeros((N, 2)), np.zeros((N, 8), np.int32), np.zeros((N, max(J, 1)))
        self.L.orc_get_task_state(self.h, _p(target), _p(counters), _p(last))
        return dict(target=target, counters=counters, last_tau=last[:, :J])

    def set_task_state(self, target=None, counters=None, last_tau=None):
        t = None if target is None else np.ascontiguousarray(target, np.float64)
        c = None if counters is None else np.ascontiguousarray(counters, np.int32)
        l = None if last_tau is None else np.ascontiguousarray(last_tau, np.float64)
        self.L.orc_set_task_state(self.h, _p(t), _p(c), _p(l))

    def first_system(self, env: int, torques, reference: bool = False):
        B = self.n_bodies
        n = 6 * B
        H, rhs = np.zeros((n, n)), np.zeros(n)
        t = np.ascontiguousarray(torques, np.float64)
        fn = self.L.orc_ref_first_system if reference else self.L.orc_first_system
        nc = fn(self.h, env, _p(t), _p(H), _p(rhs))
        return H, rhs, nc
