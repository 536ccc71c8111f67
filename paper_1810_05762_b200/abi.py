"""ctypes mirror of include/stampede_sim.h (the C-ABI boundary).

The structures below must match the C header field for field; the
layout test (tests/test_abi.py) checks every sizeof against the compiled
library's own view (``stp_struct_sizes``).
"""
from __future__ import annotations

import ctypes as C
import os

MAX_BODIES = 32
MAX_JOINTS = 31
MAX_FEET = 4
STATE_STRIDE = 13

SPHERE, CAPSULE, BOX = 0, 1, 2
TASK_ANT, TASK_HUMANOID, TASK_HFH, TASK_HFH_TERRAIN = 0, 1, 2, 3
PRECISION_F32, PRECISION_F64 = 0, 1
STP_OK, STP_EINVAL, STP_ENOMEM, STP_ECUDA, STP_ESTATE = 0, 22, 12, 100, 101

D3 = C.c_double * 3
D4 = C.c_double * 4


class Body(C.Structure):
    _fields_ = [
        ("shape", C.c_int32),
        ("is_static", C.c_int32),
        ("radius", C.c_double),
        ("half_length", C.c_double),
        ("half_extents", D3),
        ("local_pos", D3),
        ("local_rot", D4),
        ("mass", C.c_double),
        ("inertia_diag", D3),
    ]


class Joint(C.Structure):
    _fields_ = [
        ("parent", C.c_int32),
        ("child", C.c_int32),
        ("anchor_parent", D3),
        ("anchor_child", D3),
        ("axis_parent", D3),
        ("axis_child", D3),
        ("rest_relative", D4),
        ("limit_lo", C.c_double),
        ("limit_hi", C.c_double),
        ("max_torque", C.c_double),
    ]


class Model(C.Structure):
    _fields_ = [
        ("name", C.c_char * 32),
        ("n_bodies", C.c_int32),
        ("n_joints", C.c_int32),
        ("root", C.c_int32),
        ("n_feet", C.c_int32),
        ("feet", C.c_int32 * MAX_FEET),
        ("bodies", Body * MAX_BODIES),
        ("joints", Joint * MAX_JOINTS),
        ("rest_state", (C.c_double * STATE_STRIDE) * MAX_BODIES),
        ("fall_height", C.c_double),
        ("alive_bonus", C.c_double),
    ]


class StepConfig(C.Structure):
    _fields_ = [
        ("dt", C.c_double),
        ("newton_iters", C.c_int32),
        ("krylov_tol", C.c_double),
        ("krylov_max_iters", C.c_int32),
        ("contact_margin", C.c_double),
        ("baumgarte", C.c_double),
        ("joint_hardness", C.c_double),
        ("contact_hardness", C.c_double),
        ("limit_hardness", C.c_double),
        ("friction_smoothing", C.c_double),
        ("limit_activation", C.c_double),
        ("gravity", D3),
        ("has_ground_plane", C.c_int32),
        ("reference_alias_quirk", C.c_int32),
    ]


class StaticBox(C.Structure):
    _fields_ = [("center", D3), ("half_extents", D3), ("yaw", C.c_double)]


class TerrainSpec(C.Structure):
    _fields_ = [
        ("count", C.c_int32),
        ("dim_lo", C.c_double),
        ("dim_hi", C.c_double),
        ("x_lo", C.c_double),
        ("x_hi", C.c_double),
        ("y_lo", C.c_double),
        ("y_hi", C.c_double),
        ("yaw_lo", C.c_double),
        ("yaw_hi", C.c_double),
        ("seed", C.c_uint64),
    ]


class Task(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("episode_cap", C.c_int32),
        ("fall_grace", C.c_int32),
        ("target_refresh", C.c_int32),
        ("target_radius", C.c_double),
        ("target_tolerance", C.c_double),
        ("spacing", C.c_double),
        ("perturb_min", C.c_int32),
        ("perturb_max", C.c_int32),
        ("perturb_force_lo", C.c_double),
        ("perturb_force_hi", C.c_double),
        ("reset_noise", C.c_double),
        ("auto_reset", C.c_int32),
        ("height_map", C.c_int32),
        ("inter_agent_collisions", C.c_int32),
    ]


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libstampede_b200.so")

_P = C.c_void_p
_I = C.c_int
_I32 = C.c_int32

# (name, restype, argtypes) for every symbol of include/stampede_sim.h
SIGNATURES = [
    ("stp_abi_version", _I, []),
    ("stp_last_error", C.c_char_p, []),
    ("stp_struct_sizes", None, [C.POINTER(C.c_int64)]),
    ("stp_default_step_config", None, [C.POINTER(StepConfig)]),
    ("stp_builtin_model", _I, [C.c_char_p, C.POINTER(Model)]),
    ("stp_validate_model", _I, [C.POINTER(Model)]),
    ("stp_model_from_text", _I, [C.c_char_p, C.POINTER(Model)]),
    ("stp_model_to_text", _I, [C.POINTER(Model), C.c_char_p, _I32, C.POINTER(_I32)]),
    ("stp_default_task", _I, [_I32, C.POINTER(Task)]),
    ("stp_generate_terrain", _I, [C.POINTER(TerrainSpec), C.POINTER(StaticBox), _I32]),
    ("stp_terrain_height", C.c_double, [C.POINTER(StaticBox), _I32, C.c_double, C.c_double]),
    ("stp_create", _P, [C.POINTER(Model), C.POINTER(Task), C.POINTER(StepConfig), _I32, _I32, C.c_uint64,
                        _I32, C.c_int64]),
    ("stp_destroy", None, [_P]),
    ("stp_set_terrain", _I, [_P, C.POINTER(StaticBox), _I32]),
    ("stp_num_envs", _I32, [_P]),
    ("stp_obs_dim", _I32, [_P]),
    ("stp_action_dim", _I32, [_P]),
    ("stp_contact_capacity", _I32, [_P]),
    ("stp_stream", _P, [_P]),
    ("stp_reset", _I, [_P, _P, _P, _P]),
    ("stp_step", _I, [_P, _P, _P, _P, _P, _P]),
    ("stp_step_host", _I, [_P, _P, _P, _P, _P]),
    ("stp_physics_step", _I, [_P, _P, _P]),
    ("stp_physics_step_host", _I, [_P, _P]),
    ("stp_random_actions", _I, [_P, _P, C.c_uint64, _P]),
    ("stp_set_state", _I, [_P, _P]),
    ("stp_get_state", _I, [_P, _P]),
    ("stp_set_external_loads", _I, [_P, _P]),
    ("stp_get_contacts", _I, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("stp_detect_inter_agent", _I, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    ("stp_snapshot_size", C.c_int64, [_P]),
    ("stp_save_snapshot", _I, [_P, _P, C.c_int64]),
    ("stp_load_snapshot", _I, [_P, _P, C.c_int64]),
    ("stp_get_report", _I, [_P, _P, _P, _P, _P]),
    ("stp_get_task_state", _I, [_P, _P, _P, _P]),
    ("stp_set_task_state", _I, [_P, _P, _P, _P]),
    ("stp_policy_forward", _I, [_P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_uint64, C.c_uint64,
                                C.c_int64, _P, _P, _P, _P, _P]),
    ("stp_gae", _I, [_P, _P, _P, _P, _I32, _I32, C.c_float, C.c_float, _P, _P, _P, _P]),
    ("stp_ppo_surrogate", _I, [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P, C.c_float, C.c_float, _P, _P, _P,
                               _P, _P, _P, _P, _P, _P]),
    ("stp_selu_backward_bias", _I, [_P, _P, C.c_int64, _I32, _P, _P, _P]),
    ("stp_bias_selu", _I, [_P, _P, C.c_int64, _I32, _I32, _P]),
    ("stp_ppo_kl", _I, [_P, _P, _P, _P, _I32, _I32, _P, _P, _P]),
    ("stp_debug_first_system", _I, [_P, _I32, _P, _P, _P, _P, _P]),
    ("stp_debug_math", _I, [_I32, _P, _P, _P, _P, C.c_int64, _P]),
]

_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Load the product library (fails loudly if it was not built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} is missing: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(p)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error(lib=None) -> str:
    lib = lib or load()
    msg = lib.stp_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "", lib=None) -> None:
    if rc != STP_OK:
        raise RuntimeError(f"{what} failed (status {rc}): {last_error(lib)}")


def model_from_text(text: str) -> Model:
    """load_model: parse a "stampede-model 1" document."""
    lib = load()
    m = Model()
    rc = lib.stp_model_from_text(text.encode(), C.byref(m))
    if rc != STP_OK:
        raise ValueError(last_error(lib))
    return m


def model_to_text(m: Model) -> str:
    lib = load()
    n = C.c_int32(0)
    check(lib.stp_model_to_text(C.byref(m), None, 0, C.byref(n)), "stp_model_to_text")
    buf = C.create_string_buffer(n.value + 1)
    check(lib.stp_model_to_text(C.byref(m), buf, n.value + 1, C.byref(n)), "stp_model_to_text")
    return buf.value.decode()


def builtin_model(name: str) -> Model:
    lib = load()
    m = Model()
    check(lib.stp_builtin_model(name.encode(), C.byref(m)), f"stp_builtin_model({name})")
    return m


def default_step_config() -> StepConfig:
    c = StepConfig()
    load().stp_default_step_config(C.byref(c))
    return c


def default_task(kind: int) -> Task:
    t = Task()
    check(load().stp_default_task(kind, C.byref(t)), "stp_default_task")
    return t
