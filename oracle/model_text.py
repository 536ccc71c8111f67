"""ORACLE — TEST INFRASTRUCTURE ONLY.  The oracle's own reader of the
"stampede-model 1" articulation documents (assets/*.model)
and its own copies of the reference defaults, so the CPU baseline and the
reference arm of bench.py never load the product library
(paper_1810_05762_b200/libstampede_b200.so).  Only the ctypes struct layouts
(paper_1810_05762_b200/abi.py, pure Python) are shared.

Defaults restated from the reference / SPEC:
  * StepConfig: types.hpp:92-107 (dt 1/120, 4 Newton iterations, Krylov 16 @
    1e-6, margin 0.02, Baumgarte 0.2, hardness 3000 / 300 / 6000, friction
    smoothing 1e-3, limit activation 0.05); gravity (0, 0, -9.8) scene.hpp:39.
  * TaskConfig: SPEC.md:240-243 and the DESIGN.md §5 decisions.
"""
from __future__ import annotations

import os

from paper_1810_05762_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
ASSETS = os.path.join(os.path.dirname(HERE), "assets")
SHAPES = {"sphere": abi.SPHERE, "capsule": abi.CAPSULE, "box": abi.BOX}


def parse_model(text: str) -> abi.Model:
    m = abi.Model()
    lines = [ln.split("#", 1)[0].split() for ln in text.splitlines()]
    lines = [ln for ln in lines if ln]
    if not lines or lines[0] != ["stampede-model", "1"]:
        raise ValueError("not a 'stampede-model 1' document")
    bodies, joints = {}, {}
    i = 1

    def nums(tok, n):
        if len(tok) != n:
            raise ValueError(f"expected {n} numbers, got {tok}")
        return [float(x) for x in tok]

    actuators, feet, root = {}, [], None
    while i < len(lines):
        key, *rest = lines[i]
        if key in ("body", "joint"):
            name, i = rest[0], i + 1
            fields = {}
            while lines[i][0] != "end":
                fields[lines[i][0]] = lines[i][1:]
                i += 1
            (bodies if key == "body" else joints)[name] = (len(bodies) if key == "body" else len(joints), fields)
        elif key == "name":
            m.name = rest[0].encode()
        elif key == "alive_bonus":
            m.alive_bonus = float(rest[0])
        elif key == "fall_height":
            m.fall_height = float(rest[0])
        elif key == "actuator":
            actuators[rest[0]] = float(rest[1])
        elif key == "foot":
            feet.append(rest[0])
        elif key == "root":
            root = rest[0]
        else:
            raise ValueError(f"unknown line '{key}'")
        i += 1
    m.n_bodies, m.n_joints = len(bodies), len(joints)
    for name, (k, f) in bodies.items():
        b = m.bodies[k]
        b.shape = SHAPES[f["shape"][0]]
        b.is_static = int(f["static"][0])
        b.radius = float(f["radius"][0])
        b.half_length = float(f["half_length"][0])
        b.half_extents[:] = nums(f["half_extents"], 3)
        b.local_pos[:] = nums(f["local_pos"], 3)
        b.local_rot[:] = nums(f["local_rot"], 4)
        b.mass = float(f["mass"][0])
        b.inertia_diag[:] = nums(f["inertia"], 3)
        m.rest_state[k][:] = nums(f["rest"], 13)
    for name, (k, f) in joints.items():
        j = m.joints[k]
        j.parent = bodies[f["parent"][0]][0]
        j.child = bodies[f["child"][0]][0]
        j.anchor_parent[:] = nums(f["anchor_parent"], 3)
        j.anchor_child[:] = nums(f["anchor_child"], 3)
        j.axis_parent[:] = nums(f["axis_parent"], 3)
        j.axis_child[:] = nums(f["axis_child"], 3)
        j.rest_relative[:] = nums(f["rest_relative"], 4)
        j.limit_lo, j.limit_hi = nums(f["limit"], 2)
        j.max_torque = actuators[name]
    m.n_feet = len(feet)
    for k, f in enumerate(feet):
        m.feet[k] = bodies[f][0]
    m.root = bodies[root][0]
    return m


def load_model(name: str) -> abi.Model:
    with open(os.path.join(ASSETS, f"{name}.model")) as f:
        return parse_model(f.read())


def default_step_config() -> abi.StepConfig:
    c = abi.StepConfig()
    c.dt = 1.0 / 120.0
    c.newton_iters, c.krylov_tol, c.krylov_max_iters = 4, 1e-6, 16
    c.contact_margin, c.baumgarte = 0.02, 0.2
    c.joint_hardness, c.contact_hardness, c.limit_hardness = 3000.0, 300.0, 6000.0
    c.friction_smoothing, c.limit_activation = 1e-3, 0.05
    c.gravity[:] = [0.0, 0.0, -9.8]
    c.has_ground_plane = 1
    c.reference_alias_quirk = 1
    return c


def default_task(kind: int) -> abi.Task:
    t = abi.Task()
    t.kind = kind
    t.episode_cap = 1000
    t.perturb_min, t.perturb_max = 200, 300
    t.perturb_force_lo, t.perturb_force_hi = 1.0, 5.0
    t.reset_noise = 0.05
    t.auto_reset = 1
    t.target_radius, t.target_tolerance = 100.0, 1.0
    hfh = kind in (abi.TASK_HFH, abi.TASK_HFH_TERRAIN)
    t.fall_grace = 160 if hfh else 0
    t.target_refresh = 200 if hfh else 0
    t.spacing = 2.0 if hfh else 3.0
    t.height_map = int(kind == abi.TASK_HFH_TERRAIN)
    t.inter_agent_collisions = int(hfh)
    return t


# --- generate_terrain, restated for the CPU arms ---------
M64 = 0xFFFFFFFFFFFFFFFF


def _mix64(z):  # splitmix64, rng.hpp:25-31
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _uniform(stream, k):  # 24-bit counter-based uniform (DESIGN.md §5 RNG)
    return (_mix64((stream + k) & M64) >> 40) * (1.0 / 16777216.0)


def generate_terrain(count, dim_lo, dim_hi, x_lo, x_hi, y_lo, y_hi, yaw_lo, yaw_hi, seed):
    """Static yaw boxes resting on z = 0: full edges U[dim_lo, dim_hi], centres
    uniform over the rectangle, yaw U[yaw_lo, yaw_hi); box i draws from
    derive_seed(seed, 5, i) (rng.hpp:35-37), the same draws as the device
    library's stp_generate_terrain."""
    out = []
    for i in range(count):
        s = _mix64(_mix64(_mix64(seed) ^ 5) ^ i)
        b = abi.StaticBox()
        for k in range(3):
            b.half_extents[k] = 0.5 * (dim_lo + (dim_hi - dim_lo) * _uniform(s, k))
        b.center[0] = x_lo + (x_hi - x_lo) * _uniform(s, 3)
        b.center[1] = y_lo + (y_hi - y_lo) * _uniform(s, 4)
        b.center[2] = b.half_extents[2]
        b.yaw = yaw_lo + (yaw_hi - yaw_lo) * _uniform(s, 5)
        out.append(b)
    return out
