"""Test scenes restated from the reference's own fixtures
(/root/reference/proj/tests/test_physics.cpp:27-120) as stp_model structs,
so the same known-answer tests run on the oracle and on the GPU path."""
from __future__ import annotations

import math

import numpy as np

from paper_1810_05762_b200 import abi


def quat_axis_angle(axis, angle):
    a = np.asarray(axis, float)
    a = a / np.linalg.norm(a)
    s = math.sin(0.5 * angle)
    return np.array([math.cos(0.5 * angle), a[0] * s, a[1] * s, a[2] * s])


def qmul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def qconj(q):
    return np.array([q[0], -q[1], -q[2], -q[3]])


def qrot(q, v):
    u = np.array(q[1:])
    t = 2.0 * np.cross(u, v)
    return np.asarray(v) + q[0] * t + np.cross(u, t)


class SceneBuilder:
    """add_body / sphere / capsule / box of test_physics.cpp:27-55."""

    def __init__(self, name="scene"):
        self.m = abi.Model()
        self.m.name = name.encode()[:31]
        self.m.fall_height = -1e9
        self.m.alive_bonus = 0.0

    def add_body(self, pos, rot=(1, 0, 0, 0), mass=1.0, inertia=(1, 1, 1), shape=None, is_static=False):
        b = self.m.n_bodies
        d = self.m.bodies[b]
        kind, radius, hl, half = shape
        d.shape = kind
        d.radius = radius
        d.half_length = hl
        for k in range(3):
            d.half_extents[k] = half[k]
            d.inertia_diag[k] = inertia[k]
        d.local_rot[0] = 1.0
        d.mass = mass
        d.is_static = 1 if is_static else 0
        st = self.m.rest_state[b]
        for k in range(3):
            st[k] = pos[k]
        for k in range(4):
            st[3 + k] = rot[k]
        self.m.n_bodies += 1
        return b

    def add_joint(self, parent, child, anchor_parent, anchor_child, axis_parent=(0, 0, 1), axis_child=(0, 0, 1),
                  rest=(1, 0, 0, 0), lo=-3.1, hi=3.1, max_torque=1.0):
        j = self.m.n_joints
        d = self.m.joints[j]
        d.parent, d.child = parent, child
        for k in range(3):
            d.anchor_parent[k] = anchor_parent[k]
            d.anchor_child[k] = anchor_child[k]
            d.axis_parent[k] = axis_parent[k]
            d.axis_child[k] = axis_child[k]
        for k in range(4):
            d.rest_relative[k] = rest[k]
        d.limit_lo, d.limit_hi, d.max_torque = lo, hi, max_torque
        self.m.n_joints += 1
        return j

    def build(self, root=None):
        self.m.root = root if root is not None else next(
            b for b in range(self.m.n_bodies) if not self.m.bodies[b].is_static)
        return self.m

    def state(self):
        return np.array([[self.m.rest_state[b][k] for k in range(13)] for b in range(self.m.n_bodies)])


def sphere(r):
    return (abi.SPHERE, r, 0.0, (0, 0, 0))


def capsule(r, hl):
    return (abi.CAPSULE, r, hl, (0, 0, 0))


def box(half):
    return (abi.BOX, 0.1, 0.0, half)


def sphere_scene(height, radius=0.5):
    """test_physics.cpp:58-63"""
    s = SceneBuilder("sphere")
    s.add_body((0, 0, height), mass=1.0, inertia=(0.1, 0.1, 0.1), shape=sphere(radius))
    return s


def box_scene():
    """test_physics.cpp:202-217: unit box resting on the ground"""
    s = SceneBuilder("box")
    s.add_body((0, 0, 0.5), mass=1.0, inertia=(1 / 6, 1 / 6, 1 / 6), shape=box((0.5, 0.5, 0.5)))
    return s


PEND_COM = 0.25
PEND_I = 1.0 * 0.5 * 0.5 / 12.0


def pendulum(lo=-3.0, hi=3.0):
    """make_pendulum, test_physics.cpp:67-96 (static base + rod on a y hinge)."""
    s = SceneBuilder("pendulum")
    base = s.add_body((0, 0, 1), mass=1.0, inertia=(1, 1, 1), shape=sphere(0.01), is_static=True)
    rod_rot = quat_axis_angle((0, 1, 0), math.pi / 2)
    rod = s.add_body((PEND_COM, 0, 1), rod_rot, 1.0, (PEND_I, PEND_I, 1e-4), capsule(0.02, 0.25))
    s.add_joint(base, rod, (0, 0, 0), (0, 0, -0.25), (0, 1, 0), (0, 1, 0), rod_rot, lo, hi, 100.0)
    return s


def chain(links=3):
    """test_physics.cpp:386-430: free swinging chain from a static base."""
    s = SceneBuilder("chain")
    base = s.add_body((0, 0, 3), mass=1, inertia=(1, 1, 1), shape=sphere(0.01), is_static=True)
    prev = base
    rot = quat_axis_angle((0, 1, 0), math.pi / 2)
    for i in range(links):
        b = s.add_body((0.25 + 0.5 * i, 0, 3), rot, 1.0, (0.02, 0.02, 1e-4), capsule(0.02, 0.24))
        ap = (0, 0, 0) if prev == base else (0, 0, 0.25)
        prev_rot = np.array(s.m.rest_state[prev][3:7])
        rest = qmul(qconj(prev_rot), rot)
        s.add_joint(prev, b, ap, (0, 0, -0.25), (0, 1, 0), (0, 1, 0), rest, -3.1, 3.1, 50.0)
        prev = b
    return s


def two_link(ox=0.0):
    """one agent of the batching test, test_physics.cpp:434-453"""
    s = SceneBuilder("two_link")
    rot = quat_axis_angle((0, 1, 0), math.pi / 2)
    a = s.add_body((ox, 0, 0.8), rot, 1.0, (0.02, 0.02, 1e-3), capsule(0.05, 0.2))
    b = s.add_body((ox + 0.5, 0, 0.8), rot, 0.7, (0.015, 0.015, 1e-3), capsule(0.04, 0.2))
    s.add_joint(a, b, (0, 0, 0.25), (0, 0, -0.25), (0, 1, 0), (0, 1, 0), (1, 0, 0, 0), -3.1, 3.1, 20.0)
    return s


def quiet_task(kind=abi.TASK_HUMANOID):
    t = abi.default_task(kind)
    t.reset_noise = 0.0
    t.perturb_min = 0
    t.perturb_max = 0
    t.auto_reset = 0
    return t


def tight_config(newton=2, kry=200):
    """test_physics.cpp:98-104"""
    c = abi.default_step_config()
    c.newton_iters = newton
    c.krylov_max_iters = kry
    c.krylov_tol = 1e-12
    return c


def no_plane(cfg):
    cfg.has_ground_plane = 0
    return cfg


def tile(state, n):
    return np.repeat(state[None], n, axis=0)


def chain_state(st, model, chains, dx=0.45):
    """Agents of each run [start, start + length) turned by 90 degrees about
    their roots and set side by side 0.45 m apart: neighbours touch hand to
    hand (<= 3 inter-agent contacts per body), one island per run."""
    q = quat_axis_angle((0, 0, 1), np.pi / 2)
    r = model.root
    for start, length in chains:
        x0, y0 = st[start, r, 0], st[start, r, 1]
        for k in range(length):
            e = start + k
            root = st[e, r, :3].copy()
            for b in range(model.n_bodies):
                st[e, b, :3] = root + qrot(q, st[e, b, :3] - root)
                st[e, b, 3:7] = qmul(q, st[e, b, 3:7])
                st[e, b, 7:10] = qrot(q, st[e, b, 7:10])
                st[e, b, 10:13] = qrot(q, st[e, b, 10:13])
            st[e, :, 0] += x0 + k * dx - st[e, r, 0]
            st[e, :, 1] += y0 - st[e, r, 1]
    return st
