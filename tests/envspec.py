"""SPEC env-layer examples (App. B/C) written once
against the VecEnv / OracleEnv method names.  `make(task_name, n)` returns an
env; `tol` is the absolute tolerance on rewards / observations (1e-9 for the
double oracle, looser for the fp32 GPU path)."""
from __future__ import annotations

import math

import numpy as np

import scenes as S
from paper_1810_05762_b200 import abi

C_FRAME, C_FLAG, C_FALL, C_NEXTP, C_EPISODE, C_FLAGDRAW, C_PERTDRAW = range(7)


def rest_state(model, lift=0.0, yaw=0.0, tilt=0.0, origin=(0.0, 0.0)):
    """Bundled rest pose, rigidly rotated about the root (yaw about z, tilt
    about x), lifted and translated."""
    st = np.array([[model.rest_state[b][k] for k in range(13)] for b in range(model.n_bodies)])
    root = st[model.root, :3].copy()
    q = S.qmul(S.quat_axis_angle((0, 0, 1), yaw), S.quat_axis_angle((1, 0, 0), tilt))
    for b in range(model.n_bodies):
        st[b, :3] = root + S.qrot(q, st[b, :3] - root)
        st[b, 3:7] = S.qmul(q, st[b, 3:7])
    st[:, 2] += lift
    st[:, 0] += origin[0]
    st[:, 1] += origin[1]
    return st


def _quiet(env):
    """No perturbation in the next steps: push the trigger out of reach."""
    ts = env.task_state()
    c = ts["counters"].copy()
    c[:, C_NEXTP] = 1 << 30
    env.set_task_state(counters=c)


def obs_dims(make, tol=0.0):
    for task, dim in [("humanoid", 76), ("hfh", 76), ("ant", 39), ("hfh_terrain", 241)]:
        assert make(task, 2).obs_dim == dim


def reward_standing_examples(make, tol):
    """2.55 upright at rest facing the target with no feet
    contact; 0.55 with both feet on the ground."""
    env = make("humanoid", 1)
    m = env.model
    env.set_state(rest_state(m, lift=0.5)[None])
    env.set_task_state(target=np.array([[env.get_state()[0, m.root, 0] + 1000.0, env.get_state()[0, m.root, 1]]]))
    _quiet(env)
    _, r, d = env.step(np.zeros((1, env.action_dim)))
    assert d[0] == 0
    assert abs(r[0] - 2.55) <= tol
    env.set_state(rest_state(m, lift=0.0)[None])
    env.set_task_state(target=np.array([[env.get_state()[0, m.root, 0] + 1000.0, env.get_state()[0, m.root, 1]]]))
    _quiet(env)
    o, r, d = env.step(np.zeros((1, env.action_dim)))
    J = env.action_dim
    assert (o[0, 11 + 3 * J: 11 + 3 * J + 2] == 1).all()  # both feet flags set
    assert abs(r[0] - 0.55) <= max(tol, 0.02)  # settling adds a small speed term


def heading_bonus_examples(make, tol):
    """cos 0.9 -> 1, 0.4 -> 0.5, -0.8 -> -1 (x 0.5 in R)."""
    for c, bonus in [(0.9, 1.0), (0.4, 0.5), (-0.8, -1.0)]:
        env = make("humanoid", 1)
        m = env.model
        st = rest_state(m, lift=0.5, yaw=math.acos(c))
        env.set_state(st[None])
        env.set_task_state(target=np.array([[st[m.root, 0] + 1000.0, st[m.root, 1]]]))
        _quiet(env)
        _, r, _ = env.step(np.zeros((1, env.action_dim)))
        assert abs(r[0] - (2.0 + 0.5 * bonus + 0.05)) <= tol * 10


def standing_bonus_examples(make, tol):
    """cos(theta_vertical) 0.95 -> 1, 0.9 -> 0."""
    for c, bonus in [(0.95, 1.0), (0.9, 0.0)]:
        env = make("humanoid", 1)
        m = env.model
        st = rest_state(m, lift=0.8, tilt=math.acos(c))
        env.set_state(st[None])
        env.set_task_state(target=np.array([[st[m.root, 0] + 1000.0, st[m.root, 1]]]))
        _quiet(env)
        _, r, _ = env.step(np.zeros((1, env.action_dim)))
        # the tilt keeps the torso heading: cos(theta_target) = 1
        assert abs(r[0] - (2.0 + 0.5 + 0.05 * bonus)) <= tol * 10


def flagrun_examples(make, tol):
    """counter 199 unchanged, 200 resample, 0.5 m resample."""
    env = make("hfh", 1)
    m = env.model
    st = rest_state(m)
    root = st[m.root, :2]
    for stored, dist, expect_new in [(198, 50.0, False), (199, 50.0, True), (36, 0.5, True)]:
        env.set_state(st[None])
        c = env.task_state()["counters"].copy()
        c[:, C_FLAG] = stored
        c[:, C_NEXTP] = 1 << 30
        tgt = np.array([[root[0] + dist, root[1]]])
        env.set_task_state(target=tgt, counters=c)
        env.step(np.zeros((1, env.action_dim)))
        ts = env.task_state()
        new = np.abs(ts["target"] - tgt).max() > 1e-3
        assert new == expect_new
        if expect_new:
            assert ts["counters"][0, C_FLAG] == 0
            assert np.linalg.norm(ts["target"][0] - env.get_state()[0, m.root, :2]) <= 100.0 + 1e-3
        else:
            assert ts["counters"][0, C_FLAG] == stored + 1


def fall_grace_examples(make, tol):
    """SPEC.md:278 / PAPER.md:210: HFH below threshold for 159 frames -> not
    done, 160th consecutive frame -> done; Humanoid (grace 0) done at once."""
    for task, stored, expect in [("hfh", 158, 0), ("hfh", 159, 1), ("humanoid", 0, 1)]:
        env = make(task, 1)
        m = env.model
        st = rest_state(m, tilt=math.pi / 2, lift=-1.05)  # lying on the floor
        env.set_state(st[None])
        c = env.task_state()["counters"].copy()
        c[:, C_FALL] = stored
        c[:, C_NEXTP] = 1 << 30
        env.set_task_state(counters=c)
        _, _, d = env.step(np.zeros((1, env.action_dim)))
        assert d[0] == expect, (task, stored)


def flat_height_map(make, tol):
    """flat ground, agent at height h -> every entry = -h."""
    env = make("hfh_terrain", 2)
    o, _, _ = env.step(np.zeros((2, env.action_dim)))
    hm = o[:, -165:]
    assert np.abs(hm + o[:, :1]).max() <= tol


def episode_cap(make, tol):
    """episodes end at 1000 frames."""
    env = make("humanoid", 1)
    env.set_state(rest_state(env.model)[None])
    c = env.task_state()["counters"].copy()
    c[:, C_FRAME] = 998
    c[:, C_NEXTP] = 1 << 30
    env.set_task_state(counters=c)
    _, _, d = env.step(np.zeros((1, env.action_dim)))
    assert d[0] == 0
    _, _, d = env.step(np.zeros((1, env.action_dim)))
    assert d[0] == 1


def perturbation_schedule(make, tol):
    """next trigger in U{200..300}; a trigger pushes the root."""
    env = make("humanoid", 64)
    nxt = env.task_state()["counters"][:, C_NEXTP]
    assert ((nxt >= 200) & (nxt <= 300)).all()
    env1 = make("humanoid", 1)
    m = env1.model
    env1.set_state(rest_state(m, lift=0.5)[None])
    c = env1.task_state()["counters"].copy()
    c[:, C_FRAME] = 5
    c[:, C_NEXTP] = 5
    env1.set_task_state(counters=c)
    env1.step(np.zeros((1, env1.action_dim)))
    after = env1.task_state()["counters"][0]
    assert 205 <= after[C_NEXTP] <= 305 and after[C_PERTDRAW] == c[0, C_PERTDRAW] + 1
    vxy = np.abs(env1.get_state()[0, m.root, 7:9]).max()
    assert vxy > 1e-4  # 1-5 N for one frame on a 40 kg articulation


ALL = [obs_dims, reward_standing_examples, heading_bonus_examples, standing_bonus_examples, flagrun_examples,
       fall_grace_examples, flat_height_map, episode_cap, perturbation_schedule]
