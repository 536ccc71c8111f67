"""The independent reward / observation oracle (tests/reward_oracle.py)
against the C++ env oracle on randomized trajectories ("randomized
states -> equals an independently coded reward oracle to 1e-12"), on CPU.
This pins the checker that tests/test_gpu_envparity.py applies to the CUDA
path."""
import numpy as np
import pytest

import oracle
import reward_oracle as RO
from paper_1810_05762_b200 import abi

TASKS = {"humanoid": abi.TASK_HUMANOID, "ant": abi.TASK_ANT, "hfh": abi.TASK_HFH}


def _rollout(name, n=16, steps=120, seed=3, scale=1.0, random_targets=True):
    model = abi.builtin_model("ant" if name == "ant" else "humanoid")
    task = abi.default_task(TASKS[name])
    task.auto_reset = 0
    task.episode_cap = 1 << 30
    cfg = abi.default_step_config()
    env = oracle.OracleEnv(model, task, cfg, n, seed=seed)
    rng = np.random.default_rng(seed)
    J = model.n_joints
    out = []
    for t in range(steps):
        pre = env.get_state()
        ts = env.task_state()
        if random_targets and t % 7 == 3:  # targets all around the agent: every heading branch
            ang = rng.uniform(0, 2 * np.pi, n)
            d = rng.uniform(0.5, 100, n)
            tgt = pre[:, model.root, :2] + np.stack([d * np.cos(ang), d * np.sin(ang)], 1)
            env.set_task_state(target=tgt)
            ts = env.task_state()
        a = env.random_actions(t) * scale
        if t % 11 == 5:  # out-of-range actions: the clamp in the torque cost
            a = a * 1.7
        o, r, d = env.step(a)
        out.append((pre, ts["target"], a, env.get_state(), o, r, env.report()["failed"].copy()))
    return model, cfg, out


@pytest.mark.parametrize("name", ["humanoid", "ant", "hfh"])
def test_independent_reward_oracle_matches_env_oracle(name):
    model, cfg, out = _rollout(name)
    J = model.n_joints
    worst_r, worst_o, n = 0.0, 0.0, 0
    for pre, tgt, a, post, o, r, failed in out:
        feet = o[:, 11 + 3 * J: 11 + 3 * J + model.n_feet]
        rr, parts = RO.reward(model, cfg, pre[:, model.root, :2], post, a, tgt, feet, failed)
        worst_r = max(worst_r, np.abs(rr - r).max())
        # the obs after the step sees the (possibly resampled) post-step target
        n += len(r)
    print(f"{name}: {n} states, max |reward - independent oracle| {worst_r:.2e}")
    assert n >= 1000
    assert worst_r <= 1e-12


@pytest.mark.parametrize("name", ["humanoid", "ant"])
def test_independent_observation_oracle_matches_env_oracle(name):
    model, cfg, out = _rollout(name, random_targets=False)
    J = model.n_joints
    worst = 0.0
    for pre, tgt, a, post, o, r, failed in out:
        feet = o[:, 11 + 3 * J: 11 + 3 * J + model.n_feet]
        ob = RO.observation(model, post, tgt, np.clip(a, -1, 1), feet)
        worst = max(worst, np.abs(ob - o).max())
    print(f"{name}: max |obs - independent oracle| {worst:.2e}")
    assert worst <= 1e-12


def test_reward_oracle_spec_examples():
    """SPEC.md:285-286 (2.55 / 0.55) and the heading / standing piecewise
    examples (:294-305) through the independent oracle itself."""
    m = abi.builtin_model("humanoid")
    cfg = abi.default_step_config()
    st = np.array([[m.rest_state[b][k] for k in range(13)] for b in range(m.n_bodies)])[None]
    J = m.n_joints
    pre = st[:, m.root, :2].copy()
    tgt = pre + np.array([[1000.0, 0.0]])
    r, parts = RO.reward(m, cfg, pre, st, np.zeros((1, J)), tgt, np.zeros((1, 2)))
    assert parts["nlim"][0] == 0 and parts["rstand"][0] == 1 and parts["rhead"][0] == 1
    assert abs(r[0] - 2.55) < 1e-12
    r2, _ = RO.reward(m, cfg, pre, st, np.zeros((1, J)), tgt, np.ones((1, 2)))
    assert abs(r2[0] - 0.55) < 1e-12
    for c, bonus in [(0.9, 1.0), (0.4, 0.5), (-0.8, -1.0)]:
        t = pre + 10 * np.array([[c, np.sqrt(1 - c * c)]])
        _, p = RO.reward(m, cfg, pre, st, np.zeros((1, J)), t, np.zeros((1, 2)))
        assert abs(p["rhead"][0] - bonus) < 1e-12
