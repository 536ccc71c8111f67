"""fp32 parity protocols for the env layer.

Shared by the GPU tests (tests/test_gpu_envparity.py, which assert the
bounds) and tools/parity_report.py (which writes profiles/r02_parity.json
for the current kernel build).  TEST INFRASTRUCTURE: the oracle is only the
checker here.

Protocols
---------
* ``reward_vs_independent_oracle`` — SPEC.md:287: the CUDA path's reward on
  >= 10^4 states against the independent numpy implementation of App. C
  (tests/reward_oracle.py) evaluated on the CUDA path's own pre / post
  states, actions, targets and feet flags.  Isolates the fp32 reward code
  (unit-vector heading, rsqrt, hinge angles) from physics error.
* ``teacher_forced_env`` — every step the double oracle's state and task
  state (target, counters, last torque) are loaded into the GPU handle (and
  into the fp32 restatement of the reference physics, the envelope); all
  three run one env_step with the same actions (auto-reset on the GPU; the
  oracles reset the same envs by mask, the same routine); obs / reward /
  done / next state are compared.  With ``source="gpu"`` the GPU runs its
  own trajectory and the oracle is teacher-forced from it (the bench
  config: 4096 envs, seed 1234).
Discrete decisions whose inputs sit within 1e-5 of a threshold (fall height,
standing bonus, joint-limit band, contact margin) are reported as
"boundary", never silently excluded.
"""
from __future__ import annotations

import os

import numpy as np

import oracle
import reward_oracle as RO
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import TASKS, VecEnv

BOUNDARY = 1e-5


def _q(a, p):
    return float(np.percentile(a, p)) if len(a) else 0.0


def summarize(a):
    a = np.asarray(a, np.float64).ravel()
    if a.size == 0:
        return {"n": 0}
    return {"n": int(a.size), "p50": _q(a, 50), "p99": _q(a, 99), "p999": _q(a, 99.9), "max": float(a.max())}


def obs_groups(J, n_feet, height_map):
    g = {"height": [0], "roll_pitch": [1, 2], "v_root": [3, 4, 5], "w_root": [6, 7, 8], "heading": [9, 10],
         "theta": list(range(11, 11 + J)), "theta_dot": list(range(11 + J, 11 + 2 * J)),
         "last_torque": list(range(11 + 2 * J, 11 + 3 * J)),
         "feet": list(range(11 + 3 * J, 11 + 3 * J + n_feet))}
    if height_map:
        k = 11 + 3 * J + n_feet
        g["height_map"] = list(range(k, k + 165))
    return g


# height-map samples: a difference above HM_JUMP (m) is a jump across a box
# edge; it is an explained edge flip when the GPU's sample is within HM_OWN of
# the double height map of the GPU's own state (counted, excluded from the
# height_map statistics, bounded by the tests)
HM_JUMP, HM_OWN = 0.05, 1e-3

# groups compared relative to max(1, |value|) (velocities: heavy-tailed)
RELATIVE = {"v_root", "w_root", "theta_dot"}

# Stated fp32 bounds of one teacher-forced env_step (Humanoid).
# Each quantity must ALSO be within 2x of the fp32 restatement of the
# reference algorithm on the same states (the intrinsic fp32 envelope,
# SURVEY §8(c)) where that envelope is measured.  (p99, max); velocities
# relative to max(1, |v|); angles in rad; reward is the continuous part
# (discrete flips of N_limits / standing counted separately); its max follows
# from the position bound, the speed term being a displacement / dt
# (5e-3 m / (1/120 s) = 0.6).  The tails (max) are absolute bounds; the
# envelope comparison applies to the bulk (p99).
BOUNDS = {
    "dx": (1e-4, 5e-3), "dv": (1e-1, None), "reward": (1e-3, 0.6),
    "height": (1e-5, 1e-3), "roll_pitch": (1e-4, 2e-2), "heading": (1e-4, 2e-2),
    "v_root": (1e-3, 0.5), "w_root": (1e-2, 1.0), "theta": (1e-3, 0.5), "theta_dot": (5e-2, None),
    "last_torque": (0.0, 0.0), "feet": (0.0, 0.0), "height_map": (1e-4, 1e-2),
}
# reset states / observations (same RNG draws, fp32 forward kinematics)
RESET_MAX = 1e-5
# independent reward oracle on the GPU's own states (fp32 reward arithmetic only)
REWARD_ORACLE = {"p99": 2e-5, "max": 1e-4}


def _task(name, **over):
    t = abi.default_task(TASKS[name])
    for k, v in over.items():
        setattr(t, k, v)
    return t


# ---------------------------------------------------------------------------
def reward_vs_independent_oracle(name="humanoid", n=4096, steps=4, warm=48, seed=1234, device=0):
    """GPU reward vs the independent App. C oracle on the GPU's own states."""
    task = _task(name, auto_reset=0, episode_cap=1 << 30)
    g = VecEnv(name, n_envs=n, seed=seed, task_config=task, device=device)
    m, cfg = g.model, g.cfg
    J, nf = g.action_dim, m.n_feet
    g.reset()
    for t in range(warm):  # a spread of upright, falling and lying states
        g.step(g.random_actions(t))
    rng = np.random.default_rng(seed)
    err, flips = [], 0
    n_states = 0
    rstand_counts = [0, 0]
    heading_branches = [0, 0]
    for t in range(steps):
        pre = g.get_state()
        ts = g.task_state()
        # targets in every direction (all heading branches), distances 0.5..100 m
        ang = rng.uniform(0, 2 * np.pi, n)
        dist = rng.uniform(0.5, 100.0, n)
        tgt = pre[:, m.root, :2] + np.stack([dist * np.cos(ang), dist * np.sin(ang)], 1)
        g.set_task_state(target=tgt)
        tgt = g.task_state()["target"]  # as the handle holds it
        a = rng.uniform(-1, 1, size=(n, J)).astype(np.float32)
        a[: n // 8] *= 1.6  # out-of-range actions: the torque-cost clamp
        o, r, d = g.step(a)
        post = g.get_state()
        failed = g.report()["failed"]
        feet = o[:, 11 + 3 * J: 11 + 3 * J + nf].astype(np.float64)
        rr, parts = RO.reward(m, cfg, pre[:, m.root, :2], post, a.astype(np.float64), tgt, feet, failed)
        e = np.abs(r.astype(np.float64) - rr)
        # a discrete term whose input is within BOUNDARY of its threshold may flip
        bnd = (parts["stand_margin"] < BOUNDARY) | (parts["limit_margin"] < BOUNDARY)
        flips += int(((e > 1e-2) & bnd).sum())
        err.append(np.where(bnd & (e > 1e-2), 0.0, e))
        n_states += n
        rstand_counts[0] += int((parts["rstand"] == 0).sum())
        rstand_counts[1] += int((parts["rstand"] == 1).sum())
        heading_branches[0] += int((parts["cth"] <= 0.8).sum())
        heading_branches[1] += int((parts["cth"] > 0.8).sum())
    g.close()
    e = np.concatenate(err)
    return {"task": name, "states": n_states, "abs_err": summarize(e), "boundary_flips": flips,
            "standing_0_1": rstand_counts, "heading_le_gt_0.8": heading_branches}


# ---------------------------------------------------------------------------
def _feet_cols(J, nf):
    return slice(11 + 3 * J, 11 + 3 * J + nf)


def teacher_forced_env(name="humanoid", n=32, steps=500, seed=7, scale=1.0, precision="f32", source="oracle",
                       envelope=True, oracle_kind="restatement", threads=None, warm=0, device=0, terrain=None):
    """Teacher-forced env_step protocol (see module docstring).  Returns a
    dict of statistics (percentiles + max) for the GPU and, with
    ``envelope``, for the fp32 restatement of the reference physics."""
    g = VecEnv(name, n_envs=n, precision=precision, seed=seed, device=device, terrain=terrain)
    m, cfg = g.model, g.cfg
    J, nf = g.action_dim, m.n_feet
    otask = _task(name, auto_reset=0)
    threads = threads or min(16, os.cpu_count() or 1)
    o = oracle.OracleEnv(m, otask, cfg, n, seed=seed, kind=oracle_kind, nthreads=threads, terrain=terrain)
    o32 = oracle.OracleEnv(m, otask, cfg, n, seed=seed, precision="f32", nthreads=threads,
                           terrain=terrain) if envelope else None
    groups = obs_groups(J, nf, bool(g.task.height_map))
    # height map: the terrain height is discontinuous at box edges, so a sample
    # within fp32 rounding of an edge can jump by a box height between the two
    # sides; a jump (> HM_JUMP) is counted as an edge flip when the GPU's value
    # equals the double height map of the GPU's own state (o_hm observes it)
    o_hm = oracle.OracleEnv(m, otask, cfg, n, seed=seed, nthreads=threads, terrain=terrain) \
        if "height_map" in groups else None
    hm_flips = 0
    thr = m.fall_height
    acc = {k: {"gpu": [], "f32": []} for k in ["dx", "dv", "reward"] + list(groups)}
    reset_err = []
    done_mism = {"gpu": 0, "f32": 0}
    done_boundary = {"gpu": 0, "f32": 0}
    feet_mism = {"gpu": 0, "f32": 0}
    flips = {"gpu": 0, "f32": 0}
    n_done = 0
    n_failed = {"gpu": 0, "oracle": 0}
    n_steps = 0
    if source == "gpu":
        g.reset()
        for t in range(warm):
            g.step(g.random_actions(t))
    for t in range(steps):
        if source == "gpu":
            pre = g.get_state()
            ts = g.task_state()
            o.set_state(pre)
            o.set_task_state(ts["target"], ts["counters"], ts["last_tau"])
        else:
            pre = o.get_state()
            ts = o.task_state()
            g.set_state(pre)
            g.set_task_state(ts["target"], ts["counters"], ts["last_tau"])
        if o32 is not None:
            o32.set_state(pre)
            o32.set_task_state(ts["target"], ts["counters"], ts["last_tau"])
        a = (o.random_actions(1000 + t) * scale).astype(np.float32)
        a64 = a.astype(np.float64)
        og, rg, dg = g.step(a)
        oo, ro, do = o.step(a64)
        post_o = o.get_state()
        n_failed["oracle"] += int(o.report()["failed"].sum())
        n_failed["gpu"] += int(g.report()["failed"].sum())
        h = post_o[:, m.root, 2]
        keep = do == 0
        if do.any():
            oo = o.reset(do)  # the auto-reset routine, by mask (same obs for the others)
        post_after = o.get_state()
        gs = g.get_state()
        n_done += int(do.sum())
        # GPU
        runs = [("gpu", og, rg, dg, gs)]
        if o32 is not None:
            o3, r3, d3 = o32.step(a64)
            s3 = o32.get_state()
            runs.append(("f32", o3, r3, d3, s3))
        for key, ob, rw, dn, st in runs:
            mis = dn != do
            bnd = np.abs(h - thr) < BOUNDARY
            done_mism[key] += int((mis & ~bnd).sum())
            done_boundary[key] += int((mis & bnd).sum())
            ok = keep & ~mis
            a_ = post_o[ok]
            b_ = st[ok]
            acc["dx"][key].append(np.abs(a_[..., :3] - b_[..., :3]).max(axis=(1, 2)))
            acc["dv"][key].append(np.abs(a_[..., 7:] - b_[..., 7:]).max(axis=(1, 2)) /
                                  np.maximum(1, np.abs(a_[..., 7:]).max(axis=(1, 2))))
            fm = np.abs(ob[:, _feet_cols(J, nf)] - oo[:, _feet_cols(J, nf)]).max(axis=1) > 0
            feet_mism[key] += int((fm & ok).sum())
            fine = ok & ~fm  # a flipped foot flag changes N_feet by 1 (counted above)
            # discrete reward terms (N_limits, standing bonus) decided on each
            # side's own state: a flip is explained by the state difference and
            # counted; the continuous remainder is what the bound applies to
            feet_o = oo[:, _feet_cols(J, nf)]
            _, pg = RO.reward(m, cfg, pre[:, m.root, :2], st, a64, ts["target"], feet_o)
            _, po = RO.reward(m, cfg, pre[:, m.root, :2], post_o, a64, ts["target"], feet_o)
            disc = -0.2 * (pg["nlim"] - po["nlim"]) + 0.05 * (pg["rstand"] - po["rstand"])
            flips[key] += int(((disc != 0) & fine).sum())
            acc["reward"][key].append(np.abs(rw.astype(np.float64) - ro - disc)[fine])
            for gname, cols in groups.items():
                d = np.abs(ob[:, cols].astype(np.float64) - oo[:, cols])
                if gname in RELATIVE:
                    d = d / np.maximum(1, np.abs(oo[:, cols]))
                if gname == "height_map" and key == "gpu" and (d > HM_JUMP).any():
                    o_hm.set_state(st)
                    own = np.abs(ob[:, cols].astype(np.float64) - o_hm.observe()[:, cols])
                    edge = (d > HM_JUMP) & (own <= HM_OWN)
                    hm_flips += int((edge & fine[:, None]).sum())
                    d = np.where(edge, 0.0, d)
                acc[gname][key].append(d.max(axis=1)[fine])
            if key == "gpu" and do.any():
                rs = do.astype(bool) & (dn == 1)
                if rs.any():
                    reset_err.append(np.abs(post_after[rs][..., :3] - st[rs][..., :3]).max(axis=(1, 2)))
                    reset_err.append(np.abs(ob[rs].astype(np.float64) - oo[rs]).max(axis=1))
        n_steps += 1
    g.close()
    o.close()
    if o32 is not None:
        o32.close()
    if o_hm is not None:
        o_hm.close()
    out = {"task": name, "precision": precision, "n_envs": n, "steps": n_steps, "torque_scale": scale,
           "source": source, "oracle": oracle_kind, "done_events": n_done, "failed": n_failed,
           "done_mismatch": done_mism, "done_boundary": done_boundary, "feet_flag_mismatch": feet_mism,
           "reward_discrete_flips": flips, "height_map_edge_flips": hm_flips,
           "reset_state_obs_err": summarize(np.concatenate(reset_err)) if reset_err else {"n": 0}}
    for k, v in acc.items():
        out[k] = {key: summarize(np.concatenate(v[key])) if v[key] else {"n": 0} for key in v}
    return out
