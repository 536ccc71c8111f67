"""Inter-agent contact detection on the GPU against the
reference: the KATs of test_physics.cpp:137-178 (flag semantics, separation of
two overlapping sphere agents, random sphere clouds vs brute force) and crowded
HFH humanoids against the compiled reference's detect_contacts with
inter_agent_collisions on (oracle/_ref, `orc_ref_detect`).

Tolerance: f64 — pair list identical, point / normal / separation within
1e-9; f32 (positions kept relative to per-env origins) — pair list identical
except pairs within 1e-4 m of the margin (counted), separation within 1e-5,
contact point within 1e-4 (closest points of near-parallel segments are
ill-conditioned: fp32 input rounding moves them more than the distance)."""
import numpy as np
import pytest

import oracle
import scenes as S
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import VecEnv

pytestmark = pytest.mark.gpu


def _pairs(d):
    return list(zip(d["body_a"].tolist(), d["body_b"].tolist()))


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_two_sphere_agents(precision):
    """test_physics.cpp:137-149: two agents' spheres 0.6 m apart (r = 0.5):
    exactly one pair, separation -0.4."""
    cfg = abi.default_step_config()
    cfg.contact_margin = 0.0
    sc = S.sphere_scene(5.0)
    g = VecEnv(model=sc.build(), task_config=S.quiet_task(), step_config=cfg, n_envs=2, precision=precision)
    st = np.stack([sc.state(), sc.state()])
    st[1, 0, 0] += 0.6
    g.set_state(st)
    d = g.detect_inter_agent()
    assert _pairs(d) == [(0, 1)]
    assert abs(d["separation"][0] + 0.4) <= (1e-12 if precision == "f64" else 1e-6)
    assert abs(abs(d["normal"][0, 0]) - 1.0) <= 1e-9
    # far apart: nothing
    st[1, 0, 0] += 10.0
    g.set_state(st)
    assert g.detect_inter_agent()["body_a"].size == 0


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_sphere_clouds_match_brute_force(precision):
    """test_physics.cpp:161-178: 5 clouds of 12 single-sphere agents (r = 0.3,
    margin 0.05): the pair set equals the brute-force overlap oracle."""
    rng = np.random.default_rng(99)
    cfg = abi.default_step_config()
    cfg.contact_margin = 0.05
    sc = S.sphere_scene(5.0, radius=0.3)
    g = VecEnv(model=sc.build(), task_config=S.quiet_task(), step_config=cfg, n_envs=12, precision=precision)
    for _ in range(5):
        pos = np.column_stack([rng.uniform(-1, 1, 12), rng.uniform(-1, 1, 12), rng.uniform(4, 6, 12)])
        st = np.repeat(sc.state()[None], 12, axis=0)
        st[:, 0, :3] = pos
        g.set_state(st)
        want = []
        for i in range(12):
            for j in range(i + 1, 12):
                if np.all(np.abs(pos[i] - pos[j]) <= 0.6 + 0.05) and np.linalg.norm(pos[i] - pos[j]) - 0.6 < 0.05:
                    want.append((i, j))
        assert _pairs(g.detect_inter_agent()) == want


@pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference (oracle/_ref) not built")
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_crowded_humanoids_match_reference(precision):
    """HFH humanoids on a grid compressed from 2 m to 0.2 m x 0.3 m spacing (and a few
    steps of motion): the GPU pair list equals the reference's inter-agent
    contacts (detect_contacts, collide.cpp:300-343) pair for pair."""
    n = 128
    g = VecEnv("hfh", n_envs=n, precision=precision, seed=21)
    o = oracle.OracleEnv(g.model, g.task, g.cfg, n, seed=21, kind="reference")
    base = o.get_state()
    tm = np.array([g.model.joints[j].max_torque for j in range(g.action_dim)])
    total = 0
    flips = 0
    for t in range(4):
        if t == 0:
            st = base.copy()
            for e in range(n):
                st[e, :, 0] -= (e % 64) * 1.8
                st[e, :, 1] -= (e // 64) * 1.7
            o.set_state(st)
        else:
            o.physics_step(o.random_actions(t) * tm)
        s = o.get_state()
        g.set_state(s)
        ref = o.ref_detect_contacts()
        inter = ref["body_b"] >= 0
        rp = list(zip(ref["body_a"][inter].tolist(), ref["body_b"][inter].tolist()))
        d = g.detect_inter_agent()
        gp = _pairs(d)
        total += len(rp)
        if precision == "f64":
            assert gp == rp
            for key in ("point", "normal", "separation"):
                assert np.abs(d[key] - ref[key][inter]).max(initial=0.0) <= 1e-9
        else:
            common = sorted(set(gp) & set(rp))
            for p in set(gp) ^ set(rp):  # only boundary cases may flip in fp32
                src = ref if p in set(rp) else d
                k = list(zip(src["body_a"].tolist(), src["body_b"].tolist())).index(p)
                assert abs(src["separation"][k] - g.cfg.contact_margin) <= 1e-4
                flips += 1
            gi = {p: i for i, p in enumerate(gp)}
            for p in common:
                i, j = gi[p], rp.index(p)
                jj = np.flatnonzero(inter)[j]
                assert np.abs(d["point"][i] - ref["point"][jj]).max() <= 1e-4
                assert abs(d["separation"][i] - ref["separation"][jj]) <= 1e-5
    print(f"{precision}: {total} reference inter-agent contacts over 4 states, {flips} boundary flips")
    assert total > 50  # the crowd actually touches


@pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference (oracle/_ref) not built")
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_contact_merged_islands_match_reference(precision):
    """HFH with inter-agent collisions: agents overlapping in
    pairs and one triple form contact-merged islands that the island launch
    solves as one system each (solver.cpp:458-502).  Teacher-forced one-step
    states against the compiled reference: f64 |dx| <= 1e-7 m, rel|dv| <= 1e-4;
    f32 the SURVEY §8(c) bounds (|dx| p99 <= 1e-4, max <= 5e-3)."""
    n = 9
    g = VecEnv("hfh", n_envs=n, precision=precision, seed=31)
    assert g.task.inter_agent_collisions == 1
    o = oracle.OracleEnv(g.model, g.task, g.cfg, n, seed=31, kind="reference")
    st = o.get_state()
    for e, dx in ((1, 1.7), (3, 1.7), (5, 1.7), (7, 1.7), (8, 3.4)):  # islands {0,1} {2,3} {4,5} {6,7,8}
        st[e, :, 0] -= dx
    o.set_state(st)
    tm = np.array([g.model.joints[j].max_torque for j in range(g.action_dim)])
    dxs, dvs = [], []
    pairs = 0
    for t in range(6):
        s = o.get_state()
        g.set_state(s)
        pairs += g.detect_inter_agent()["body_a"].size
        tq = o.random_actions(t) * tm
        o.physics_step(tq)
        g.physics_step(tq)
        so, sg = o.get_state(), g.get_state()
        if precision == "f64":  # the ordered contact lists, inter-agent contacts included
            co, cg = o.contact_arrays(g.contact_capacity), g.contact_arrays()
            np.testing.assert_array_equal(co["count"], cg["count"])
            for e in range(n):
                c = co["count"][e]
                np.testing.assert_array_equal(co["body_a"][e, :c], cg["body_a"][e, :c])
                np.testing.assert_array_equal(co["body_b"][e, :c], cg["body_b"][e, :c])
                assert np.abs(co["point"][e, :c] - cg["point"][e, :c]).max(initial=0.0) <= 1e-7
                assert np.abs(co["separation"][e, :c] - cg["separation"][e, :c]).max(initial=0.0) <= 1e-9
                pn = co["normal_impulse"][e, :c]
                assert np.abs(pn - cg["normal_impulse"][e, :c]).max(initial=0.0) <= 1e-5 * max(1.0, np.abs(pn).max(initial=0.0))
        dxs.append(np.abs(so[..., 0:3] - sg[..., 0:3]).max(axis=(1, 2)))
        dvs.append(np.abs(so[..., 7:13] - sg[..., 7:13]).max(axis=(1, 2)) / np.maximum(1, np.abs(so[..., 7:13]).max(axis=(1, 2))))
        assert g.report()["overflow"].sum() == 0
    dx, dv = np.concatenate(dxs), np.concatenate(dvs)
    print(f"{precision}: {pairs} inter-agent contacts over 6 states; |dx| max {dx.max():.2e} p99 "
          f"{np.quantile(dx, 0.99):.2e}; rel|dv| max {dv.max():.2e}")
    assert pairs > 6
    if precision == "f64":
        assert dx.max() <= 1e-7 and dv.max() <= 1e-4
    else:
        assert np.quantile(dx, 0.99) <= 1e-4 and dx.max() <= 5e-3


def _chains(o, n, chains):
    o.set_state(S.chain_state(o.get_state(), o.model, chains))


@pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference (oracle/_ref) not built")
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_big_islands_match_reference(precision):
    """Islands of any size (solver.cpp:458-502 has no cap): a 12-agent chain
    and a 5-agent chain (more envs than one island CTA holds: 8 in f32, 4 in
    f64) are solved by the multi-CTA island launch as one system each.
    Teacher-forced against the compiled reference: f64 |dx| <= 1e-7 m with
    identical ordered contact lists, f32 the SURVEY §8(c) bounds; no env
    reports an overflow."""
    n = 24
    g = VecEnv("hfh", n_envs=n, precision=precision, seed=41)
    o = oracle.OracleEnv(g.model, g.task, g.cfg, n, seed=41, kind="reference")
    _chains(o, n, [(0, 12), (12, 5), (18, 2)])
    tm = np.array([g.model.joints[j].max_torque for j in range(g.action_dim)])
    dxs = []
    for t in range(5):
        s = o.get_state()
        g.set_state(s)
        if t == 0:  # the chains really are single islands: consecutive members touch
            d = g.detect_inter_agent()
            nb = g.n_bodies
            links = {(a // nb, b // nb) for a, b in zip(d["body_a"].tolist(), d["body_b"].tolist())}
            for start, length in [(0, 12), (12, 5)]:
                assert all((e, e + 1) in links for e in range(start, start + length - 1)), links
        tq = o.random_actions(t) * tm
        o.physics_step(tq)
        g.physics_step(tq)
        so, sg = o.get_state(), g.get_state()
        if precision == "f64":
            co, cg = o.contact_arrays(g.contact_capacity), g.contact_arrays()
            np.testing.assert_array_equal(co["count"], cg["count"])
            for e in range(n):
                c = co["count"][e]
                np.testing.assert_array_equal(co["body_a"][e, :c], cg["body_a"][e, :c])
                np.testing.assert_array_equal(co["body_b"][e, :c], cg["body_b"][e, :c])
        dxs.append(np.abs(so[..., :3] - sg[..., :3]).max(axis=(1, 2)))
        rep = g.report()
        assert rep["overflow"].sum() == 0 and rep["failed"].sum() == 0
    dx = np.concatenate(dxs)
    print(f"{precision}: |dx| max {dx.max():.2e} p99 {np.quantile(dx, 0.99):.2e}")
    if precision == "f64":
        assert dx.max() <= 1e-7
    else:
        assert np.quantile(dx, 0.99) <= 1e-4 and dx.max() <= 5e-3


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_island_over_launch_budget_is_flagged_and_stepped(precision):
    """An island whose CTA parts exceed the co-resident budget (lowered to 1
    here through STP_ISLAND_BUDGET) is not frozen: its envs step one by one
    without the cross contacts, report overflow, and env_step writes their
    obs / reward / done."""
    import os
    import subprocess
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
from paper_1810_05762_b200.sim import VecEnv
sys.path.insert(0, {os.path.join(ROOT, "tests")!r})
from scenes import chain_state
g = VecEnv("hfh", n_envs=24, precision="{precision}", seed=41)
st = chain_state(g.get_state(), g.model, [(0, 12)])
g.set_state(st)
a = torch.zeros((24, g.action_dim), device="cuda")
obs = torch.full((24, g.obs_dim), float("nan"), device="cuda")
rew = torch.full((24,), float("nan"), device="cuda")
done = torch.full((24,), 7, dtype=torch.uint8, device="cuda")
g.step(a, obs, rew, done)
torch.cuda.synchronize()
rep = g.report()
assert rep["overflow"][:12].all() and not rep["overflow"][12:].any(), rep["overflow"]
assert torch.isfinite(obs).all() and torch.isfinite(rew).all() and (done <= 1).all()
assert not np.array_equal(g.get_state()[:12], st[:12])
print("ok")
"""
    env = dict(os.environ, STP_ISLAND_BUDGET="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_island_grid_hint_does_not_change_results(precision):
    """The persistent island grid is sized from the previous step's island
    count (a pinned host hint, sim_step.cuh launch_island).  A handle whose
    last step had no islands launches 8 island CTAs for 12 two-agent islands
    (some CTAs loop over two); a fresh handle launches 12.  Both must give
    bit-identical states, contact counts and reports, with no env flagged."""
    n = 24
    chains = [(2 * k, 2) for k in range(12)]
    g0 = VecEnv("hfh", n_envs=n, precision=precision, seed=41)
    o = oracle.OracleEnv(g0.model, g0.task, g0.cfg, n, seed=41)
    calm = o.get_state()
    crowded = S.chain_state(calm.copy(), g0.model, chains)
    tm = np.array([g0.model.joints[j].max_torque for j in range(g0.action_dim)])
    tq = o.random_actions(0) * tm
    fresh = VecEnv("hfh", n_envs=n, precision=precision, seed=41)
    stale = VecEnv("hfh", n_envs=n, precision=precision, seed=41)
    stale.set_state(calm)
    stale.physics_step(np.zeros_like(tq))  # no islands: the next grid is 2 * 0 + 8 CTAs
    assert stale.report()["overflow"].sum() == 0
    for h in (fresh, stale):
        h.set_state(crowded)
    dd = fresh.detect_inter_agent()
    nb = fresh.n_bodies
    links = {(a // nb, b // nb) for a, b in zip(dd["body_a"].tolist(), dd["body_b"].tolist())}
    assert all((s0, s0 + 1) in links for s0, _ in chains), "every pair must touch (12 islands)"
    for t in range(3):
        fresh.physics_step(tq * (0.5 + 0.25 * t))
        stale.physics_step(tq * (0.5 + 0.25 * t))
        np.testing.assert_array_equal(fresh.get_state(), stale.get_state())
        np.testing.assert_array_equal(fresh.contact_arrays()["count"], stale.contact_arrays()["count"])
        rf, rs = fresh.report(), stale.report()
        assert rf["overflow"].sum() == 0 and rs["overflow"].sum() == 0
        np.testing.assert_array_equal(rf["failed"], rs["failed"])
