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
