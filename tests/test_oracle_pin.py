"""Pins the CPU restatement (oracle/phys_oracle.hpp + env layer) to the
reference: golden fixtures produced by the compiled, unmodified reference
(tests/golden/make_golden.py) and, when oracle/_ref is built, a direct
bit-for-bit comparison."""
import os

import numpy as np
import pytest

import oracle
from paper_1810_05762_b200 import abi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


TASK_OF = {"ant": abi.TASK_ANT, "humanoid": abi.TASK_HUMANOID, "hfh": abi.TASK_HFH}


def _env(name, kind="restatement", n=None, seed=None, precision="f64"):
    g = np.load(os.path.join(GOLDEN, f"golden_{name}.npz"))
    model = abi.builtin_model("ant" if name == "ant" else "humanoid")
    task = abi.default_task(TASK_OF[name])
    cfg = abi.default_step_config()
    env = oracle.OracleEnv(model, task, cfg, int(n or g["n"]), seed=int(seed or g["seed"]), kind=kind,
                           precision=precision)
    return env, g


@pytest.mark.parametrize("name", ["ant", "humanoid", "hfh"])
def test_restatement_replays_reference_golden(name):
    """Free-running replay of the reference's fixture (terminations,
    auto-resets, HFH fall grace and flagrun redraws) by the restatement."""
    env, g = _env(name)
    S = g["states"]
    for t in range(int(g["steps"])):
        np.testing.assert_array_equal(env.get_state(), S[t])
        o, r, d = env.step(g["actions"][t])
        np.testing.assert_array_equal(env.get_state(), S[t + 1])
        np.testing.assert_array_equal(r, g["reward"][t])
        np.testing.assert_array_equal(d, g["done"][t])
        np.testing.assert_array_equal(o.astype(np.float32), g["obs"][t])
        ts = env.task_state()
        if t + 1 < int(g["steps"]):
            np.testing.assert_array_equal(ts["target"], g["target"][t + 1])
            np.testing.assert_array_equal(ts["counters"], g["counters"][t + 1])
        c = env.contact_arrays(64)
        np.testing.assert_array_equal(c["count"], g["contact_count"][t])
        np.testing.assert_array_equal(c["body_a"].astype(np.int8), g["contact_body"][t])
        np.testing.assert_array_equal(c["separation"].astype(np.float32), g["contact_sep"][t])
    if name != "ant":
        assert g["done"].sum() > 0  # the fixture holds terminations


@pytest.mark.parametrize("name", ["ant", "humanoid"])
def test_restatement_bit_exact_vs_compiled_reference(name):
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    a, _ = _env(name, "restatement", n=32, seed=99)
    b, _ = _env(name, "reference", n=32, seed=99)
    for t in range(60):
        act = a.random_actions(t)
        oa, ra, da = a.step(act)
        ob, rb, db = b.step(act)
        np.testing.assert_array_equal(a.get_state(), b.get_state())
        np.testing.assert_array_equal(ra, rb)
        np.testing.assert_array_equal(da, db)
        np.testing.assert_array_equal(oa, ob)


def test_assembly_quirk_pattern():
    """Reference aliasing quirk (solver.cpp:350-351 + block_sparse.cpp:33-37):
    the Humanoid's assembled H is symmetric, the Ant's loses anchor row 0 of
    joint 3 in block (3, 4) only; the restatement reproduces the reference's
    matrix bit-for-bit either way."""
    for name, sym in [("humanoid", True), ("ant", False)]:
        env, _ = _env(name, n=1, seed=5)
        tq = np.zeros(env.action_dim)
        H, rhs, _ = env.first_system(0, tq)
        if oracle.available("reference"):
            ref, _ = _env(name, "reference", n=1, seed=5)
            Hr, rr, _ = ref.first_system(0, tq, reference=True)
            np.testing.assert_array_equal(H, Hr)
            np.testing.assert_array_equal(rhs, rr)
        asym = np.abs(H - H.T)
        blocks = {(i // 6, j // 6) for i, j in zip(*np.nonzero(asym > 1e-9 * np.abs(H).max()))}
        if sym:
            assert not blocks
        else:
            assert blocks == {(3, 4), (4, 3)}


def test_f32_restatement_envelope():
    """The fp32 instantiation of the reference algorithm stays within the
    SURVEY §8(c) one-step envelope of the double oracle (teacher-forced)."""
    d64, _ = _env("humanoid", n=16, seed=3)
    d32, _ = _env("humanoid", n=16, seed=3, precision="f32")
    tm = np.array([d64.model.joints[j].max_torque for j in range(d64.action_dim)])
    dx, dv = [], []
    for t in range(60):
        s = d64.get_state()
        d32.set_state(s)
        tq = d64.random_actions(t) * tm
        d64.physics_step(tq)
        d32.physics_step(tq)
        a, b = d64.get_state(), d32.get_state()
        dx.append(np.abs(a[..., :3] - b[..., :3]).max(axis=(1, 2)))
        dv.append(np.abs(a[..., 7:] - b[..., 7:]).max(axis=(1, 2)) / np.maximum(1, np.abs(a[..., 7:]).max(axis=(1, 2))))
    dx, dv = np.concatenate(dx), np.concatenate(dv)
    assert np.percentile(dx, 99) <= 1e-4 and dx.max() <= 5e-3
    assert np.median(dv) <= 2e-3 and np.percentile(dv, 99) <= 1e-1


@pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference not built")
def test_reference_inter_agent_hook_kat():
    """orc_ref_detect (the checker of the GPU inter-agent detection) reproduces
    test_physics.cpp:137-149 on the compiled reference: two single-sphere
    agents 0.6 m apart -> one inter-agent contact, separation -0.4."""
    import scenes as S
    cfg = abi.default_step_config()
    cfg.contact_margin = 0.0
    sc = S.sphere_scene(5.0)
    o = oracle.OracleEnv(sc.build(), S.quiet_task(), cfg, 2, kind="reference")
    st = np.stack([sc.state(), sc.state()])
    st[1, 0, 0] += 0.6
    o.set_state(st)
    c = o.ref_detect_contacts()
    assert list(zip(c["body_a"].tolist(), c["body_b"].tolist())) == [(0, 1)]
    assert abs(c["separation"][0] + 0.4) <= 1e-12


@pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference not built")
def test_reference_snapshot_hooks_round_trip():
    """orc_ref_save_snapshot / orc_ref_load_snapshot (the checkers of the GPU's
    SSNP format) round-trip through the compiled reference's Scene and reject
    a wrong body count with its message (scene.cpp:94-98)."""
    import scenes as S
    cfg = abi.default_step_config()
    sc = S.sphere_scene(3.0)
    o = oracle.OracleEnv(sc.build(), S.quiet_task(), cfg, 2, kind="reference")
    st = np.stack([sc.state(), sc.state()])
    st[1, 0, 2] = 7.0
    o.set_state(st)
    snap = o.ref_save_snapshot()
    assert snap[:4] == b"SSNP" and len(snap) == 16 + 2 * 13 * 8
    o2 = oracle.OracleEnv(sc.build(), S.quiet_task(), cfg, 2, kind="reference")
    o2.ref_load_snapshot(snap)
    np.testing.assert_array_equal(o2.get_state(), st)
    o1 = oracle.OracleEnv(sc.build(), S.quiet_task(), cfg, 1, kind="reference")
    with pytest.raises(RuntimeError, match="body count mismatch"):
        o1.ref_load_snapshot(snap)
