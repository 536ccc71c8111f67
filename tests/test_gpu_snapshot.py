"""Scene snapshot "SSNP" v1 (scene.cpp:80-104): the
reference's round-trip KAT (test_physics.cpp:487-505), byte compatibility with
the compiled reference's Scene::save_snapshot, and a replay harness: a GPU
snapshot seeds the reference and both continue with the same torques."""
import numpy as np
import pytest

import oracle
import scenes as S
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import VecEnv

pytestmark = pytest.mark.gpu
need_ref = pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference not built")


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_snapshot_round_trip_kat(precision):
    """test_physics.cpp:487-505: save after 5 steps, load into a scene built
    elsewhere -> same state; a scene with another body count rejects it."""
    cfg = abi.default_step_config()
    sc = S.sphere_scene(3.0)
    g = VecEnv(model=sc.build(), task_config=S.quiet_task(), step_config=cfg, n_envs=1, precision=precision)
    g.set_state(sc.state()[None])
    for _ in range(5):
        g.physics_step(np.zeros((1, 0)))
    snap = g.save_snapshot()
    assert snap[:4] == b"SSNP" and len(snap) == 16 + 13 * 8
    r = VecEnv(model=S.sphere_scene(99.0).build(), task_config=S.quiet_task(), step_config=cfg, n_envs=1,
               precision=precision)
    r.load_snapshot(snap)
    np.testing.assert_array_equal(r.get_state(), g.get_state())
    two = VecEnv(model=sc.build(), task_config=S.quiet_task(), step_config=cfg, n_envs=2, precision=precision)
    with pytest.raises(ValueError, match="body count mismatch"):  # STP_EINVAL
        two.load_snapshot(snap)
    with pytest.raises(ValueError, match="bad magic"):
        r.load_snapshot(b"XXXX" + snap[4:])


@need_ref
def test_snapshot_bytes_match_reference():
    """The GPU's SSNP bytes of a state equal the reference's save_snapshot of it
    (f64 handle: the state round trip through the device is exact)."""
    n = 4
    g = VecEnv("humanoid", n_envs=n, precision="f64", seed=8)
    o = oracle.OracleEnv(g.model, g.task, g.cfg, n, seed=8, kind="reference")
    g.set_state(o.get_state())
    assert g.save_snapshot() == o.ref_save_snapshot()


@need_ref
@pytest.mark.parametrize("task", ["humanoid", "hfh"])
def test_replay_from_gpu_snapshot(task):
    """Replay harness: run the GPU (f64) for a few env steps, hand its snapshot
    to the compiled reference, then step both with the same torques: states
    agree to the f64 parity bound."""
    n = 8
    g = VecEnv(task, n_envs=n, precision="f64", seed=12)
    o = oracle.OracleEnv(g.model, g.task, g.cfg, n, seed=12, kind="reference")
    g.reset()
    import torch
    for t in range(5):
        g.step(g.random_actions(t))
    torch.cuda.synchronize()
    o.ref_load_snapshot(g.save_snapshot())
    np.testing.assert_array_equal(o.get_state(), g.get_state())
    tm = np.array([g.model.joints[j].max_torque for j in range(g.action_dim)])
    for t in range(3):
        tq = o.random_actions(100 + t) * tm
        o.physics_step(tq)
        g.physics_step(tq)
        assert np.abs(o.get_state()[..., :3] - g.get_state()[..., :3]).max() <= 1e-7
