"""The reference's assemble_system / solve_krylov / clamp_torques known-answer
tests restated on the CUDA path:

* assemble_system (solver.hpp:41-44) through the step kernel's own first
  linearisation (stp_debug_first_system) against the compiled reference's
  assemble_system (oracle/_ref, orc_ref_first_system): block pattern
  (test_physics.cpp:258-301), symmetry on random scenes (:303-341), the
  reference's aliasing block (solver.cpp:350-351 + block_sparse.cpp:33-37).
* solve_krylov edge cases (test_linalg.cpp:118-198) as the fused step meets
  them: a block-diagonal (identity after the block-Jacobi split) system
  converges in one iteration, a zero right-hand side takes no iteration, a
  truncated solve (2 iterations at tol 1e-14) returns a finite iterate; the
  per-Newton Krylov counts equal the compiled reference's.
* clamp_torques (test_physics.cpp:180-191): |tau| > tau_max is clamped.
"""
import math

import numpy as np
import pytest

import oracle
import scenes as S
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import VecEnv

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not oracle.available("reference"), reason="compiled reference (oracle/_ref) not built")
TOL = {"f64": 1e-9, "f32": 2e-5}  # relative to max(1, |H|max)


def _make(model, cfg=None, task=None, n=1, precision="f64"):
    cfg = cfg or abi.default_step_config()
    task = task or S.quiet_task()
    return VecEnv(model=model, task_config=task, step_config=cfg, n_envs=n, precision=precision)


def _ref(model, cfg, state, task=None):
    o = oracle.OracleEnv(model, task or S.quiet_task(), cfg, len(state), kind="reference")
    o.set_state(state)
    return o


def _blocks_present(H, S_):
    return {(i, j) for i in range(S_) for j in range(S_) if np.abs(H[6 * i:6 * i + 6, 6 * j:6 * j + 6]).max() > 0}


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_one_hinge_couples_one_block_pair(precision):
    """test_physics.cpp:270-301: a static base contributes no slot; a
    two-dynamic-body hinge has exactly one off-diagonal block pair."""
    p = S.pendulum()
    g = _make(p.build(), S.tight_config(), precision=precision)
    g.set_state(p.state()[None])
    H, rhs, kry, ns = g.first_system(0, np.zeros((1, 1)))
    assert ns == 1 and H.shape == (6, 6)
    tl = S.two_link()
    cfg = S.no_plane(abi.default_step_config())
    g = _make(tl.build(), cfg, precision=precision)
    g.set_state(tl.state()[None])
    H, rhs, kry, ns = g.first_system(0, np.zeros((1, 1)))
    assert ns == 2
    assert _blocks_present(H, 2) == {(0, 0), (0, 1), (1, 0), (1, 1)}


def _random_chain(rng, k=4):
    """test_physics.cpp:303-330: k capsules at random poses / velocities,
    chained by y hinges whose rest_relative is the current relative rotation."""
    sb = S.SceneBuilder("randchain")
    quats = []
    for i in range(k):
        axis = rng.uniform(-1, 1, 3)
        q = S.quat_axis_angle(axis / np.linalg.norm(axis), rng.uniform(-1, 1))
        quats.append(q / np.linalg.norm(q))
        sb.add_body((rng.uniform(-1, 1) * 2, rng.uniform(-1, 1) * 2, 0.3 + 0.5 * i), quats[-1],
                    0.5 + abs(rng.uniform(-1, 1)), (0.1, 0.12, 0.08), S.capsule(0.1, 0.2))
    for i in range(k - 1):
        rest = S.qmul(S.qconj(quats[i]), quats[i + 1])
        sb.add_joint(i, i + 1, (0, 0, -0.3), (0, 0, 0.3), (0, 1, 0), (0, 1, 0), rest, -3.1, 3.1, 2.0)
    st = sb.state()
    st[:, 7:10] = rng.uniform(-1, 1, (k, 3))
    st[:, 10:13] = rng.uniform(-1, 1, (k, 3))
    return sb.build(root=0), st


@needs_ref
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_assembled_system_matches_reference_and_is_symmetric(precision):
    """test_physics.cpp:303-341 on the device path: random chains (contacts
    with the ground, torques 1): H equals the compiled reference's
    assemble_system and is symmetric."""
    rng = np.random.default_rng(31)
    cfg = abi.default_step_config()
    worst = 0.0
    for trial in range(5):
        m, st = _random_chain(rng)
        g = _make(m, cfg, precision=precision)
        g.set_state(st[None])
        s0 = g.get_state()
        tq = np.ones((1, m.n_joints))
        H, rhs, kry, ns = g.first_system(0, tq)
        np.testing.assert_array_equal(g.get_state(), s0)  # the hook leaves the state untouched
        o = _ref(m, cfg, st[None])
        Hr, rr, nc = o.first_system(0, tq[0], reference=True)
        scale = max(1.0, np.abs(Hr).max())
        err = max(np.abs(H - Hr).max(), np.abs(rhs - rr).max() / max(1.0, np.abs(rr).max() / scale)) / scale
        worst = max(worst, err)
        assert np.abs(H - H.T).max() <= TOL[precision] * scale
        np.testing.assert_array_equal(np.abs(H) > 0, np.abs(Hr) > 0)  # same block / entry pattern
    print(f"{precision}: max relative |H - H_ref| {worst:.2e}")
    assert worst <= TOL[precision]


@needs_ref
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_aliasing_quirk_block_matches_reference(precision):
    """The reference's block-pointer aliasing (solver.cpp:350-351 +
    block_sparse.cpp:33-37): in the 9-body Ant, creating block (3, 4) at a
    power-of-two block count reallocates the pool and the first anchor row's
    contribution to the other block of the pair is lost.  The device path's
    H is non-symmetric in exactly that block and equals the reference's."""
    m = abi.builtin_model("ant")
    cfg = abi.default_step_config()
    g = VecEnv("ant", n_envs=1, precision=precision, seed=3)
    st = g.get_state()
    tq = np.zeros((1, m.n_joints))
    H, rhs, kry, ns = g.first_system(0, tq)
    o = _ref(m, cfg, st, task=abi.default_task(abi.TASK_ANT))
    Hr, rr, _ = o.first_system(0, tq[0], reference=True)
    scale = max(1.0, np.abs(Hr).max())
    assert np.abs(H - Hr).max() <= TOL[precision] * scale
    asym = np.abs(Hr - Hr.T) > 1e-4 * scale
    assert asym.any()  # the quirk is live in the reference
    np.testing.assert_array_equal(np.abs(H - H.T) > 1e-4 * scale, asym)


def _floating_two_link(dt):
    """Two vertical capsules in the air on a y hinge, the joint exactly
    satisfied (anchors at z = 1.75 for both, identity orientations), both
    given v_z = 9.8 dt so that v_free = v + dt g = 0 exactly (dt a power of
    two, unit masses so m g / m = g exactly): every row bias and every rhs
    entry is zero."""
    sb = S.SceneBuilder("vertical_two_link")
    a = sb.add_body((0, 0, 2.0), (1, 0, 0, 0), 1.0, (0.02, 0.02, 1e-3), S.capsule(0.05, 0.2))
    b = sb.add_body((0, 0, 1.5), (1, 0, 0, 0), 1.0, (0.015, 0.015, 1e-3), S.capsule(0.04, 0.2))
    sb.add_joint(a, b, (0, 0, -0.25), (0, 0, 0.25), (0, 1, 0), (0, 1, 0), (1, 0, 0, 0), -3.1, 3.1, 20.0)
    st = sb.state()
    st[:, 9] = 9.8 * dt
    return sb.build(root=0), st


@needs_ref
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_zero_rhs_takes_no_krylov_iteration(precision):
    """test_linalg.cpp:129-137 in the step: b = 0 -> x = 0, no iteration."""
    cfg = S.no_plane(abi.default_step_config())
    cfg.dt = 1.0 / 128.0
    m, st = _floating_two_link(cfg.dt)
    g = _make(m, cfg, precision=precision)
    g.set_state(st[None])
    H, rhs, kry, ns = g.first_system(0, np.zeros((1, 1)))
    assert np.abs(rhs).max() == 0.0
    assert list(kry) == [0] * cfg.newton_iters
    o = _ref(m, cfg, st[None])
    o.physics_step(np.zeros((1, 1)))
    assert o.report()["krylov_iterations"][0] == 0
    g.physics_step(np.zeros((1, 1)))
    assert g.report()["krylov_iterations"][0] == 0
    s1 = g.get_state()
    assert np.abs(s1[0, :, 7:10]).max() == 0.0  # u = 0 exactly


@needs_ref
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_block_diagonal_system_converges_in_one_iteration(precision):
    """test_linalg.cpp:118-127 in the step: a single sphere pressed into the
    ground (contact rows only touch its own diagonal block): after the
    block-Jacobi split the system is the identity, so every Newton iteration's
    CR converges in one iteration — as in the compiled reference."""
    sc = S.sphere_scene(0.45)  # r = 0.5: 5 cm penetration
    m = sc.build()
    cfg = abi.default_step_config()
    g = _make(m, cfg, precision=precision)
    st = sc.state()[None]
    st[0, 0, 7:10] = (0.3, -0.2, -1.0)
    g.set_state(st)
    H, rhs, kry, ns = g.first_system(0, np.zeros((1, 0)))
    assert np.abs(rhs).max() > 0
    o = _ref(m, cfg, st)
    o.physics_step(np.zeros((1, 0)))
    g.physics_step(np.zeros((1, 0)))
    # Newton 1 starts from the pre-step velocities: one iteration; later ones
    # start from an iterate the identity system already solved (0 or 1)
    assert kry[0] == 1 and max(kry) == 1
    # StepReport.krylov_iterations is the scene total (types.hpp:115-120)
    assert int(g.report()["krylov_iterations"].sum()) == int(o.report()["krylov_iterations"][0]) == int(sum(kry))


@needs_ref
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_truncated_solve_returns_finite_iterate(precision):
    """test_linalg.cpp:186-198 in the step: Krylov capped at 2 iterations with
    tol 1e-14 on saturating Humanoid torques: exactly 2 iterations per Newton
    (as the reference), finite state, not rolled back."""
    cfg = abi.default_step_config()
    cfg.krylov_max_iters = 2
    cfg.krylov_tol = 1e-14
    m = abi.builtin_model("humanoid")
    task = S.quiet_task()
    g = VecEnv(model=m, task_config=task, step_config=cfg, n_envs=8, precision=precision, seed=4)
    o = oracle.OracleEnv(m, task, cfg, 8, seed=4, kind="reference")
    g.set_state(o.get_state())
    tm = np.array([m.joints[j].max_torque for j in range(m.n_joints)])
    tq = o.random_actions(0) * tm
    H, rhs, kry, ns = g.first_system(0, tq)
    assert list(kry) == [2] * cfg.newton_iters
    g.physics_step(tq)
    o.physics_step(tq)
    rep = g.report()
    assert (rep["krylov_iterations"] == 2 * cfg.newton_iters).all() and rep["failed"].sum() == 0
    # StepReport.krylov_iterations: the scene total over islands (types.hpp:115-120)
    assert int(rep["krylov_iterations"].sum()) == int(o.report()["krylov_iterations"][0])
    assert np.isfinite(g.get_state()).all()


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_clamp_torques(precision):
    """test_physics.cpp:180-191: torques beyond +-tau_max are clamped (the
    pendulum's tau_max = 100: +-150 steps exactly like +-100, unlike 50); a
    torque vector of the wrong length is rejected."""
    p = S.pendulum()
    cfg = S.tight_config()
    runs = {}
    for tau in (150.0, 100.0, 50.0, -150.0, -100.0):
        g = _make(p.build(), cfg, precision=precision)
        g.set_state(p.state()[None])
        g.physics_step(np.array([[tau]]))
        runs[tau] = g.get_state()
    np.testing.assert_array_equal(runs[150.0], runs[100.0])
    np.testing.assert_array_equal(runs[-150.0], runs[-100.0])
    assert not np.array_equal(runs[100.0], runs[50.0])
    with pytest.raises(ValueError):
        g.physics_step(np.zeros((1, 2)))
