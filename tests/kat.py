"""Known-answer tests of the reference (test_physics.cpp:124-485), written once
against the common VecEnv/OracleEnv method names and run on every backend:
the restated oracle, the compiled reference (oracle/_ref) and the GPU kernel
in f64 and f32.  Tolerances are the reference's; the f32 GPU path gets the
stated fp32 allowances passed in `tol`."""
from __future__ import annotations

import math

import numpy as np

import scenes as S


def joint_angle(state, joint):
    """joint_angle, solver.cpp:405-411"""
    qp = state[joint.parent, 3:7]
    qc = state[joint.child, 3:7]
    rest = np.array(joint.rest_relative[:])
    rel = S.qmul(S.qconj(qp), qc)
    d = S.qmul(S.qconj(rest), rel)
    if d[0] < 0:
        d = -d
    proj = d[1] * joint.axis_child[0] + d[2] * joint.axis_child[1] + d[3] * joint.axis_child[2]
    return 2.0 * math.atan2(proj, d[0])


def joint_velocity(state, joint):
    axw = S.qrot(state[joint.child, 3:7], np.array(joint.axis_child[:]))
    return float(axw @ (state[joint.child, 10:13] - state[joint.parent, 10:13]))


def kat_sphere_contact(make):
    """test_physics.cpp:124-135"""
    cfg = S.abi.default_step_config()
    cfg.contact_margin = 0.0
    sc = S.sphere_scene(0.4)
    env = make(sc.build(), S.quiet_task(), cfg, 1)
    env.set_state(sc.state()[None])
    env.physics_step(np.zeros((1, 0)))
    c = env.contact_arrays()
    assert c["count"][0] == 1
    assert abs(c["separation"][0, 0] - (-0.1)) <= 1e-6 * 0.1 + 1e-12
    assert abs(c["normal"][0, 0, 2] - 1.0) <= 1e-12
    assert c["body_b"][0, 0] == -1
    cfg.contact_margin = 0.01
    sc2 = S.sphere_scene(10.0)
    env2 = make(sc2.build(), S.quiet_task(), cfg, 1)
    env2.set_state(sc2.state()[None])
    env2.physics_step(np.zeros((1, 0)))
    assert env2.contact_arrays()["count"][0] == 0


def kat_free_fall(make, rel=1e-12):
    """test_physics.cpp:193-200"""
    sc = S.sphere_scene(100.0)
    env = make(sc.build(), S.quiet_task(), S.abi.default_step_config(), 1)
    env.set_state(sc.state()[None])
    env.physics_step(np.zeros((1, 0)))
    s = env.get_state()[0, 0]
    assert abs(s[9] - (-9.8 / 120.0)) <= rel * 9.8 / 120.0
    assert abs(s[2] - (100.0 - 9.8 / 120.0 / 120.0)) <= rel * 100.0


def kat_box_rest(make):
    """test_physics.cpp:202-217"""
    sc = S.box_scene()
    env = make(sc.build(), S.quiet_task(), S.abi.default_step_config(), 1)
    env.set_state(sc.state()[None])
    for _ in range(10):
        env.physics_step(np.zeros((1, 0)))
    s = env.get_state()[0, 0]
    assert abs(0.5 - s[2]) <= 1e-3
    assert abs(s[9]) <= 1e-3
    env.physics_step(np.zeros((1, 0)))
    c = env.contact_arrays()
    total = c["normal_impulse"][0, : c["count"][0]].sum()
    assert abs(total - 9.8 / 120.0) <= 0.05 * 9.8 / 120.0


def kat_pendulum(make, tol1=1e-4, tol11=5e-3):
    """test_physics.cpp:219-245"""
    sc = S.pendulum()
    model = sc.build()
    cfg = S.no_plane(S.tight_config())
    env = make(model, S.quiet_task(), cfg, 1)
    env.set_state(sc.state()[None])
    ip = S.PEND_I + S.PEND_COM ** 2
    theta = omega = 0.0
    omega += cfg.dt * 9.8 * S.PEND_COM * math.cos(theta) / ip
    theta += cfg.dt * omega
    env.physics_step(np.zeros((1, 1)))
    assert abs(joint_angle(env.get_state()[0], model.joints[0]) - theta) <= tol1
    for _ in range(10):
        omega += cfg.dt * 9.8 * S.PEND_COM * math.cos(theta) / ip
        theta += cfg.dt * omega
        env.physics_step(np.zeros((1, 1)))
    assert abs(joint_angle(env.get_state()[0], model.joints[0]) - theta) <= tol11


def kat_motor(make):
    """test_physics.cpp:247-256"""
    sc = S.pendulum()
    model = sc.build()
    env = make(model, S.quiet_task(), S.no_plane(S.tight_config()), 1)
    env.set_state(sc.state()[None])
    env.physics_step(np.full((1, 1), 5.0))
    assert joint_velocity(env.get_state()[0], model.joints[0]) > 0.245


def kat_friction_cone(make, pushes=(5.0, 15.0, 40.0)):
    """test_physics.cpp:343-364"""
    for push in pushes:
        sc = S.box_scene()
        env = make(sc.build(), S.quiet_task(), S.abi.default_step_config(), 1)
        env.set_state(sc.state()[None])
        for _ in range(60):
            env.physics_step(np.zeros((1, 0)))
        for _ in range(60):
            loads = np.zeros((1, 1, 6))
            loads[0, 0, 0] = push
            env.set_external_loads(loads)
            env.physics_step(np.zeros((1, 0)))
            c = env.contact_arrays()
            n = c["count"][0]
            pn = c["normal_impulse"][0, :n]
            pt = np.linalg.norm(c["tangential_impulse"][0, :n], axis=1)
            assert (pn >= -1e-9).all()
            assert (pt <= pn * (1 + 1e-6) + 1e-9).all()
        vx = env.get_state()[0, 0, 7]
        if push == 40.0:
            assert vx > 0.05
        if push == 5.0:
            assert vx < 0.01


def kat_joint_limits(make, tol=1e-3):
    """test_physics.cpp:366-384"""
    sc = S.pendulum(-0.5, 0.5)
    model = sc.build()
    env = make(model, S.quiet_task(), S.no_plane(S.tight_config(4, 200)), 1)
    env.set_state(sc.state()[None])
    for torque in (100.0, -100.0):
        for _ in range(240):
            env.physics_step(np.full((1, 1), torque))
            a = joint_angle(env.get_state()[0], model.joints[0])
            assert -0.5 - tol <= a <= 0.5 + tol


def kat_energy(make, rel=1e-3):
    """test_physics.cpp:386-430"""
    sc = S.chain(3)
    model = sc.build()
    env = make(model, S.quiet_task(), S.no_plane(S.tight_config(2, 100)), 1)
    env.set_state(sc.state()[None])

    def energy(st):
        e = 0.0
        for b in range(1, 4):
            s = st[b]
            m = model.bodies[b].mass
            I = np.array(model.bodies[b].inertia_diag[:])
            e += 0.5 * m * s[7:10] @ s[7:10]
            R = np.array([S.qrot(s[3:7], ax) for ax in np.eye(3)]).T
            Iw = R @ np.diag(I) @ R.T
            e += 0.5 * s[10:13] @ Iw @ s[10:13] + m * 9.8 * s[2]
        return e

    e0 = energy(env.get_state()[0])
    for _ in range(120):
        env.physics_step(np.zeros((1, 3)))
        assert energy(env.get_state()[0]) <= e0 + rel * (abs(e0) + 1.0)


def kat_batching(make, tol=1e-6, steps=50):
    """test_physics.cpp:432-485: 3 agents batched == 3 single scenes."""
    M = 3
    sc = S.two_link()
    model = sc.build()
    cfg = S.abi.default_step_config()
    batched = make(model, S.quiet_task(), cfg, M)
    st = np.stack([S.two_link(2.0 * a).state() for a in range(M)])
    batched.set_state(st)
    singles = [make(model, S.quiet_task(), cfg, 1) for _ in range(M)]
    for a in range(M):
        singles[a].set_state(st[a:a + 1])
    for t in range(steps):
        tq = np.array([[3.0 * math.sin(0.1 * t + a)] for a in range(M)])
        batched.physics_step(tq)
        for a in range(M):
            singles[a].physics_step(tq[a:a + 1])
    bs = batched.get_state()
    for a in range(M):
        ss = singles[a].get_state()[0]
        assert np.abs(bs[a][:, [0, 1, 2, 3, 7]] - ss[:, [0, 1, 2, 3, 7]]).max() <= tol


ALL = [kat_sphere_contact, kat_free_fall, kat_box_rest, kat_pendulum, kat_motor, kat_friction_cone,
       kat_joint_limits, kat_energy, kat_batching]
