"""Independent reward / observation oracle (TEST INFRASTRUCTURE ONLY).

A second implementation of the env layer's scalar functions, written from
PAPER.md App. B/C and SPEC.md:279-305 (compute_reward), :243-246 (the
observation layout) and the decisions of DESIGN.md §5, in vectorised numpy
and with different formulas from the C++ oracle (oracle/env_oracle.cpp) and
the CUDA epilogue:

  * heading: cos(theta_target) from the body x axis projected on the ground
    (the yaw direction = the first column of R(q)) against the direction to
    the target, instead of cos(atan2(target - root) - yaw);
  * uprightness: R(q)[2, 2] from the rotation matrix;
  * joint angles: from the relative rotation matrix's axis-angle (the
    rotation angle of rest^-1 * q_p^-1 * q_c projected on the hinge axis, via
    the quaternion's vector part as in joint_angle, solver.cpp:405-411, but
    computed from matrices), not the quaternion product chain.

SPEC.md:287 asks for "randomized states -> equals an independently coded
reward oracle"; tests/test_gpu_envparity.py evaluates it on the CUDA path's
own pre / post states, actions, targets and feet flags.
"""
from __future__ import annotations

import numpy as np


def quat_to_mat(q):
    """[..., 4] (w x y z) -> [..., 3, 3] rotation matrices."""
    q = np.asarray(q, np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _mat_to_quat(R):
    """Rotation matrices -> unit quaternions with w >= 0 (Shepperd's method)."""
    R = np.asarray(R, np.float64)
    out = np.empty(R.shape[:-2] + (4,))
    tr = R[..., 0, 0] + R[..., 1, 1] + R[..., 2, 2]
    cand = np.stack([tr, R[..., 0, 0], R[..., 1, 1], R[..., 2, 2]], -1)
    k = np.argmax(cand, -1)
    for i in range(4):
        m = k == i
        if not m.any():
            continue
        Rm = R[m]
        if i == 0:
            s = np.sqrt(1 + Rm[:, 0, 0] + Rm[:, 1, 1] + Rm[:, 2, 2]) * 2
            q = np.stack([s / 4, (Rm[:, 2, 1] - Rm[:, 1, 2]) / s, (Rm[:, 0, 2] - Rm[:, 2, 0]) / s,
                          (Rm[:, 1, 0] - Rm[:, 0, 1]) / s], -1)
        elif i == 1:
            s = np.sqrt(1 + Rm[:, 0, 0] - Rm[:, 1, 1] - Rm[:, 2, 2]) * 2
            q = np.stack([(Rm[:, 2, 1] - Rm[:, 1, 2]) / s, s / 4, (Rm[:, 0, 1] + Rm[:, 1, 0]) / s,
                          (Rm[:, 0, 2] + Rm[:, 2, 0]) / s], -1)
        elif i == 2:
            s = np.sqrt(1 + Rm[:, 1, 1] - Rm[:, 0, 0] - Rm[:, 2, 2]) * 2
            q = np.stack([(Rm[:, 0, 2] - Rm[:, 2, 0]) / s, (Rm[:, 0, 1] + Rm[:, 1, 0]) / s, s / 4,
                          (Rm[:, 1, 2] + Rm[:, 2, 1]) / s], -1)
        else:
            s = np.sqrt(1 + Rm[:, 2, 2] - Rm[:, 0, 0] - Rm[:, 1, 1]) * 2
            q = np.stack([(Rm[:, 1, 0] - Rm[:, 0, 1]) / s, (Rm[:, 0, 2] + Rm[:, 2, 0]) / s,
                          (Rm[:, 1, 2] + Rm[:, 2, 1]) / s, s / 4], -1)
        out[m] = q
    out *= np.where(out[..., :1] < 0, -1.0, 1.0)
    return out


def joint_tables(model):
    J = model.n_joints
    par = np.array([model.joints[j].parent for j in range(J)])
    chi = np.array([model.joints[j].child for j in range(J)])
    axis = np.array([[model.joints[j].axis_child[k] for k in range(3)] for j in range(J)])
    rest = np.array([[model.joints[j].rest_relative[k] for k in range(4)] for j in range(J)])
    lo = np.array([model.joints[j].limit_lo for j in range(J)])
    hi = np.array([model.joints[j].limit_hi for j in range(J)])
    return par, chi, axis, rest, lo, hi


def joint_angles(model, state):
    """Hinge angles [N, J] of states [N, B, 13] (joint_angle semantics,
    solver.cpp:405-411) from rotation matrices."""
    par, chi, axis, rest, _, _ = joint_tables(model)
    Rb = quat_to_mat(state[:, :, 3:7])
    Rrest = quat_to_mat(rest)  # [J, 3, 3]
    # D = Rrest^T Rp^T Rc  (relative rotation away from the rest orientation)
    rel = np.einsum("njba,njbc->njac", Rb[:, par], Rb[:, chi])
    D = np.einsum("jba,njbc->njac", Rrest, rel)
    dq = _mat_to_quat(D)  # w >= 0, like the dq.w < 0 flip
    proj = np.einsum("njk,jk->nj", dq[..., 1:], axis)
    return 2.0 * np.arctan2(proj, dq[..., 0])


def joint_rates(model, state):
    """Hinge rates [N, J]: child-axis projection of w_child - w_parent
    (joint_velocity, solver.cpp:413-417)."""
    par, chi, axis, _, _, _ = joint_tables(model)
    Rc = quat_to_mat(state[:, chi, 3:7])
    axw = np.einsum("njab,jb->nja", Rc, axis)
    return np.einsum("nja,nja->nj", axw, state[:, chi, 10:13] - state[:, par, 10:13])


def reward(model, cfg, pre_root_xy, post, actions, target, feet, failed=None):
    """compute_reward (App. C), vectorised over envs.

    pre_root_xy [N, 2]: root xy before the step; post [N, B, 13]: state after
    it; actions [N, A] (normalised torques); target [N, 2] (the target the step
    ran against); feet [N, n_feet] (0/1 static contact of each foot this step).
    Returns (total [N], parts dict) with the discrete decisions' margins."""
    r = model.root
    _, _, _, _, lo, hi = joint_tables(model)
    root = post[:, r]
    R = quat_to_mat(root[:, 3:7])
    to_tgt0 = target - pre_root_xy
    dist0 = np.linalg.norm(to_tgt0, axis=1)
    disp = root[:, :2] - pre_root_xy
    S = np.where(dist0 > 0, np.einsum("nk,nk->n", disp, to_tgt0) / np.where(dist0 > 0, dist0, 1) / cfg.dt, 0.0)
    fwd = R[:, :2, 0]
    to_tgt = target - root[:, :2]
    cth = np.einsum("nk,nk->n", fwd, to_tgt) / (np.linalg.norm(fwd, axis=1) * np.linalg.norm(to_tgt, axis=1))
    rhead = np.where(cth > 0.8, 1.0, cth / 0.8)
    cvert = R[:, 2, 2]
    rstand = (cvert > 0.93).astype(np.float64)
    u = np.asarray(actions, np.float64)
    tcost = np.abs(np.clip(u, -1.0, 1.0)).sum(1)
    ucost = (u * u).sum(1)
    ang = joint_angles(model, post)
    act = cfg.limit_activation
    at_lim = ((ang - lo) < act) | ((hi - ang) < act)
    nlim = at_lim.sum(1)
    nfeet = np.asarray(feet, np.float64).sum(1)
    total = model.alive_bonus + S + 0.5 * rhead + 0.05 * rstand - 4.0 * tcost - 0.5 * ucost - 0.2 * nlim - nfeet
    if failed is not None:
        total = np.where(np.asarray(failed) != 0, 0.0, total)
    lim_margin = np.minimum(np.abs(ang - lo - act), np.abs(hi - ang - act)).min(1)
    return total, dict(S=S, rhead=rhead, rstand=rstand, nlim=nlim, nfeet=nfeet, cth=cth, cvert=cvert,
                       stand_margin=np.abs(cvert - 0.93), limit_margin=lim_margin, angles=ang)


def observation(model, post, target, last_tau, feet):
    """The 11 + 3J + n_feet observation:
    [h, roll, pitch, v (yaw frame) 3, w (yaw frame) 3, sin / cos(target
    bearing - yaw), theta J, theta_dot J, last clamped torque J, feet]."""
    r = model.root
    root = post[:, r]
    R = quat_to_mat(root[:, 3:7])
    fwd = R[:, :2, 0] / np.linalg.norm(R[:, :2, 0], axis=1, keepdims=True)  # (cos yaw, sin yaw)
    c, s = fwd[:, 0], fwd[:, 1]
    roll = np.arctan2(R[:, 2, 1], R[:, 2, 2])
    pitch = np.arcsin(np.clip(-R[:, 2, 0], -1, 1))
    v, w = root[:, 7:10], root[:, 10:13]
    to_tgt = target - root[:, :2]
    bearing = to_tgt / np.linalg.norm(to_tgt, axis=1, keepdims=True)
    sin_h = bearing[:, 1] * c - bearing[:, 0] * s
    cos_h = bearing[:, 0] * c + bearing[:, 1] * s
    cols = [root[:, 2:3], roll[:, None], pitch[:, None],
            np.stack([c * v[:, 0] + s * v[:, 1], -s * v[:, 0] + c * v[:, 1], v[:, 2]], 1),
            np.stack([c * w[:, 0] + s * w[:, 1], -s * w[:, 0] + c * w[:, 1], w[:, 2]], 1),
            sin_h[:, None], cos_h[:, None], joint_angles(model, post), joint_rates(model, post),
            np.asarray(last_tau, np.float64), np.asarray(feet, np.float64)]
    return np.concatenate(cols, 1)
