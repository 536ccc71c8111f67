"""fp32 env-layer parity of the CUDA path:
observation / reward / termination of the product precision against the
double oracle, the independent App. C reward oracle, and the fp32-only
elementary functions.  Protocols and stated bounds: tests/parity.py."""
import numpy as np
import pytest

import parity as P

pytestmark = pytest.mark.gpu


def _show(name, rep):
    keys = ["dx", "dv", "reward"] + [k for k in P.BOUNDS if k in rep and k not in ("dx", "dv", "reward")]
    print(f"\n{name}: {rep['steps']} steps x {rep['n_envs']} envs, done events {rep['done_events']}, "
          f"done mismatch {rep['done_mismatch']} boundary {rep['done_boundary']}, feet {rep['feet_flag_mismatch']}, "
          f"reward flips {rep['reward_discrete_flips']}, reset err {rep['reset_state_obs_err'].get('max')}")
    for k in keys:
        g, f = rep[k]["gpu"], rep[k].get("f32", {})
        line = f"  {k:12s} gpu p99 {g.get('p99', 0):.2e} max {g.get('max', 0):.2e}"
        if f.get("n"):
            line += f" | fp32 restatement p99 {f['p99']:.2e} max {f['max']:.2e}"
        print(line)


def _check(rep, absolute=True):
    env_steps = rep["steps"] * rep["n_envs"]
    assert rep["done_mismatch"]["gpu"] == 0, rep["done_mismatch"]
    # boundary terminations (|h - threshold| < 1e-5) are reported, and rare
    assert rep["done_boundary"]["gpu"] <= max(2, 1e-3 * env_steps)
    assert rep["failed"]["gpu"] == rep["failed"]["oracle"] == 0
    env = rep["dx"].get("f32", {}).get("n", 0) > 0
    assert rep["feet_flag_mismatch"]["gpu"] <= max(2 * rep["feet_flag_mismatch"]["f32"], 1e-3 * env_steps)
    assert rep["reward_discrete_flips"]["gpu"] <= max(2 * rep["reward_discrete_flips"]["f32"], 5e-3 * env_steps)
    if rep["reset_state_obs_err"]["n"]:
        assert rep["reset_state_obs_err"]["max"] <= P.RESET_MAX
    for k, (p99, mx) in P.BOUNDS.items():
        if k not in rep:
            continue
        g, f = rep[k]["gpu"], rep[k].get("f32", {})
        assert g["n"] > 0
        if env and f.get("n"):  # bulk never worse than 2x the reference algorithm in fp32
            assert g["p99"] <= max(2 * f["p99"], p99 / 10), (k, g, f)
        if absolute:
            assert g["p99"] <= p99, (k, g)
            if mx is not None:
                assert g["max"] <= mx, (k, g)


@pytest.mark.parametrize("name,scale", [("humanoid", 1.0), ("humanoid", 0.1), ("ant", 1.0)])
def test_teacher_forced_env_step_fp32(name, scale):
    """32 envs x 500 env_steps, teacher-forced from the double oracle,
    saturating and low torques; Humanoids fall and auto-reset."""
    rep = P.teacher_forced_env(name, n=32, steps=500, seed=7, scale=scale)
    _show(f"{name} x{scale}", rep)
    if name == "humanoid" and scale == 1.0:
        assert rep["done_events"] >= 100  # falls + auto-resets exercised
        assert rep["reset_state_obs_err"]["n"] > 0
    _check(rep, absolute=(name == "humanoid"))


def test_teacher_forced_hfh_with_interagent_against_reference():
    """HFH (fall grace 160, flagrun, inter-agent collisions): teacher-forced
    against the compiled reference physics (contact-merged islands)."""
    rep = P.teacher_forced_env("hfh", n=32, steps=300, seed=7, envelope=False, oracle_kind="reference")
    _show("hfh", rep)
    _check(rep, absolute=True)


def _terrain(n_boxes=160, seed=3):
    from paper_1810_05762_b200 import abi
    spec = abi.TerrainSpec(count=n_boxes, dim_lo=0.2, dim_hi=1.0, x_lo=-3.0, x_hi=66.0, y_lo=-3.0, y_hi=3.0,
                           yaw_lo=0.0, yaw_hi=3.141592653589793, seed=seed)
    boxes = (abi.StaticBox * n_boxes)()
    assert abi.load().stp_generate_terrain(spec, boxes, n_boxes) == n_boxes
    return list(boxes)


def test_teacher_forced_hfh_terrain_fp32():
    """HFH on complex terrain (config C4 shape: 160 yaw boxes over the 32 envs'
    strip): teacher-forced env_step over 200 steps against the compiled
    reference physics (inter-agent islands on, as for flat HFH): box contacts,
    the 15 x 11 height-map observation, flagrun and falls."""
    rep = P.teacher_forced_env("hfh_terrain", n=32, steps=200, seed=7, terrain=_terrain(), envelope=False,
                               oracle_kind="reference")
    _show("hfh terrain", rep)
    assert "height_map" in rep
    # samples at box edges may jump between the sides (explained by each side's
    # own state; tests/parity.py HM_JUMP / HM_OWN): at most 0.1 % of them
    assert rep["height_map_edge_flips"] <= 1e-3 * 165 * rep["height_map"]["gpu"]["n"]
    _check(rep, absolute=True)


def test_bench_config_teacher_forced():
    """The bench workload itself: 4096 Humanoids, seed 1234, auto-reset, after
    64 free-running GPU steps; 3 steps with the oracle teacher-forced from the
    GPU's state."""
    rep = P.teacher_forced_env("humanoid", n=4096, steps=3, seed=1234, source="gpu", warm=64)
    _show("bench config", rep)
    assert rep["done_events"] > 0
    _check(rep, absolute=True)


@pytest.mark.parametrize("name", ["humanoid", "ant"])
def test_reward_matches_independent_oracle(name):
    """>= 10^4 randomized states (random targets in every
    direction, out-of-range actions, upright / falling / lying bodies)."""
    rep = P.reward_vs_independent_oracle(name, n=4096 if name == "humanoid" else 2560, steps=4)
    print(rep)
    assert rep["states"] >= 10_000
    assert rep["abs_err"]["p99"] <= P.REWARD_ORACLE["p99"] and rep["abs_err"]["max"] <= P.REWARD_ORACLE["max"]
    assert rep["boundary_flips"] <= 1e-3 * rep["states"]
    assert min(rep["heading_le_gt_0.8"]) > 100
    if name == "humanoid":
        assert min(rep["standing_0_1"]) > 100


def _debug_math(fn, x, y=None):
    import ctypes as C
    import torch
    from paper_1810_05762_b200 import abi
    xs = torch.as_tensor(x, dtype=torch.float32, device="cuda")
    ys = torch.as_tensor(y if y is not None else x, dtype=torch.float32, device="cuda")
    o0, o1 = torch.empty_like(xs), torch.empty_like(xs)
    rc = abi.load().stp_debug_math(fn, C.c_void_p(xs.data_ptr()), C.c_void_p(ys.data_ptr()),
                                   C.c_void_p(o0.data_ptr()), C.c_void_p(o1.data_ptr()), xs.numel(), None)
    assert rc == 0
    torch.cuda.synchronize()
    return o0.cpu().numpy().astype(np.float64), o1.cpu().numpy().astype(np.float64)


def test_fp32_sincos_bound():
    """The fp32 step's sincos (Cody-Waite + Cephes): against
    double sin / cos of the same fp32 argument, |err| <= 2.4e-7 (2 ulp of 1)
    for |x| <= 1e4; NaN / inf give NaN (the divergence votes rely on it)."""
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-4, 4, 1 << 20), rng.uniform(-1e4, 1e4, 1 << 20),
                        np.arange(-64, 65) * np.pi / 4, [0.0, -0.0, 1e-30, -1e-30]]).astype(np.float32)
    s, c = _debug_math(0, x)
    xd = x.astype(np.float64)
    es, ec = np.abs(s - np.sin(xd)), np.abs(c - np.cos(xd))
    print(f"sincos: max |sin err| {es.max():.2e}, |cos err| {ec.max():.2e} over {x.size} args")
    assert es.max() <= 2.4e-7 and ec.max() <= 2.4e-7
    s, c = _debug_math(0, np.array([np.nan, np.inf, -np.inf], np.float32))
    assert np.isnan(s).all() and np.isnan(c).all()


def test_fp32_unit_direction_bound():
    """The fp32 heading terms' (sin, cos) of atan2(y, x) from the unit vector
    (one rsqrt): |err| <= 3e-7 against double; atan2(0, 0) -> (0, 1)."""
    rng = np.random.default_rng(1)
    y = np.concatenate([rng.normal(size=1 << 20) * 10 ** rng.uniform(-3, 2, 1 << 20), [0.0]]).astype(np.float32)
    x = np.concatenate([rng.normal(size=1 << 20) * 10 ** rng.uniform(-3, 2, 1 << 20), [0.0]]).astype(np.float32)
    s, c = _debug_math(1, y, x)
    a = np.arctan2(y.astype(np.float64), x.astype(np.float64))
    es, ec = np.abs(s - np.sin(a)), np.abs(c - np.cos(a))
    print(f"unit_dir: max |sin err| {es.max():.2e}, |cos err| {ec.max():.2e}")
    assert es.max() <= 3e-7 and ec.max() <= 3e-7
    assert s[-1] == 0.0 and c[-1] == 1.0
