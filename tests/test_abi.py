"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/stampede_sim.h declares, agrees with the Python struct layouts, and
rejects invalid input the way the reference does (std::invalid_argument ->
STP_EINVAL + stp_last_error)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1810_05762_b200 import abi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "stampede_sim.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(stp_[a-z0-9_]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    names = {n for n, _, _ in abi.SIGNATURES}
    assert set(declared()) <= names, set(declared()) - names


def test_struct_layouts_match():
    out = (C.c_int64 * 7)()
    abi.load().stp_struct_sizes(out)
    py = [C.sizeof(t) for t in (abi.Body, abi.Joint, abi.Model, abi.StepConfig, abi.StaticBox, abi.TerrainSpec,
                                abi.Task)]
    assert list(out) == py


def test_builtin_models_and_defaults():
    h = abi.builtin_model("humanoid")
    a = abi.builtin_model("ant")
    assert (h.n_bodies, h.n_joints, h.n_feet) == (22, 21, 2)  # "28 DoF" = 7 root + 21 hinges
    assert (a.n_bodies, a.n_joints, a.n_feet) == (9, 8, 4)
    assert abs(sum(h.bodies[b].mass for b in range(22)) - 40.0) < 1e-9
    lib = abi.load()
    assert lib.stp_validate_model(C.byref(h)) == 0 and lib.stp_validate_model(C.byref(a)) == 0
    c = abi.default_step_config()  # types.hpp:92-107
    assert (c.newton_iters, c.krylov_max_iters, c.krylov_tol, c.contact_margin) == (4, 16, 1e-6, 0.02)
    assert abs(c.dt - 1 / 120) < 1e-15 and c.gravity[2] == -9.8


def test_invalid_inputs_are_rejected():
    lib = abi.load()
    m = abi.Model()
    assert lib.stp_builtin_model(b"spider", C.byref(m)) == abi.STP_EINVAL
    assert "unknown model" in abi.last_error()
    m = abi.builtin_model("humanoid")
    m.joints[3].limit_lo, m.joints[3].limit_hi = 1.0, 0.5
    assert lib.stp_validate_model(C.byref(m)) == abi.STP_EINVAL
    assert "limits out of order" in abi.last_error()
    m = abi.builtin_model("humanoid")
    m.joints[0].axis_child[0] = 0.5
    assert lib.stp_validate_model(C.byref(m)) == abi.STP_EINVAL
    m = abi.builtin_model("ant")
    m.bodies[2].mass = 0.0
    assert lib.stp_validate_model(C.byref(m)) == abi.STP_EINVAL


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: without a device stp_create returns NULL with a CUDA error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = abi.load()
    m, t, c = abi.builtin_model("humanoid"), abi.default_task(abi.TASK_HUMANOID), abi.default_step_config()
    h = lib.stp_create(C.byref(m), C.byref(t), C.byref(c), 8, 0, 1, 0, 0)
    assert not h
    assert abi.last_error()
    c.gravity[2] = -9.81  # scene.cpp:40-41: |g| must be 9.8 (checked before the device)
    assert not lib.stp_create(C.byref(m), C.byref(t), C.byref(c), 8, 0, 1, 0, 0)
    assert "gravity" in abi.last_error()


def test_terrain_generation_deterministic_and_in_range():
    lib = abi.load()
    spec = abi.TerrainSpec(count=500, dim_lo=0.2, dim_hi=1.0, x_lo=-50, x_hi=50, y_lo=-50, y_hi=50, yaw_lo=0,
                           yaw_hi=3.141592653589793, seed=7)
    a = (abi.StaticBox * 500)()
    b = (abi.StaticBox * 500)()
    assert lib.stp_generate_terrain(C.byref(spec), a, 500) == 500
    assert lib.stp_generate_terrain(C.byref(spec), b, 500) == 500
    for i in range(500):
        assert bytes(a[i]) == bytes(b[i])
        for k in range(3):
            assert 0.1 <= a[i].half_extents[k] <= 0.5
        assert a[i].center[2] == a[i].half_extents[2]
    spec.count = 0
    assert lib.stp_generate_terrain(C.byref(spec), a, 500) == 0


def test_terrain_generation_is_uniform():
    """10^4 samples -> every dimension inside its declared range
    and Kolmogorov-Smirnov vs uniform passes at alpha = 0.01 (dims, x, y, yaw)."""
    from scipy import stats
    lib = abi.load()
    n = 10000
    spec = abi.TerrainSpec(count=n, dim_lo=0.2, dim_hi=1.0, x_lo=-30, x_hi=70, y_lo=-5, y_hi=5, yaw_lo=0,
                           yaw_hi=3.141592653589793, seed=2024)
    out = (abi.StaticBox * n)()
    assert lib.stp_generate_terrain(C.byref(spec), out, n) == n
    cols = {
        "dim_x": ([2 * out[i].half_extents[0] for i in range(n)], 0.2, 1.0),
        "dim_y": ([2 * out[i].half_extents[1] for i in range(n)], 0.2, 1.0),
        "dim_z": ([2 * out[i].half_extents[2] for i in range(n)], 0.2, 1.0),
        "x": ([out[i].center[0] for i in range(n)], -30.0, 70.0),
        "y": ([out[i].center[1] for i in range(n)], -5.0, 5.0),
        "yaw": ([out[i].yaw for i in range(n)], 0.0, 3.141592653589793),
    }
    for name, (v, lo, hi) in cols.items():
        assert lo <= min(v) and max(v) <= hi, name
        assert stats.kstest(v, "uniform", args=(lo, hi - lo)).pvalue > 0.01, name
