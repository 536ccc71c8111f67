"""The INTEGRATION.md adapter compiled: integration/gpu_stepper.hpp
(GpuStepper, the glue a reference maintainer would add) built against the
reference's own headers, stepping one reference Scene next to the unmodified
physics::step (solver.hpp:52-53) and comparing states, ordered contact lists,
iteration totals and failed_agents (types.hpp:115-120).  The binary is built
where /root/reference exists (integration/Makefile, from __graft_entry__.build)
and travels with the repo like the other built libraries."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_gpu_stepper")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build/test_gpu_stepper not built")]


@pytest.mark.parametrize("precision,agents,steps", [("f64", 16, 40), ("f32", 16, 40), ("f64", 3, 120)])
def test_gpu_stepper_matches_physics_step(precision, agents, steps):
    r = subprocess.run([BIN, precision, str(agents), str(steps)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
