"""SPEC env-layer examples on the CPU oracle env layer (restated physics and,
when built, the compiled reference physics underneath)."""
import pytest

import envspec
import oracle
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import MODEL_OF_TASK, TASKS


def maker(kind):
    if not oracle.available(kind):
        pytest.skip(f"oracle backend {kind} not built")

    def make(task, n):
        env = oracle.OracleEnv(abi.builtin_model(MODEL_OF_TASK[task]), abi.default_task(TASKS[task]),
                               abi.default_step_config(), n, seed=11, kind=kind)
        return env
    return make


@pytest.mark.parametrize("kind", ["restatement", "reference"])
@pytest.mark.parametrize("case", envspec.ALL, ids=lambda f: f.__name__)
def test_env_spec(kind, case):
    case(maker(kind), 1e-4)  # S picks up ~1e-5 m/s of joint-solver drift
