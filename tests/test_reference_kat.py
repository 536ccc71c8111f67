"""The reference's known-answer physics tests (test_physics.cpp:124-485) on the
CPU oracle: the restated physics and, when built, the compiled reference."""
import pytest

import kat
import oracle

BACKENDS = ["restatement", "reference"]


def maker(kind):
    if not oracle.available(kind):
        pytest.skip(f"oracle backend {kind} not built (needs /root/reference)")

    def make(model, task, cfg, n):
        return oracle.OracleEnv(model, task, cfg, n, kind=kind)
    return make


@pytest.mark.parametrize("kind", BACKENDS)
@pytest.mark.parametrize("case", kat.ALL, ids=lambda f: f.__name__)
def test_kat(kind, case):
    case(maker(kind))
