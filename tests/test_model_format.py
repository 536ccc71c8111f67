"""Articulation text format "stampede-model 1" (SPEC.md:198-205 load_model,
:223-226 round trip): the bundled assets equal the built-in models, load ->
serialize -> load is the identity, the SPEC examples hold, and malformed
documents fail with descriptive errors.  Host-only (no GPU)."""
import os

import pytest

from paper_1810_05762_b200 import abi

ASSETS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "assets")


def _read(name):
    with open(os.path.join(ASSETS, f"{name}.model")) as f:
        return f.read()


@pytest.mark.parametrize("name", ["ant", "humanoid"])
def test_bundled_asset_is_the_builtin_model(name):
    assert bytes(abi.model_from_text(_read(name))) == bytes(abi.builtin_model(name))


@pytest.mark.parametrize("name", ["ant", "humanoid"])
def test_round_trip_identity(name):
    m = abi.builtin_model(name)
    text = abi.model_to_text(m)
    m2 = abi.model_from_text(text)
    assert bytes(m2) == bytes(m)
    assert abi.model_to_text(m2) == text  # canonical form is a fixed point


def test_spec_examples():
    """ant 8 actuated joints / 4 feet; humanoid 21 actuated
    joints and 28 DoF (7 root pose coordinates + 21 hinges)."""
    ant = abi.model_from_text(_read("ant"))
    assert ant.n_joints == 8 and ant.n_feet == 4
    hum = abi.model_from_text(_read("humanoid"))
    assert hum.n_joints == 21 and 7 + hum.n_joints == 28


MINI = """stampede-model 1
name mini
body a
  shape capsule
  radius 0.05
  half_length 0.2
  mass 1
  inertia 0.1 0.1 0.01
  rest 0 0 1 1 0 0 0 0 0 0 0 0 0
end
body b
  shape sphere
  radius 0.05
  mass 0.5
  inertia 0.001 0.001 0.001
  rest 0 0 0.6 1 0 0 0 0 0 0 0 0 0
end
joint j
  parent a
  child b
  anchor_parent 0 0 -0.2
  anchor_child 0 0 0.2
  axis_parent 0 1 0
  axis_child 0 1 0
  limit -1 1
end
actuator j 10
root a
"""


def test_minimal_document_parses():
    m = abi.model_from_text(MINI)
    assert m.n_bodies == 2 and m.n_joints == 1 and m.root == 0
    assert m.joints[0].parent == 0 and m.joints[0].child == 1 and m.joints[0].max_torque == 10


@pytest.mark.parametrize("bad,msg", [
    (MINI.replace("root a\n", ""), "missing field 'root'"),
    (MINI.replace("  mass 1\n", "  mass 0\n"), "nonpositive mass"),
    (MINI.replace("  parent a\n  child b\n", "  parent b\n  child b\n"), "cyclic joint graph"),
    (MINI.replace("  radius 0.05\n  half_length", "  radiuz 0.05\n  half_length"), "line 5: unknown body field 'radiuz'"),
    (MINI.replace("  local_pos", "  local_pos").replace("  inertia 0.1 0.1 0.01", "  inertia 0.1 0.1"),
     "expected 3 number(s) after 'inertia'"),
    (MINI.replace("actuator j 10\n", ""), "without an 'actuator'"),
    (MINI.replace("stampede-model 1", "stampede-model 2"), "unsupported model format version 2"),
    ("", "empty document"),
])
def test_malformed_documents_are_rejected(bad, msg):
    with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        abi.model_from_text(bad)


@pytest.mark.parametrize("name", ["ant", "humanoid"])
def test_oracle_reader_matches_builtin(name):
    """The oracle's own reader (oracle/model_text.py, used by bench.py's CPU
    arms so they never load the product library) yields the same bytes as the
    product's built-in model, and the same defaults."""
    import ctypes as C

    import model_text
    a, b = model_text.load_model(name), abi.builtin_model(name)
    assert bytes(a) == bytes(b)
    assert bytes(model_text.default_step_config()) == bytes(abi.default_step_config())
    for k in (abi.TASK_ANT, abi.TASK_HUMANOID, abi.TASK_HFH, abi.TASK_HFH_TERRAIN):
        assert bytes(model_text.default_task(k)) == bytes(abi.default_task(k))
    assert C.sizeof(a) == C.sizeof(abi.Model)


def test_oracle_terrain_generator_matches_device_library():
    """The CPU arms' terrain restatement draws exactly the boxes of
    stp_generate_terrain (same counter-based RNG)."""
    import model_text
    spec = abi.TerrainSpec(count=200, dim_lo=0.2, dim_hi=1.0, x_lo=-3.0, x_hi=131.0, y_lo=-3.0, y_hi=131.0,
                           yaw_lo=0.0, yaw_hi=3.141592653589793, seed=3)
    boxes = (abi.StaticBox * 200)()
    assert abi.load().stp_generate_terrain(spec, boxes, 200) == 200
    ours = model_text.generate_terrain(200, 0.2, 1.0, -3.0, 131.0, -3.0, 131.0, 0.0, 3.141592653589793, 3)
    for a, b in zip(boxes, ours):
        assert bytes(a) == bytes(b)
