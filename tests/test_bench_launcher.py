"""bench.py's multi-rank launch and the reference arm's
isolation from the product library, on CPU: `--impl
reference --gpus 2` re-launches itself as 2 ranks (torch.distributed.run,
gloo), rank 0 alone prints one JSON line."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not oracle.available("reference_fast") and not oracle.available("restatement"),
                    reason="oracle not built")
def test_reference_arm_self_launches_two_ranks():
    env = dict(os.environ, STP_BENCH_CPU_BUDGET_S="1.5", CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.bench_config(2)
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and "value_1_thread" in cb and "cpu_model" in cb
    libs = d["repo_libraries_loaded"]
    assert libs is not None and not any("libstampede_b200" in p for p in libs), libs
    assert any(p.startswith("oracle") for p in libs), libs
