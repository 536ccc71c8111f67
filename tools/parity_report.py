#!/usr/bin/env python3
"""Run the fp32 env-layer parity protocols (tests/parity.py) on cuda:0 and
write the statistics to profiles/<name>.json (default r02_parity.json).

    python tools/parity_report.py [--out profiles/r02_parity.json] [--quick]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import parity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_parity.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    steps = 60 if args.quick else 500
    t0 = time.time()
    rep = {"kernel_build": os.environ.get("STP_BUILD") or subprocess.run(
               ["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True, text=True).stdout.strip() or None,
           "protocols": {}}
    P = rep["protocols"]
    P["reward_independent_oracle_humanoid"] = parity.reward_vs_independent_oracle("humanoid")
    P["reward_independent_oracle_ant"] = parity.reward_vs_independent_oracle("ant", n=2048)
    P["teacher_forced_humanoid_saturating"] = parity.teacher_forced_env("humanoid", steps=steps, scale=1.0)
    P["teacher_forced_humanoid_low"] = parity.teacher_forced_env("humanoid", steps=steps, scale=0.1)
    P["teacher_forced_ant_saturating"] = parity.teacher_forced_env("ant", steps=steps, scale=1.0)
    P["teacher_forced_hfh_reference"] = parity.teacher_forced_env("hfh", steps=steps, envelope=False,
                                                                  oracle_kind="reference")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_envparity import _terrain  # noqa: E402
    P["teacher_forced_hfh_terrain_reference"] = parity.teacher_forced_env(
        "hfh_terrain", steps=min(steps, 200), terrain=_terrain(), envelope=False, oracle_kind="reference")
    P["bench_config_4096_seed1234"] = parity.teacher_forced_env("humanoid", n=4096, steps=3, seed=1234,
                                                               source="gpu", warm=64, envelope=True)
    rep["seconds"] = time.time() - t0
    with open(args.out, "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
