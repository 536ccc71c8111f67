"""Step throughput of every BASELINE config on one B200 (random actions, auto-reset, hot L2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import VecEnv


def terrain(n_boxes, extent, seed=3):
    spec = abi.TerrainSpec(count=n_boxes, dim_lo=0.2, dim_hi=1.0, x_lo=-3.0, x_hi=extent, y_lo=-3.0, y_hi=extent,
                           yaw_lo=0.0, yaw_hi=3.141592653589793, seed=seed)
    boxes = (abi.StaticBox * n_boxes)()
    assert abi.load().stp_generate_terrain(spec, boxes, n_boxes) == n_boxes
    return list(boxes)


def run(task, n, boxes=None, steps=30):
    env = VecEnv(task, n_envs=n, seed=3, terrain=boxes)
    env.reset()
    acts = [env.random_actions(s) for s in range(steps)]
    for s in range(5):
        env.step(acts[s])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(5, steps):
        env.step(acts[s])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (steps - 5)
    rep = env.report()
    print(f"{task:12s} n {n:5d} boxes {0 if boxes is None else len(boxes):5d}  ms {ms:.4f}  Menv-steps/s {n / ms / 1e3:6.2f}"
          f"  overflow {int(rep['overflow'].sum())} failed {int(rep['failed'].sum())}")
    env.close()


if __name__ == "__main__":
  if os.environ.get("ONLY") == "ant":
    for n in (64, 512, 1024, 1776, 2048, 4096):
      run("ant", n)
    sys.exit(0)
  run("ant", 64)
  run("ant", 4096)
  run("humanoid", 1024)
  run("humanoid", 4096)
  run("hfh", 4096)
# HFH env grid: 64 columns x 2 m -> 4096 envs span ~128 m x 128 m
  run("hfh_terrain", 4096, terrain(2048, 131.0))
  run("hfh_terrain", 4096, terrain(8192, 131.0))
