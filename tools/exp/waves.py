"""Step time vs env count (wave quantisation of k_env_step): 148 SMs x 12 resident warps = 1776 envs per wave."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200.sim import VecEnv

for n in [592, 1184, 1776, 2368, 2960, 3552, 4096, 4440, 5328, 7104, 8192]:
    env = VecEnv("humanoid", n_envs=n, seed=3)
    env.reset()
    acts = [env.random_actions(s) for s in range(20)]
    for s in range(5):
        env.step(acts[s])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(5, 20):
        env.step(acts[s])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 15
    print(f"n {n:5d}  waves {n / 1776:5.2f}  ms {ms:.4f}  us/env {ms * 1e3 / n * 1e3:.2f} ns  Menv-steps/s {n / ms / 1e3:.2f}")
    env.close()
