"""Ant at 4096 envs: a few env steps (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200.sim import VecEnv

env = VecEnv("ant", n_envs=4096, seed=3)
env.reset()
for s in range(12):
    env.step(env.random_actions(s))
torch.cuda.synchronize()
rep = env.report()
print("ok krylov per env-step", float(rep["krylov_iterations"].mean()), "newton", float(rep["newton_iterations"].mean()))
