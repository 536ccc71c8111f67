"""HFH on terrain at 4096 envs (config C4 shape): a few steps for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200.sim import VecEnv
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from configs import terrain  # noqa: E402

env = VecEnv("hfh_terrain", n_envs=4096, seed=3, terrain=terrain(2048, 131.0))
env.reset()
for s in range(12):
    env.step(env.random_actions(s))
torch.cuda.synchronize()
print("ok")
