import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200.sim import VecEnv
env = VecEnv("hfh", n_envs=4096, seed=1234)
hits = []
for t in range(int(os.environ.get("STEPS", "200"))):
    n = len(env.detect_inter_agent()["body_a"])
    if n:
        hits.append(t)
    env.step(env.random_actions(t))
print("steps with inter-agent contacts:", hits[:20], len(hits))
