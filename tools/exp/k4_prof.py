"""Drive K4 (rollout policy forward, 4096 Humanoid envs) for an ncu capture:
ncu ... -k regex:k_policy -s 20 -c 1 python tools/exp/k4_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1810_05762_b200.policy import ActorCritic, PolicyKernel  # noqa: E402
from paper_1810_05762_b200.sim import VecEnv  # noqa: E402

env = VecEnv("humanoid", n_envs=4096)
obs = env.reset()
kern = PolicyKernel(ActorCritic(env.obs_dim, env.action_dim).to("cuda"), "cuda:0")
m_ = torch.zeros(env.obs_dim, device="cuda")
s_ = torch.ones(env.obs_dim, device="cuda")
for it in range(30):
    _, a, _, _ = kern.forward(obs, m_, s_, step=it)
    obs, _, _ = env.step(a)
torch.cuda.synchronize()
print("ok")
