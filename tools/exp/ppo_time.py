"""PPO iteration time (rollout of 32 frames x 4096 envs + 20-epoch update) with
fp32 or TF32 learner GEMMs (experiment; GPU box).  usage: python tools/exp/ppo_time.py [tf32]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_1810_05762_b200.policy import HIDDEN, ActorCritic, PolicyKernel, RunningStat
from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner, gae
from paper_1810_05762_b200.ppo import rollout as ppo_rollout
from paper_1810_05762_b200.sim import VecEnv

if "tf32" in sys.argv[1:]:
    torch.backends.cuda.matmul.allow_tf32 = True
N = 4096
env = VecEnv("humanoid", n_envs=N, seed=1)
torch.manual_seed(0)
model = ActorCritic(env.obs_dim, env.action_dim, HIDDEN["humanoid"]).cuda()
cfg = PPOConfig()
learner = PPOLearner(model, cfg)
kern = PolicyKernel(model, "cuda:0")
st = RunningStat(env.obs_dim, device="cuda:0")
env.last_obs = env.reset()
st.push(env.last_obs)
times, upd = [], []
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    data, last_val = ppo_rollout(env, kern, st, cfg.frames_per_iter, 1, 1000 + it * cfg.frames_per_iter)
    loc = RunningStat(env.obs_dim, device="cuda:0")
    loc.push(data["obs"].reshape(-1, env.obs_dim))
    st._merge(loc.n, loc.mean, loc.m2)
    adv, ret = gae(data["rew"], data["val"], data["done"], last_val, cfg.gamma, cfg.lam)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stats = learner.update(st.whiten(data["obs"].reshape(-1, env.obs_dim)), data["act"].reshape(-1, env.action_dim),
                           None, adv.reshape(-1), ret.reshape(-1))
    kern.refresh()
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
    upd.append(time.perf_counter() - t1)
print(f"{'tf32' if 'tf32' in sys.argv[1:] else 'fp32'}: iteration {statistics.median(times[1:]) * 1e3:.1f} ms, "
      f"update {statistics.median(upd[1:]) * 1e3:.1f} ms, kl {stats['kl']:.2e} aborted {stats['aborted']}")
