"""Where a C5 PPO iteration (4096 Humanoid envs, 32 frames, 20 epochs) spends
its time: torch.profiler kernel totals for one update after a warm-up."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1810_05762_b200.policy import HIDDEN, ActorCritic, PolicyKernel, RunningStat  # noqa: E402
from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner, gae, rollout  # noqa: E402
from paper_1810_05762_b200.sim import VecEnv  # noqa: E402

if os.environ.get("EPI"):
    import paper_1810_05762_b200.ppo as _ppo
    _ppo.FORWARD_EPILOGUE = os.environ["EPI"]
if os.environ.get("TF32") == "1":
    torch.backends.cuda.matmul.allow_tf32 = True
env = VecEnv("humanoid", n_envs=4096, seed=1234)
dev = torch.device("cuda:0")
torch.manual_seed(0)
model = ActorCritic(env.obs_dim, env.action_dim, HIDDEN["humanoid"]).to(dev)
cfg = PPOConfig(frames_per_iter=int(os.environ.get("FRAMES", "32")))
learner = PPOLearner(model, cfg)
kern = PolicyKernel(model, dev)
st = RunningStat(env.obs_dim, device=dev)
env.last_obs = env.reset()
st.push(env.last_obs)


def one(it):
    data, last_val = rollout(env, kern, st, cfg.frames_per_iter, 1234, 1000 + it * cfg.frames_per_iter)
    st.push(data["obs"].reshape(-1, env.obs_dim))
    ast = torch.zeros(3, dtype=torch.float64, device=dev)
    adv, ret = gae(data["rew"], data["val"], data["done"], last_val, cfg.gamma, cfg.lam, stats=ast)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = learner.update(st.whiten(data["obs"].reshape(-1, env.obs_dim)), data["act"].reshape(-1, env.action_dim),
                       None, adv.reshape(-1), ret.reshape(-1), adv_stats=ast)
    torch.cuda.synchronize()
    kern.refresh()
    return time.perf_counter() - t0, s


for it in range(2):
    print("update s", one(it))
ts = []
for it in range(2, 6):
    ts.append(one(it)[0])
print("update s median", sorted(ts)[len(ts) // 2], flush=True)
print("graphs", {str(k): v.captures for k, v in learner._mbs.items()}, flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    one(6)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18))
