"""HFH step time as the scene evolves (falls, piles, islands), random actions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1810_05762_b200.sim import VecEnv
env = VecEnv("hfh", n_envs=4096, seed=1234)
obs = torch.empty((4096, env.obs_dim), device="cuda"); r = torch.empty(4096, device="cuda"); d = torch.empty(4096, dtype=torch.uint8, device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(800)]
for t in range(800):
    a = env.random_actions(t)
    ev[t][0].record(); env.step(a, obs, r, d); ev[t][1].record()
    if t % 100 == 99:
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ev[t - 99:t + 1]]
        dets = env.detect_inter_agent()
        nb = env.n_bodies
        envs = set((dets["body_a"] // nb).tolist()) | set((dets["body_b"] // nb).tolist())
        print(f"steps {t-99:3d}-{t}: {np.median(ms):.4f} ms median, max {max(ms):.4f}; inter-agent contacts {len(dets['body_a'])}, envs touching {len(envs)}, overflow {int(env.report()['overflow'].sum())}", flush=True)
