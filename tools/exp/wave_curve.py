"""Step time vs env count (Humanoid, random actions, L2 flushed between steps):
where the wave quantisation of the step kernel shows (12 resident warps / SM x
148 SMs = 1776 envs per wave)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1810_05762_b200.sim import VecEnv  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for n in [int(x) for x in os.environ.get("NS", "592,1184,1776,2368,2960,3552,4096,4736,5328").split(",")]:
    env = VecEnv("humanoid", n_envs=n, seed=1234)
    env.reset()
    acts = [env.random_actions(s) for s in range(40)]
    for s in range(10):
        env.step(acts[s])
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
    for i in range(30):
        flush.fill_(float(i))
        ev[i][0].record()
        env.step(acts[10 + i])
        ev[i][1].record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)[15]
    print(f"n {n:5d}  waves {n / 1776:4.2f}  ms {ms:.4f}  us/env-wave-slot {1e3 * ms / max(1, -(-n // 1776)):.1f}  "
          f"M env-steps/s {n / ms / 1e3:.1f}", flush=True)
    del env
