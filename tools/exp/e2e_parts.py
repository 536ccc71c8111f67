"""Where does the e2e (stp_step_host) time go?  Per-call wall time of
stp_step_host at several env counts next to the device-timed step of the same
envs (experiment; run on the GPU box)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_1810_05762_b200.sim import VecEnv

for n in [int(x) for x in os.environ.get("NS", "64 1024 4096").split()]:
    env = VecEnv("humanoid", n_envs=n, seed=1)
    obs = env.reset()
    acts = [env.random_actions(s) for s in range(16)]
    rew = torch.empty(n, device="cuda")
    done = torch.empty(n, dtype=torch.uint8, device="cuda")
    for s in range(10):
        env.step(acts[s % 16], obs, rew, done)
    torch.cuda.synchronize()
    K = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(K):
        env.step(acts[s % 16], obs, rew, done)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / K
    h_acts = [a.cpu().pin_memory() for a in acts]
    h_obs = torch.empty((n, env.obs_dim), pin_memory=True)
    h_rew = torch.empty(n, pin_memory=True)
    h_done = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pa = [ctypes.c_void_p(t.data_ptr()) for t in h_acts]
    po = [ctypes.c_void_p(t.data_ptr()) for t in (h_obs, h_rew, h_done)]
    f = env.lib.stp_step_host
    for s in range(10):
        f(env._h, pa[s % 16], *po)
    t0 = time.perf_counter()
    for s in range(K):
        f(env._h, pa[s % 16], *po)
    host_ms = (time.perf_counter() - t0) / K * 1e3
    # the same call without outputs: H2D + kernel + sync only
    t0 = time.perf_counter()
    for s in range(K):
        f(env._h, pa[s % 16], None, None, None)
    in_ms = (time.perf_counter() - t0) / K * 1e3
    print(f"n {n:5d}  device step {dev_ms * 1e3:7.1f} us   step_host {host_ms * 1e3:7.1f} us   "
          f"(no outputs {in_ms * 1e3:7.1f} us)   overhead {host_ms * 1e3 - dev_ms * 1e3:6.1f} us")
