"""Host enqueue cost vs device time of the HFH step (inter-agent path)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200.sim import VecEnv
for task in ("humanoid", "hfh"):
    env = VecEnv(task, n_envs=4096, seed=3)
    acts = [env.random_actions(s) for s in range(50)]
    obs = torch.empty((4096, env.obs_dim), device="cuda"); r = torch.empty(4096, device="cuda"); d = torch.empty(4096, dtype=torch.uint8, device="cuda")
    for s in range(5): env.step(acts[s], obs, r, d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(5, 50): env.step(acts[s], obs, r, d)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{task}: host enqueue {1e6*(t1-t0)/45:.1f} us/step, wall incl. sync {1e6*(t2-t0)/45:.1f} us/step")
