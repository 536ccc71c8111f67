"""HFH host-buffer step (stp_step_host, the e2e path): CUPTI timeline of
copies and kernels and the host API time per call."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1810_05762_b200.sim import VecEnv  # noqa: E402

task = os.environ.get("TASK", "hfh")
env = VecEnv(task, n_envs=4096, seed=1234)
env.reset()
acts = [env.random_actions(s).cpu().numpy() for s in range(20)]
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
acts = [pin(a) for a in acts]
obs = pin(np.empty((4096, env.obs_dim), np.float32))
rew = pin(np.empty(4096, np.float32))
done = pin(np.empty(4096, np.uint8))
for s in range(10):
    env.step_host(acts[s], obs, rew, done)
torch.cuda.synchronize()
t = time.perf_counter()
for s in range(10):
    env.step_host(acts[s % 20], obs, rew, done)
print(f"wall per step_host call {1e6 * (time.perf_counter() - t) / 10:.1f} us")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for s in range(3):
        env.step_host(acts[s], obs, rew, done)
prof.export_chrome_trace("/tmp/e2e_trace.json")
ev = json.load(open("/tmp/e2e_trace.json"))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
rt = sorted([e for e in ev if e.get("cat") == "cuda_runtime"], key=lambda e: e["ts"])
t0 = min(k[0]["ts"], rt[0]["ts"])
for e in sorted(k + [r for r in rt if r["dur"] > 3], key=lambda e: e["ts"])[:60]:
    print(f"{e['ts'] - t0:9.1f} dur {e['dur']:7.1f} {e.get('cat'):12s} {e['name'][:70]}")
