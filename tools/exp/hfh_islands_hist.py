"""HFH (4096 envs, random actions) as the scene evolves: step time and the
contact-merged island size histogram (union-find over the inter-agent contact
pairs of detect_inter_agent), to see which island path dominates."""
import os
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_05762_b200.sim import VecEnv  # noqa: E402

task = os.environ.get("TASK", "hfh")
env = VecEnv(task, n_envs=4096, seed=1234)
env.reset()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(int(os.environ.get("STEPS", "400")))]
for t in range(int(os.environ.get("STEPS", "400"))):
    a = env.random_actions(t)
    ev[t][0].record()
    env.step(a)
    ev[t][1].record()
    if t % 50 == 49:
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ev[t - 49:t + 1]]
        d = env.detect_inter_agent()
        nb = env.n_bodies
        ea, eb = (d["body_a"] // nb).astype(np.int64), (d["body_b"] // nb).astype(np.int64)
        par = list(range(4096))

        def f(x):
            while par[x] != x:
                par[x] = par[par[x]]
                x = par[x]
            return x
        for x, y in zip(ea.tolist(), eb.tolist()):
            rx, ry = f(x), f(y)
            if rx != ry:
                par[rx] = ry
        sizes = Counter(Counter(f(x) for x in set(ea.tolist()) | set(eb.tolist())).values())
        print(f"steps {t - 49:3d}-{t}: median {np.median(ms):.4f} ms, max {max(ms):.4f}; islands by size "
              f"{dict(sorted(sizes.items()))}", flush=True)
