"""Kernel timeline of the HFH step (torch.profiler / CUPTI activity): start, end and
gaps of every kernel in a few steps, to see where the HFH step spends the time the
step kernel does not.  usage: WL=hfh4096 python tools/exp/hfh_timeline.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1810_05762_b200.sim import VecEnv  # noqa: E402

wl = bench.WORKLOADS[os.environ.get("WL", "hfh4096")]
kw = {}
if wl.get("boxes"):
    kw["terrain"] = bench.terrain_boxes(wl["boxes"], wl["extent"])
env = VecEnv(wl["task"], n_envs=wl["n"], seed=1234, **kw)
env.reset()
WARM = int(os.environ.get("WARM", "20"))  # WARM=160: a crowded scene (2-env islands)
acts = [env.random_actions(s) for s in range(WARM + 10)]
for s in range(WARM):
    env.step(acts[s])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for s in range(WARM, WARM + 5):
        env.step(acts[s])
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/hfh_trace.json")
ev = json.load(open("/tmp/hfh_trace.json"))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
t0 = k[0]["ts"]
prev_end = None
for e in k:
    gap = "" if prev_end is None else f"gap {e['ts'] - prev_end:7.1f}"
    print(f"{e['ts'] - t0:9.1f} us  dur {e['dur']:7.1f}  stream {e['args'].get('stream')}  {gap}  {e['name'][:60]}")
    prev_end = max(prev_end or 0, e["ts"] + e["dur"])
print(f"span {prev_end - t0:.1f} us for 5 steps")

# host side: runtime API calls per step (cuda_runtime events) and wall time per env.step
rt = sorted([e for e in ev if e.get("cat") == "cuda_runtime"], key=lambda e: e["ts"])
from collections import defaultdict  # noqa: E402
agg = defaultdict(lambda: [0, 0.0])
for e in rt:
    agg[e["name"]][0] += 1
    agg[e["name"]][1] += e["dur"]
print("runtime API over 5 steps:")
for name, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {name:40s} calls {c:4d}  total {d:8.1f} us  mean {d / c:6.1f} us")
import time  # noqa: E402
torch.cuda.synchronize()
t = time.perf_counter()
for s in range(50):
    env.step(acts[s % len(acts)])
t_host = (time.perf_counter() - t) / 50
torch.cuda.synchronize()
t_all = (time.perf_counter() - t) / 50
print(f"host time per env.step (no sync) {1e6 * t_host:.1f} us; wall per step incl. drain {1e6 * t_all:.1f} us")
