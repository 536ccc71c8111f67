"""Step time under three cache conditions: L2 flushed between steps (256 MiB
write), inputs larger than L2 (H handles of 4096 envs stepped round-robin,
no flush: state / obs / actions of each step not L2-resident, kernel code
cached), and hot (one handle, no flush)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1810_05762_b200.sim import VecEnv
N, K, H = 4096, 60, 24
envs = [VecEnv("humanoid", n_envs=N, seed=1234 + h) for h in range(H)]
bufs = [(torch.empty((N, e.obs_dim), device="cuda"), torch.empty(N, device="cuda"),
         torch.empty(N, dtype=torch.uint8, device="cuda")) for e in envs]
acts = [[e.random_actions(s) for s in range(4)] for e in envs]
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
for e, b, a in zip(envs, bufs, acts):
    for s in range(3):
        e.step(a[s], *b)
torch.cuda.synchronize()
def run(mode):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        h = k % H if mode == "rotate" else 0
        if mode == "flush":
            flush.fill_(float(k))
        ev[k][0].record()
        envs[h].step(acts[h][k % 4], *bufs[h])
        ev[k][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / K
for m in ["flush", "rotate", "hot", "flush", "rotate", "hot"]:
    print(f"{m:7s} {run(m):.4f} ms/step")
