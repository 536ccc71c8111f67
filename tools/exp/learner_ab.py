"""A/B of the PPO learner's minibatch step (config C5, Humanoid pi + V SELU
MLPs (256, 128, 64), fp32): the per-module autograd graph (two MLPs, cuBLAS
per Linear) against pi and V grouped (layer 1 as one [O, 512] GEMM, layers
2-3 as batched GEMMs over the two nets, the heads separate).  Times forward +
backward of the surrogate-shaped loss with CUDA events, per minibatch size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_1810_05762_b200.policy import ActorCritic  # noqa: E402

dev = torch.device("cuda:0")
O, A = 77, 21


def plain(m, x):
    return m.pi(x), m.v(x).squeeze(-1)


def grouped(m, x):
    p, v = m.pi.layers, m.v.layers
    w1 = torch.cat([p[0].weight, v[0].weight], 0)
    b1 = torch.cat([p[0].bias, v[0].bias], 0)
    h = F.selu(torch.addmm(b1, x, w1.t()))                      # [B, 512]
    h = h.view(-1, 2, p[0].out_features).transpose(0, 1)        # [2, B, 256]
    for li in (1, 2):
        w = torch.stack([p[li].weight, v[li].weight]).transpose(1, 2)
        b = torch.stack([p[li].bias, v[li].bias]).unsqueeze(1)
        h = F.selu(torch.baddbmm(b, h, w))
    mu = torch.addmm(p[3].bias, h[0], p[3].weight.t())
    val = torch.addmm(v[3].bias, h[1], v[3].weight.t()).squeeze(-1)
    return mu, val


def run(fn, m, x, reps=20):
    def once():
        mu, val = fn(m, x)
        loss = (mu * mu).mean() + (val * val).mean()
        m.zero_grad(set_to_none=False)
        loss.backward()
    for _ in range(3):
        once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


torch.manual_seed(0)
m = ActorCritic(O, A).to(dev)
for B in (131072, 32768):
    x = torch.randn(B, O, device=dev)
    # same gradients
    m.zero_grad()
    mu, val = plain(m, x)
    ((mu * mu).mean() + (val * val).mean()).backward()
    g0 = [p.grad.clone() for p in m.parameters() if p.grad is not None]
    m.zero_grad()
    mu, val = grouped(m, x)
    ((mu * mu).mean() + (val * val).mean()).backward()
    g1 = [p.grad.clone() for p in m.parameters() if p.grad is not None]
    err = max(float((a - b).abs().max() / (a.abs().max() + 1e-30)) for a, b in zip(g0, g1))
    for tf32 in (False, True):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        print(f"B={B} tf32={tf32} plain {run(plain, m, x):.3f} ms  grouped {run(grouped, m, x):.3f} ms  "
              f"grad rel diff {err:.2e}", flush=True)
    torch.backends.cuda.matmul.allow_tf32 = False
