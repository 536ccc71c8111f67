"""Gaussian SELU policy / value networks (Table 4)
with the rollout forward on the tcgen05 kernel (K4, csrc/policy_mlp.cu) and
observation whitening by a mergeable RunningStat.

The torch modules are the fp32 reference and the PPO learner's autograd
graph; `PolicyKernel.forward` runs the packed bf16 weights on the tensor
cores through the C-ABI `stp_policy_forward`.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch
import torch.nn as nn

from . import abi

SELU_L = 1.0507009873554805
SELU_A = 1.6732632423543772
HIDDEN = {"ant": (128, 64, 32), "humanoid": (256, 128, 64), "hfh": (256, 128, 64)}


def _pad16(x: int) -> int:
    return (x + 15) // 16 * 16


class MLP(nn.Module):
    """affine-SELU chain, identity output."""

    def __init__(self, sizes):
        super().__init__()
        self.layers = nn.ModuleList(nn.Linear(a, b) for a, b in zip(sizes[:-1], sizes[1:]))
        for l in self.layers:  # LeCun normal for SELU
            nn.init.normal_(l.weight, 0.0, 1.0 / math.sqrt(l.in_features))
            nn.init.zeros_(l.bias)

    def forward(self, x):
        for i, l in enumerate(self.layers):
            x = l(x)
            if i < len(self.layers) - 1:
                x = torch.selu(x)
        return x


class RunningStat:
    """count / mean / M2 with Chan's parallel merge.

    `merge_allreduce` combines the statistics of all ranks with one SUM
    allreduce of [n, n*mean, M2 + n*mean^2] (the obs-statistics allreduce)."""

    def __init__(self, dim: int, device="cpu"):
        self.n = torch.zeros((), dtype=torch.float64, device=device)
        self.mean = torch.zeros(dim, dtype=torch.float64, device=device)
        self.m2 = torch.zeros(dim, dtype=torch.float64, device=device)

    def push(self, x: torch.Tensor):
        x = x.to(torch.float64).reshape(-1, self.mean.numel())
        nb = x.shape[0]
        if nb == 0:
            return
        mb = x.mean(0)
        m2b = ((x - mb) ** 2).sum(0)
        self._merge(torch.tensor(float(nb), dtype=torch.float64, device=self.mean.device), mb, m2b)

    def _merge(self, nb, mb, m2b):
        n = self.n + nb
        d = mb - self.mean
        self.mean = self.mean + d * (nb / n)
        self.m2 = self.m2 + m2b + d * d * (self.n * nb / n)
        self.n = n

    def merge_allreduce(self, local: "RunningStat", group=None):
        """self += sum over ranks of `local` (exact Chan merge via moments)."""
        import torch.distributed as dist
        buf = torch.cat([local.n.reshape(1), local.n * local.mean, local.m2 + local.n * local.mean ** 2])
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        n = buf[0]
        if n > 0:
            mean = buf[1:1 + self.mean.numel()] / n
            m2 = buf[1 + self.mean.numel():] - n * mean ** 2
            self._merge(n, mean, m2.clamp_min(0))

    @property
    def std(self):
        """max(std, 1e-6) of the count-based variance M2 / n (whiten)."""
        var = self.m2 / torch.clamp(self.n, min=1.0)
        return torch.clamp(torch.sqrt(var), min=1e-6)

    def whiten(self, x):
        return torch.clamp((x - self.mean.to(x.dtype)) / self.std.to(x.dtype), -10.0, 10.0)


class ActorCritic(nn.Module):
    def __init__(self, obs_dim: int, act_dim: int, hidden=(256, 128, 64)):
        super().__init__()
        self.obs_dim, self.act_dim, self.hidden = obs_dim, act_dim, tuple(hidden)
        self.pi = MLP([obs_dim, *hidden, act_dim])
        self.v = MLP([obs_dim, *hidden, 1])
        self.log_std = nn.Parameter(torch.full((act_dim,), -0.5))

    def forward_ref(self, xw: torch.Tensor):
        """fp32 reference on whitened observations: (mean, value)."""
        return self.pi(xw), self.v(xw).squeeze(-1)

    def log_prob(self, xw, actions):
        mu = self.pi(xw)
        std = torch.exp(self.log_std)
        return (-0.5 * ((actions - mu) / std) ** 2 - self.log_std - 0.5 * math.log(2 * math.pi)).sum(-1)


def pack_linear(layer: nn.Linear, device):
    """bf16 weights in the UMMA K-major core-matrix layout [K/8][N][8] (padded to 16)."""
    w = layer.weight.detach().to(torch.float32)
    n, k = w.shape
    npad, kpad = _pad16(n), _pad16(k)
    wp = torch.zeros(npad, kpad, dtype=torch.float32, device=w.device)
    wp[:n, :k] = w
    packed = wp.view(npad, kpad // 8, 8).permute(1, 0, 2).contiguous().to(torch.bfloat16).to(device)
    b = torch.zeros(npad, dtype=torch.float32, device=device)
    b[:n] = layer.bias.detach().to(device)
    return packed, b


class PolicyKernel:
    """Packed copy of an ActorCritic for the tcgen05 rollout forward (K4)."""

    def __init__(self, model: ActorCritic, device="cuda:0"):
        self.lib = abi.load()
        self.device = torch.device(device)
        self.model = model
        self.refresh()

    def refresh(self):
        """Re-pack after a learner update."""
        m = self.model
        self.pi = [pack_linear(l, self.device) for l in m.pi.layers]
        self.v = [pack_linear(l, self.device) for l in m.v.layers]
        self.log_std = m.log_std.detach().to(self.device, torch.float32).contiguous()
        self.dims_pi = (C.c_int32 * 5)(m.obs_dim, *m.hidden, m.act_dim)
        self.dims_v = (C.c_int32 * 5)(m.obs_dim, *m.hidden, 1)
        self._wpi = (C.c_void_p * 4)(*[w.data_ptr() for w, _ in self.pi])
        self._bpi = (C.c_void_p * 4)(*[b.data_ptr() for _, b in self.pi])
        self._wv = (C.c_void_p * 4)(*[w.data_ptr() for w, _ in self.v])
        self._bv = (C.c_void_p * 4)(*[b.data_ptr() for _, b in self.v])

    def forward(self, obs: torch.Tensor, obs_mean: torch.Tensor, obs_std: torch.Tensor, seed: int = 0,
                step: int = 0, env_offset: int = 0, sample: bool = True, value: bool = True):
        n, od = obs.shape
        dev = self.device
        obs = obs.to(dev, torch.float32).contiguous()
        mean = obs_mean.to(dev, torch.float32).contiguous()
        std = obs_std.to(dev, torch.float32).contiguous()
        mu = torch.empty((n, self.model.act_dim), dtype=torch.float32, device=dev)
        act = torch.empty_like(mu) if sample else None
        logp = torch.empty((n,), dtype=torch.float32, device=dev) if sample else None
        val = torch.empty((n,), dtype=torch.float32, device=dev) if value else None
        p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)
        h = torch.cuda.current_stream(dev).cuda_stream
        rc = self.lib.stp_policy_forward(p(obs), n, od, p(mean), p(std), self.dims_pi,
                                         C.cast(self._wpi, C.c_void_p), C.cast(self._bpi, C.c_void_p),
                                         self.dims_v, C.cast(self._wv, C.c_void_p), C.cast(self._bv, C.c_void_p),
                                         p(self.log_std), C.c_uint64(seed), C.c_uint64(step),
                                         C.c_int64(env_offset), p(mu), p(act), p(logp), p(val),
                                         C.c_void_p(h if h else 1))
        if rc != abi.STP_OK:
            raise RuntimeError(f"stp_policy_forward failed ({rc}): {abi.last_error()}")
        return mu, act, logp, val


# -- counter-based Gaussian noise of the kernel, restated for tests -----------
def _mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def kernel_noise(seed: int, env: int, step: int, act_dim: int) -> np.ndarray:
    """The policy noise of K4 (policy_mlp.cu, noise lambda): Box-Muller pairs,
    one splitmix64 hash per pair of actions q = 0, 1, ...: u1 = bits 40-63,
    u2 = bits 16-39 (24-bit uniforms), r = sqrt(-2 ln max(u1, 1e-7)),
    theta = 2 pi u2 - pi; eps[2q] = r cos(theta), eps[2q + 1] = r sin(theta)."""
    s = _mix64(_mix64(_mix64(seed) ^ 6) ^ ((env << 32) | (step & 0xFFFFFFFF)))
    out = np.zeros(act_dim, np.float32)
    for q in range((act_dim + 1) // 2):
        z = _mix64((s + q) & 0xFFFFFFFFFFFFFFFF)
        u1 = np.float32((z >> 40) * (1.0 / 16777216.0))
        u2 = np.float32(((z >> 16) & 0xFFFFFF) * (1.0 / 16777216.0))
        u1 = max(u1, np.float32(1e-7))
        rad = math.sqrt(-2.0 * math.log(u1))
        th = 2 * math.pi * float(u2) - math.pi
        out[2 * q] = rad * math.cos(th)
        if 2 * q + 1 < act_dim:
            out[2 * q + 1] = rad * math.sin(th)
    return out
