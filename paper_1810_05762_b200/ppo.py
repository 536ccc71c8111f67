"""PPO rollout + update for config C5 (SPEC.md:361-506 ppo, :508-577 dist).

Rollout: VecEnv (fused sm_100a step) + the tcgen05 policy forward (K4) on each
GPU's env shard.  Update: torch autograd on the ActorCritic; every minibatch
gradient is averaged across ranks with one allreduce of the flattened
gradient (the paper's Horovod/NCCL gradient averaging);
advantages are normalised with global statistics; the
observation RunningStat is merged across ranks once per iteration
(SPEC.md:374-377).  Parameters are broadcast from rank 0 at start
 so all ranks stay bit-identical.
"""
from __future__ import annotations

import dataclasses

import torch
import torch.distributed as dist

from .policy import ActorCritic, RunningStat


@dataclasses.dataclass
class PPOConfig:  # PAPER.md Table 4 (Humanoid)
    frames_per_iter: int = 32
    epochs: int = 20
    minibatch_per_agent: int = 32
    desired_kl: float = 0.02
    clip: float = 0.2
    gamma: float = 0.99
    lam: float = 0.95
    lr: float = 3e-4
    vf_coef: float = 0.5


def _dist():
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def broadcast_params(model: torch.nn.Module, src: int = 0):
    if _dist():
        for p in model.parameters():
            dist.broadcast(p.data, src)


def allreduce_mean_grads(model: torch.nn.Module):
    """Average gradients across ranks: ONE flattened allreduce per minibatch."""
    if not _dist():
        return
    grads = [p.grad for p in model.parameters() if p.grad is not None]
    flat = torch.cat([g.reshape(-1) for g in grads])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    flat /= dist.get_world_size()
    off = 0
    for g in grads:
        n = g.numel()
        g.copy_(flat[off:off + n].view_as(g))
        off += n


def global_normalize(adv: torch.Tensor) -> torch.Tensor:
    """Advantage normalisation with statistics over all ranks."""
    s = torch.stack([torch.tensor(float(adv.numel()), device=adv.device, dtype=torch.float64),
                     adv.double().sum(), (adv.double() ** 2).sum()])
    if _dist():
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
    n, sm, sq = s[0], s[1], s[2]
    mean = sm / n
    std = torch.sqrt(torch.clamp(sq / n - mean * mean, min=0.0)) + 1e-8
    return ((adv.double() - mean) / std).to(adv.dtype)


def gae(rewards, values, dones, last_value, gamma, lam):
    """Generalised advantage estimation over [T, N] tensors."""
    T = rewards.shape[0]
    adv = torch.zeros_like(rewards)
    last = torch.zeros_like(rewards[0])
    for t in reversed(range(T)):
        nv = last_value if t == T - 1 else values[t + 1]
        nonterm = 1.0 - dones[t].to(rewards.dtype)
        delta = rewards[t] + gamma * nv * nonterm - values[t]
        last = delta + gamma * lam * nonterm * last
        adv[t] = last
    return adv, adv + values


class PPOLearner:
    def __init__(self, model: ActorCritic, cfg: PPOConfig):
        self.model, self.cfg = model, cfg
        self.opt = torch.optim.Adam(model.parameters(), lr=cfg.lr)
        broadcast_params(model)

    def update(self, xw, actions, old_logp, adv, ret, generator: torch.Generator | None = None):
        """Clipped-surrogate PPO epochs with KL-adaptive step size.
        xw: whitened obs [B, O]; all tensors flat over (time, agents) of this rank."""
        cfg = self.cfg
        adv = global_normalize(adv)
        B = xw.shape[0]
        # Table 4: frames per iteration / minibatch size per agent = minibatches per epoch
        n_mb = max(1, cfg.frames_per_iter // max(1, cfg.minibatch_per_agent))
        mb = max(1, B // n_mb)
        stats = {}
        for epoch in range(cfg.epochs):
            perm = torch.randperm(B, generator=generator, device="cpu").to(xw.device)
            for s in range(0, B, mb):
                idx = perm[s:s + mb]
                logp = self.model.log_prob(xw[idx], actions[idx])
                ratio = torch.exp(logp - old_logp[idx])
                a = adv[idx]
                pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg.clip, 1 + cfg.clip) * a).mean()
                v = self.model.v(xw[idx]).squeeze(-1)
                vf = ((v - ret[idx]) ** 2).mean()
                loss = pg + cfg.vf_coef * vf
                self.opt.zero_grad(set_to_none=False)
                loss.backward()
                allreduce_mean_grads(self.model)
                self.opt.step()
            with torch.no_grad():  # KL-adaptive learning rate
                kl = (old_logp - self.model.log_prob(xw, actions)).mean()
                if _dist():
                    dist.all_reduce(kl, op=dist.ReduceOp.SUM)
                    kl /= dist.get_world_size()
                lr = self.opt.param_groups[0]["lr"]
                if kl > 2.0 * cfg.desired_kl:
                    lr = max(lr / 1.5, 1e-6)
                elif kl < 0.5 * cfg.desired_kl:
                    lr = min(lr * 1.5, 1e-2)
                for g in self.opt.param_groups:
                    g["lr"] = lr
                stats = {"kl": float(kl), "lr": lr, "loss": float(loss)}
        return stats


def rollout(env, kernel, obs_stat: RunningStat, frames: int, seed: int, step0: int, env_offset: int = 0):
    """Collect `frames` env steps for every agent of this rank on the GPU.
    Returns [T, N] tensors and the raw observations (for the RunningStat)."""
    dev = torch.device("cuda", env.device)
    obs = env.reset() if step0 == 0 else env.last_obs
    N, O = obs.shape
    A = env.action_dim
    buf = {k: [] for k in ("obs", "act", "logp", "val", "rew", "done")}
    mean = obs_stat.mean.to(dev, torch.float32)
    std = obs_stat.std.to(dev, torch.float32)
    for t in range(frames):
        mu, act, logp, val = kernel.forward(obs, mean, std, seed=seed, step=step0 + t, env_offset=env_offset)
        nobs, rew, done = env.step(act.clamp(-1.0, 1.0))
        for k, v in zip(("obs", "act", "logp", "val", "rew", "done"), (obs, act, logp, val, rew, done)):
            buf[k].append(v.clone())
        obs = nobs
    _, _, _, last_val = kernel.forward(obs, mean, std, seed=seed, step=step0 + frames, env_offset=env_offset,
                                       sample=False)
    env.last_obs = obs
    return {k: torch.stack(v) for k, v in buf.items()}, last_val
