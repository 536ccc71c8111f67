"""PPO rollout + update for config C5 (SPEC.md:361-506 ppo, :508-577 dist).

Rollout: VecEnv (fused sm_100a step) + the tcgen05 policy forward (K4) on each
GPU's env shard.  Update: per minibatch one gather of the observations, the
two MLPs' explicit forward / backward (cuBLAS GEMMs; each hidden SELU's
backward fused with its bias gradient, stp_selu_backward_bias), the loss head
and its output gradients in one CUDA kernel pair (stp_ppo_surrogate: log-prob,
ratio, clipped surrogate on the globally normalised advantages, value MSE,
the heads' bias gradients, the rollout columns gathered in-kernel) — all of
it one CUDA graph replay — then the fused Adam step; the GAE is a CUDA kernel
(stp_gae).  Host (CPU) tensors (the gloo tests of the distributed logic) run
the same loss under autograd.  Every minibatch
gradient is averaged across ranks with one allreduce of the flattened
gradient (the paper's Horovod/NCCL gradient averaging);
advantages are normalised with global statistics; the
observation RunningStat is merged across ranks once per iteration
(SPEC.md:374-377).  Parameters are broadcast from rank 0 at start
 so all ranks stay bit-identical.
"""
from __future__ import annotations

import copy
import dataclasses
import math
import os

import numpy as np
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
    # "fp32": IEEE fp32 GEMMs (cuBLAS SIMT kernels at these shapes); "tf32":
    # the GEMMs on the tensor cores with TF32 inputs (10-bit mantissa, fp32
    # accumulation): the 4096-env update 0.116 -> 0.063 s, but over 8 Adam
    # steps the parameter step moves 14 % from the fp64 restatement's (fp32:
    # 3e-5; tests/test_gpu_ppo.py bounds both), so it is opt-in
    matmul: str = "fp32"


def _dist():
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def broadcast_params(model: torch.nn.Module, src: int = 0):
    if _dist():
        for p in model.parameters():
            dist.broadcast(p.data, src)


def allreduce_mean_grads(model: torch.nn.Module, flat: torch.Tensor | None = None):
    """Average gradients across ranks: ONE flattened allreduce per minibatch.
    `flat`: the buffer every parameter's .grad is a view of (the GPU learner),
    reduced in place without the gather / scatter copies."""
    if not _dist():
        return
    if flat is not None:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
        flat /= dist.get_world_size()
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


def global_stats(adv: torch.Tensor, stats: torch.Tensor | None = None) -> torch.Tensor:
    """[count, sum, sum of squares] (float64) of the advantages over all ranks
    (SPEC.md:532-540): `stats` from the GAE kernel or computed here, then one
    SUM allreduce; no host synchronisation."""
    if stats is None:
        stats = torch.stack([torch.tensor(float(adv.numel()), device=adv.device, dtype=torch.float64),
                             adv.double().sum(), (adv.double() ** 2).sum()])
    s = stats.to(torch.float64).clone()
    if _dist():
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return s


FORWARD_EPILOGUE = "kernel"  # hidden layers: "kernel" = GEMM + stp_bias_selu; "addmm" = cuBLAS bias + torch SELU


def mlp_forward(layers, x):
    """Affine-SELU chain keeping every layer's input:
    returns [x, y_1, ..., y_L] (y_L = the identity output); each hidden
    SELU is applied in place on its GEMM's output (only the output is kept:
    the backward derives selu' from it)."""
    acts = [x]
    for i, l in enumerate(layers):
        hidden = i < len(layers) - 1
        if FORWARD_EPILOGUE == "kernel" and hidden:
            import ctypes as C
            from . import abi
            z = torch.mm(acts[-1], l.weight.detach().t())
            h = torch.cuda.current_stream(z.device).cuda_stream
            rc = abi.load().stp_bias_selu(C.c_void_p(z.data_ptr()), C.c_void_p(l.bias.data_ptr()), z.shape[0],
                                          z.shape[1], 1, C.c_void_p(h if h else 1))
            if rc != abi.STP_OK:
                raise RuntimeError(f"stp_bias_selu failed ({rc}): {abi.last_error()}")
            acts.append(z)
            continue
        z = torch.addmm(l.bias.detach(), acts[-1], l.weight.detach().t())
        acts.append(torch.selu_(z) if hidden else z)
    return acts


def mlp_backward(layers, acts, g, scratch):
    """Backward of mlp_forward for dL/d output g [B, out]: weight gradients
    g^T x into each layer's .grad (cuBLAS), the input gradient g W, then the
    hidden SELU backward fused with the bias gradient (stp_selu_backward_bias)
    into the previous layer's bias .grad.  The output layer's bias gradient
    is the caller's (the loss-head kernel reduces it); the first layer's input
    gradient is not formed."""
    import ctypes as C
    from . import abi
    lib = abi.load()
    h = torch.cuda.current_stream(g.device).cuda_stream
    for i in reversed(range(len(layers))):
        l = layers[i]
        torch.mm(g.t(), acts[i], out=l.weight.grad)
        if i == 0:
            break
        gx = torch.mm(g, l.weight.detach())
        y = acts[i]
        rc = lib.stp_selu_backward_bias(C.c_void_p(gx.data_ptr()), C.c_void_p(y.data_ptr()), gx.shape[0],
                                        gx.shape[1], C.c_void_p(layers[i - 1].bias.grad.data_ptr()),
                                        C.c_void_p(scratch.data_ptr()), C.c_void_p(h if h else 1))
        if rc != abi.STP_OK:
            raise RuntimeError(f"stp_selu_backward_bias failed ({rc}): {abi.last_error()}")
        g = gx


def surrogate_grad(mu, log_std, v, actions, old_logp, adv, ret, idx, adv_stats, clip, vf_coef, bad,
                   d_mu_bias=None, d_value_bias=None):
    """The minibatch loss head of ppo_update on the GPU (stp_ppo_surrogate,
    SPEC.md:455-467): returns (dL/dmu [mb, A], dL/dV [mb], dL/dlog_std [A],
    loss) for mu / v = the networks' outputs on the samples idx (None: rows
    0 .. mb-1) of the rollout
    columns; advantages normalised in-kernel from `adv_stats`; `bad` (float
    device scalar) is set to 1 when the loss is not finite; the output layers'
    bias gradients are written to d_mu_bias [A] / d_value_bias [1] if given."""
    import ctypes as C
    from . import abi
    mb, A = mu.shape
    dev = mu.device
    for name, t in (("actions", actions), ("old_logp", old_logp), ("adv", adv), ("ret", ret)):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError(f"surrogate_grad: {name} must be a contiguous float32 CUDA tensor")
    mu, v, log_std = mu.contiguous(), v.contiguous(), log_std.to(torch.float32).contiguous()
    idx = idx.to(torch.int64).contiguous() if idx is not None else None
    dmu, dv = torch.empty_like(mu), torch.empty_like(v)
    dls = torch.empty(A, dtype=torch.float32, device=dev)
    loss = torch.empty(3, dtype=torch.float32, device=dev)
    scratch = torch.empty(max(1, (mb + 127) // 128) * (2 * A + 3), dtype=torch.float64, device=dev)
    p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)
    h = torch.cuda.current_stream(dev).cuda_stream
    rc = abi.load().stp_ppo_surrogate(p(mu), p(log_std), p(v), p(actions), p(old_logp), p(adv), p(ret), p(idx), mb,
                                      A, p(adv_stats), C.c_float(clip), C.c_float(vf_coef), p(dmu), p(dv), p(dls),
                                      p(d_mu_bias), p(d_value_bias), p(loss), p(bad), p(scratch),
                                      C.c_void_p(h if h else 1))
    if rc != abi.STP_OK:
        raise RuntimeError(f"stp_ppo_surrogate failed ({rc}): {abi.last_error()}")
    return dmu, dv, dls, loss[0]


def global_normalize(adv: torch.Tensor, stats: torch.Tensor | None = None) -> torch.Tensor:
    """Advantage normalisation with statistics over all ranks.
    `stats` = [count, sum, sum of squares] (float64, e.g. from the GAE kernel);
    computed here when absent.  One SUM allreduce, no host synchronisation."""
    s = global_stats(adv, stats)
    n, sm, sq = s[0], s[1], s[2]
    mean = sm / n
    std = torch.sqrt(torch.clamp(sq / n - mean * mean, min=0.0)) + 1e-8
    return ((adv.double() - mean) / std).to(adv.dtype)


def gae(rewards, values, dones, last_value, gamma, lam, stats: torch.Tensor | None = None):
    """Generalised advantage estimation over [T, N] tensors.

    CUDA tensors run the product kernel (stp_gae: one thread per env, the
    backward recursion, the advantages' count / sum / sum of squares added into
    `stats` for the normalisation); host tensors (the gloo tests of the
    distributed logic) run the same recursion vectorised over the envs."""
    T = rewards.shape[0]
    if rewards.is_cuda:
        import ctypes as C
        from . import abi
        N = rewards.shape[1] if rewards.dim() > 1 else 1
        r = rewards.to(torch.float32).contiguous()
        v = values.to(torch.float32).contiguous()
        d = dones.to(torch.uint8).contiguous()
        lv = last_value.to(torch.float32).contiguous()
        adv, ret = torch.empty_like(r), torch.empty_like(r)
        p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)
        h = torch.cuda.current_stream(r.device).cuda_stream
        rc = abi.load().stp_gae(p(r), p(v), p(d), p(lv), T, N, C.c_float(gamma), C.c_float(lam), p(adv), p(ret),
                                p(stats), C.c_void_p(h if h else 1))
        if rc != abi.STP_OK:
            raise RuntimeError(f"stp_gae failed ({rc}): {abi.last_error()}")
        return adv.to(rewards.dtype), ret.to(rewards.dtype)
    adv = torch.zeros_like(rewards)
    last = torch.zeros_like(rewards[0])
    for t in reversed(range(T)):
        nv = last_value if t == T - 1 else values[t + 1]
        nonterm = 1.0 - dones[t].to(rewards.dtype)
        delta = rewards[t] + gamma * nv * nonterm - values[t]
        last = delta + gamma * lam * nonterm * last
        adv[t] = last
    return adv, adv + values


class _MinibatchStep:
    """The GPU minibatch gradient of ppo_update: gather the minibatch's
    observations, both MLPs' explicit forward, the loss head with its output
    gradients (stp_ppo_surrogate, the rollout columns read through idx), both
    explicit backwards — every parameter's .grad written in place.  It reads
    only static buffers (the update's rollout columns are copied in once per
    update), so it is captured as one CUDA graph per shape and replayed per
    minibatch (~40 launches -> one graph launch; STP_LEARNER_GRAPH=0 runs it
    eagerly)."""

    def __init__(self, model: ActorCritic, cfg: PPOConfig, B: int, mb: int, O: int, A: int, dev):
        self.model, self.cfg, self.mb = model, cfg, mb
        f32 = dict(dtype=torch.float32, device=dev)
        self.xw = torch.empty(B, O, **f32)
        self.act = torch.empty(B, A, **f32)
        self.old = torch.empty(B, **f32)
        self.adv = torch.empty(B, **f32)
        self.ret = torch.empty(B, **f32)
        self.stats = torch.empty(3, dtype=torch.float64, device=dev)
        # one minibatch per epoch (the C5 config): the whole batch in row order —
        # a permutation would change only the summation order of the gradient
        self.full = mb == B
        self.idx = torch.empty(mb, dtype=torch.int64, device=dev)
        self.bad = torch.zeros((), **f32)
        self.scratch = torch.empty(592 * max(model.hidden), **f32)
        self.graph, self.loss, self.captures = None, None, 0
        self.use_graph = os.environ.get("STP_LEARNER_GRAPH", "1") != "0"
        self.key = self._key()

    def _key(self):
        return (tuple(p.data_ptr() for p in self.model.parameters()),
                tuple(p.grad.data_ptr() for p in self.model.parameters()), self.cfg.matmul, self.cfg.clip,
                self.cfg.vf_coef)

    def load(self, xw, act, old, adv, ret, stats):
        self.xw.copy_(xw)
        self.act.copy_(act)
        self.old.copy_(old)
        self.adv.copy_(adv)
        self.ret.copy_(ret)
        self.stats.copy_(stats)
        self.bad.zero_()

    def _body(self):
        m, cfg = self.model, self.cfg
        x = self.xw if self.full else self.xw.index_select(0, self.idx)  # the minibatch's observations
        idx = None if self.full else self.idx
        pi_l, v_l = m.pi.layers, m.v.layers
        a_pi, a_v = mlp_forward(pi_l, x), mlp_forward(v_l, x)
        dmu, dv, dls, loss = surrogate_grad(a_pi[-1], m.log_std.detach(), a_v[-1].view(-1), self.act, self.old,
                                            self.adv, self.ret, idx, self.stats, cfg.clip, cfg.vf_coef,
                                            self.bad, d_mu_bias=pi_l[-1].bias.grad, d_value_bias=v_l[-1].bias.grad)
        m.log_std.grad.copy_(dls)
        mlp_backward(pi_l, a_pi, dmu, self.scratch)
        mlp_backward(v_l, a_v, dv.view(-1, 1), self.scratch)
        return loss

    def run(self, idx):
        if not self.full:
            self.idx.copy_(idx)
        if not self.use_graph:
            return self._body()
        if self.graph is None:
            # warm-up on a side stream (cuBLAS handles / workspaces), then capture;
            # the warm-up computes this same minibatch, so its flag contribution
            # is the replay's
            side = torch.cuda.Stream(device=self.idx.device)
            side.wait_stream(torch.cuda.current_stream(self.idx.device))
            with torch.cuda.stream(side):
                self._body()
            torch.cuda.current_stream(self.idx.device).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.loss = self._body()
            self.graph = g
            self.captures += 1
        self.graph.replay()
        return self.loss


class PPOLearner:
    def __init__(self, model: ActorCritic, cfg: PPOConfig):
        self.model, self.cfg = model, cfg
        # one fused multi-tensor Adam kernel per step on the GPU (SPEC.md:488-496:
        # beta 0.9 / 0.999, eps 1e-8, bias correction)
        cuda = next(model.parameters()).is_cuda
        self.opt = torch.optim.Adam(model.parameters(), lr=cfg.lr, fused=cuda)
        self._mbs = {}
        broadcast_params(model)

    def _minibatch_step(self, B, mb, xw, actions, old_logp, adv, ret, stats):
        """The (cached) captured minibatch step for this shape, loaded with this
        update's rollout columns."""
        key = (B, mb, xw.shape[1], actions.shape[1], xw.device)
        st = self._mbs.get(key)
        if st is None or st.key != st._key():
            st = _MinibatchStep(self.model, self.cfg, B, mb, xw.shape[1], actions.shape[1], xw.device)
            self._mbs = {key: st}  # one shape at a time: drop graphs of older shapes
        st.load(xw, actions, old_logp, adv, ret, stats)
        return st

    def update(self, xw, actions, old_logp=None, adv=None, ret=None, generator: torch.Generator | None = None,
               adv_stats: torch.Tensor | None = None):
        """ppo_update on the whitened batch xw [B, O] of this
        rank (time x agents flattened).  The old policy is snapshotted on the
        same whitened batch before the first epoch (its log-probs, not the
        rollout's, which were taken under the previous observation statistics);
        clipped-surrogate + value epochs over shuffled minibatches with every
        gradient averaged across ranks; then KL(old || new) of the diagonal
        Gaussians, averaged over states and ranks, adapts the learning rate
        once (adapt_learning_rate, :468-475).  A non-finite loss restores the
        snapshot, halves the learning rate and reports `aborted`: the check is
        one device flag read once after the epochs (no host synchronisation per
        minibatch) — the steps after a non-finite loss are discarded with the
        restore, so the outcome equals aborting at the first one."""
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = self.cfg.matmul == "tf32"
        try:
            return self._update(xw, actions, adv, ret, generator, adv_stats)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    def _update(self, xw, actions, adv, ret, generator, adv_stats):
        cfg = self.cfg
        fused = xw.is_cuda
        if fused:  # the kernel normalises on the fly with the global statistics
            adv_raw = adv.to(torch.float32).contiguous()
            adv_stats_g = global_stats(adv_raw, adv_stats)
            actions = actions.to(torch.float32).contiguous()
            ret = ret.to(torch.float32).contiguous()
            # every .grad a view of one flat buffer, written in place by the
            # explicit backward and averaged across ranks in place
            params = list(self.model.parameters())
            # 128-byte aligned views: cuBLAS writes the weight gradients in place
            # and the fused Adam reads them vectorised (unaligned views cost
            # 1.7 ms per update)
            offs = np.cumsum([0] + [(q.numel() + 31) // 32 * 32 for q in params])
            total = int(offs[-1])
            flat = getattr(self, "_flat_grad", None)
            if os.environ.get("STP_FLAT_GRAD", "1") == "0":
                for p_ in params:
                    if p_.grad is None or p_.grad._base is not None:
                        p_.grad = torch.zeros_like(p_)
                flat = self._flat_grad = None
            elif (flat is None or flat.numel() != total or flat.device != xw.device or
                    any(p_.grad is None or p_.grad.data_ptr() != flat[int(o):].data_ptr()
                        for p_, o in zip(params, offs))):
                flat = torch.zeros(total, dtype=torch.float32, device=xw.device)
                for p_, o in zip(params, offs):
                    p_.grad = flat[int(o):int(o) + p_.numel()].view_as(p_)
                self._flat_grad = flat
        else:
            adv = global_normalize(adv, adv_stats)
        B = xw.shape[0]
        with torch.no_grad():
            mu_old = self.model.pi(xw)
            ls_old = self.model.log_std.detach().clone()
            old_logp = gaussian_logp(actions, mu_old, ls_old).contiguous()
            snapshot = [p.detach().clone() for p in self.model.parameters()]
            opt_state = copy.deepcopy(self.opt.state_dict())
        # Table 4: frames per iteration / minibatch size per agent = minibatches per epoch
        n_mb = max(1, cfg.frames_per_iter // max(1, cfg.minibatch_per_agent))
        mb = max(1, B // n_mb)
        lr = self.opt.param_groups[0]["lr"]
        loss = torch.zeros((), device=xw.device)
        bad = torch.zeros((), device=xw.device, dtype=torch.float32)  # 1 once any loss was not finite
        if fused:
            mbg = self._minibatch_step(B, mb, xw, actions, old_logp, adv_raw, ret, adv_stats_g)
            bad = mbg.bad
        for epoch in range(cfg.epochs):
            if fused and mbg.full:  # one minibatch = the whole batch: no permutation to draw
                perm = None
            elif generator is None and xw.is_cuda:  # drawn on the device: no host round trip
                perm = torch.randperm(B, device=xw.device)
            else:  # an explicit (CPU) generator: reproducible permutations (tests)
                perm = torch.randperm(B, generator=generator, device="cpu").to(xw.device)
            for s0 in range(0, B, mb):
                idx = perm[s0:s0 + mb] if perm is not None else None
                if not fused:
                    x = xw.index_select(0, idx)
                    self.opt.zero_grad(set_to_none=False)
                if fused:
                    loss = mbg.run(idx)
                else:
                    logp = self.model.log_prob(x, actions[idx])
                    ratio = torch.exp(logp - old_logp[idx])
                    a = adv[idx]
                    pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg.clip, 1 + cfg.clip) * a).mean()
                    v = self.model.v(x).squeeze(-1)
                    vf = ((v - ret[idx]) ** 2).mean()
                    loss = pg + cfg.vf_coef * vf
                    bad = torch.maximum(bad, (~torch.isfinite(loss)).to(bad.dtype))
                    loss.backward()
                allreduce_mean_grads(self.model, flat if fused else None)
                self.opt.step()
        if _dist():
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if bad.item() > 0:  # abort: restore the snapshot, halve the learning rate
            with torch.no_grad():
                for p_, s_ in zip(self.model.parameters(), snapshot):
                    p_.copy_(s_)
            self.opt.load_state_dict(opt_state)
            lr = max(lr / 2.0, 1e-6)
            for g in self.opt.param_groups:
                g["lr"] = lr
            return {"kl": 0.0, "lr": lr, "loss": float("nan"), "aborted": True}
        with torch.no_grad():
            if fused:
                kl = policy_kl(mu_old, ls_old, self.model.pi(xw), self.model.log_std.detach())
            else:
                kl = gaussian_kl(mu_old, ls_old, self.model.pi(xw), self.model.log_std).mean()
            if _dist():
                dist.all_reduce(kl, op=dist.ReduceOp.SUM)
                kl /= dist.get_world_size()
            lr = adapt_learning_rate(lr, float(kl), cfg.desired_kl)
            for g in self.opt.param_groups:
                g["lr"] = lr
        return {"kl": float(kl), "lr": lr, "loss": float(loss.detach()), "aborted": False}


def adapt_learning_rate(lr: float, measured_kl: float, desired_kl: float) -> float:
    """adapt_learning_rate: /1.5 above 2x the target KL, x1.5
    below half of it, clamped to [1e-6, 1e-2]."""
    if measured_kl > 2.0 * desired_kl:
        lr = lr / 1.5
    elif measured_kl < 0.5 * desired_kl:
        lr = lr * 1.5
    return min(max(lr, 1e-6), 1e-2)


def gaussian_logp(actions, mu, log_std):
    """log N(actions; mu, exp(log_std)^2) summed over action dims."""
    return (-0.5 * ((actions - mu) / torch.exp(log_std)) ** 2 - log_std - 0.5 * math.log(2 * math.pi)).sum(-1)


def policy_kl(mu0, ls0, mu1, ls1) -> torch.Tensor:
    """Mean KL(old || new) over the batch on the GPU (stp_ppo_kl; a device
    scalar, deterministic)."""
    import ctypes as C
    from . import abi
    B, A = mu0.shape
    dev = mu0.device
    t = [x.to(torch.float32).contiguous() for x in (mu0, ls0, mu1, ls1)]
    out = torch.empty((), dtype=torch.float32, device=dev)
    scratch = torch.empty(max(1, (B + 255) // 256), dtype=torch.float64, device=dev)
    h = torch.cuda.current_stream(dev).cuda_stream
    rc = abi.load().stp_ppo_kl(*[C.c_void_p(x.data_ptr()) for x in t], B, A, C.c_void_p(out.data_ptr()),
                               C.c_void_p(scratch.data_ptr()), C.c_void_p(h if h else 1))
    if rc != abi.STP_OK:
        raise RuntimeError(f"stp_ppo_kl failed ({rc}): {abi.last_error()}")
    return out


def gaussian_kl(mu0, ls0, mu1, ls1):
    """KL(N0 || N1) of diagonal Gaussians per state (kl_diag_gaussian)."""
    v0, v1 = torch.exp(2 * ls0), torch.exp(2 * ls1)
    return (ls1 - ls0 + (v0 + (mu0 - mu1) ** 2) / (2 * v1) - 0.5).sum(-1)


def rollout(env, kernel, obs_stat: RunningStat, frames: int, seed: int, step0: int, env_offset: int = 0):
    """Collect `frames` env steps for every agent of this rank on the GPU.
    Returns [T, N] tensors and the raw observations (for the RunningStat)."""
    dev = torch.device("cuda", env.device)
    obs = getattr(env, "last_obs", None)
    if obs is None:  # first rollout of a fresh env (train.py resets once and sets last_obs)
        obs = env.reset()
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
