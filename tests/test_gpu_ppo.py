"""Config C5 learner data path on the GPU:
the GAE kernel (stp_gae) against the SPEC's brute-force O(T^2) estimator
 in fp64, and one PPO update (ppo_update, SPEC.md:455-475:
clipped surrogate + value MSE, Adam, KL-adaptive learning rate) on the GPU in
fp32 against an independent fp64 CPU restatement written here (explicit SELU
MLP, autograd-exact gradients in float64, textbook Adam).

Stated bounds: GAE |err| <= 1e-5 (1 + |A|) (fp32 recursion over T = 32);
update: relative parameter-step error ||d32 - d64|| / ||d64|| <= 1e-3 per
tensor (observed 2.7e-5 on B200; Adam's g / sqrt(v) normalisation amplifies
rounding of near-zero gradient components), KL / loss within 1e-3 relative,
the same learning rate."""
import math

import numpy as np
import pytest
import torch

from paper_1810_05762_b200.policy import ActorCritic
from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner, adapt_learning_rate, gae

pytestmark = pytest.mark.gpu


def _gae_brute(r, v, d, lv, gamma, lam):
    """O(T^2) oracle: A_t = sum_k (gamma lam)^k delta_{t+k}, the sum and the
    bootstrap cut at the first episode end (done), fp64."""
    T, N = r.shape
    vn = np.concatenate([v[1:], lv[None]], 0)
    delta = r + gamma * vn * (1 - d) - v
    A = np.zeros((T, N))
    for t in range(T):
        for n in range(N):
            acc, w = 0.0, 1.0
            for k in range(t, T):
                acc += w * delta[k, n]
                if d[k, n]:
                    break
                w *= gamma * lam
            A[t, n] = acc
    return A, A + v


@pytest.mark.parametrize("gamma,lam", [(0.99, 0.95), (0.99, 0.0), (1.0, 1.0)])
def test_gae_kernel_matches_brute_force(gamma, lam):
    rng = np.random.default_rng(3)
    T, N = 32, 333
    r = rng.normal(size=(T, N))
    v = rng.normal(size=(T, N))
    d = (rng.uniform(size=(T, N)) < 0.05).astype(np.uint8)
    lv = rng.normal(size=N)
    A, R = _gae_brute(r, v, d, lv, gamma, lam)
    f = lambda x, dt=torch.float32: torch.tensor(x, dtype=dt, device="cuda")
    stats = torch.zeros(3, dtype=torch.float64, device="cuda")
    adv, ret = gae(f(r), f(v), f(d, torch.uint8), f(lv), gamma, lam, stats=stats)
    adv, ret = adv.cpu().numpy(), ret.cpu().numpy()
    # fp32 inputs / arithmetic: compare with the oracle on the same fp32-rounded inputs
    A32, R32 = _gae_brute(r.astype(np.float32).astype(np.float64), v.astype(np.float32).astype(np.float64), d,
                          lv.astype(np.float32).astype(np.float64), gamma, lam)
    assert np.abs(adv - A32).max() <= 1e-5 * (1 + np.abs(A32).max())
    assert np.abs(ret - R32).max() <= 1e-5 * (1 + np.abs(R32).max())
    s = stats.cpu().numpy()
    assert s[0] == T * N
    assert abs(s[1] - adv.astype(np.float64).sum()) <= 1e-6 * (1 + abs(s[1]))
    assert abs(s[2] - (adv.astype(np.float64) ** 2).sum()) <= 1e-6 * s[2]
    if lam == 0.0:  # lambda = 0 -> r + gamma V(s') - V(s)
        vn = np.concatenate([v[1:], lv[None]], 0)
        np.testing.assert_allclose(A, r + gamma * vn * (1 - d) - v, atol=1e-12)


def _selu(x):
    return 1.0507009873554805 * torch.where(x > 0, x, 1.6732632423543772 * (torch.exp(x) - 1))


def _mlp(params, prefix, x, n_layers=4):
    for i in range(n_layers):
        x = x @ params[f"{prefix}.layers.{i}.weight"].T + params[f"{prefix}.layers.{i}.bias"]
        if i < n_layers - 1:
            x = _selu(x)
    return x


def _update_fp64(params, xw, act, adv, ret, cfg, perms):
    """ppo_update restated in float64: old policy snapshot,
    normalised advantages, clipped surrogate + value MSE per minibatch, Adam
    (beta 0.9 / 0.999, eps 1e-8, bias correction), KL(old || new) mean, lr rule."""
    P = {k: v.detach().clone().double().requires_grad_(True) for k, v in params.items()}
    m = {k: torch.zeros_like(v) for k, v in P.items()}
    s = {k: torch.zeros_like(v) for k, v in P.items()}
    adv = (adv - adv.mean()) / (torch.sqrt(torch.clamp((adv * adv).mean() - adv.mean() ** 2, min=0)) + 1e-8)

    def logp(P, x, a):
        mu = _mlp(P, "pi", x)
        ls = P["log_std"]
        return (-0.5 * ((a - mu) / torch.exp(ls)) ** 2 - ls - 0.5 * math.log(2 * math.pi)).sum(-1), mu

    with torch.no_grad():
        old_lp, mu_old = logp(P, xw, act)
        ls_old = P["log_std"].clone()
    B = xw.shape[0]
    n_mb = max(1, cfg.frames_per_iter // max(1, cfg.minibatch_per_agent))
    mb = max(1, B // n_mb)
    step, lr = 0, cfg.lr
    loss = None
    for e in range(cfg.epochs):
        for s0 in range(0, B, mb):
            idx = perms[e][s0:s0 + mb]
            lp, _ = logp(P, xw[idx], act[idx])
            ratio = torch.exp(lp - old_lp[idx])
            a = adv[idx]
            pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg.clip, 1 + cfg.clip) * a).mean()
            v = _mlp(P, "v", xw[idx]).squeeze(-1)
            loss = pg + cfg.vf_coef * ((v - ret[idx]) ** 2).mean()
            grads = torch.autograd.grad(loss, list(P.values()))
            step += 1
            with torch.no_grad():
                for (k, p), g in zip(P.items(), grads):
                    m[k] = 0.9 * m[k] + 0.1 * g
                    s[k] = 0.999 * s[k] + 0.001 * g * g
                    mh, sh = m[k] / (1 - 0.9 ** step), s[k] / (1 - 0.999 ** step)
                    p -= lr * mh / (torch.sqrt(sh) + 1e-8)
    with torch.no_grad():
        _, mu_new = logp(P, xw, act)
        v0, v1 = torch.exp(2 * ls_old), torch.exp(2 * P["log_std"])
        kl = (P["log_std"] - ls_old + (v0 + (mu_old - mu_new) ** 2) / (2 * v1) - 0.5).sum(-1).mean()
    return P, float(kl), float(loss), adapt_learning_rate(lr, float(kl), cfg.desired_kl)


# worst relative parameter-step error, relative KL / loss error vs the fp64
# restatement: IEEE fp32 GEMMs (the default; measured 2.7e-5 / 3e-7 / 1e-7)
# and the opt-in TF32 tensor-core GEMMs (measured 0.137 / 1.4e-2 / 7.4e-4:
# Adam's normalisation amplifies the TF32 rounding of small gradients)
UPDATE_BOUNDS = {"fp32": (1e-3, 1e-3, 1e-3), "tf32": (0.3, 5e-2, 5e-3)}


@pytest.mark.parametrize("matmul", ["fp32", "tf32"])
def test_ppo_update_matches_fp64_restatement(matmul):
    torch.manual_seed(0)
    O, A, B = 76, 21, 512
    model = ActorCritic(O, A).cuda()
    params0 = {k: v.detach().cpu().double() for k, v in model.named_parameters()}
    cfg = PPOConfig(frames_per_iter=32, epochs=4, minibatch_per_agent=16, lr=3e-4,  # 2 minibatches per epoch
                    matmul=matmul)
    g = torch.Generator().manual_seed(5)
    xw = torch.randn(B, O, generator=g).clamp(-10, 10)
    with torch.no_grad():
        mu = model.pi(xw.cuda()).cpu()
    act = mu + 0.6 * torch.randn(B, A, generator=g)
    adv = torch.randn(B, generator=g) * 2 + 0.3
    ret = torch.randn(B, generator=g)
    learner = PPOLearner(model, cfg)
    gen = torch.Generator().manual_seed(11)
    st = learner.update(xw.cuda(), act.cuda(), None, adv.cuda(), ret.cuda(), generator=gen)
    gen = torch.Generator().manual_seed(11)
    perms = [torch.randperm(B, generator=gen) for _ in range(cfg.epochs)]
    P64, kl64, loss64, lr64 = _update_fp64(params0, xw.double(), act.double(), adv.double(), ret.double(), cfg, perms)
    worst = 0.0
    for k, p in model.named_parameters():
        d32 = p.detach().cpu().double() - params0[k]
        d64 = P64[k].detach() - params0[k]
        rel = float((d32 - d64).norm() / max(d64.norm(), 1e-12))
        worst = max(worst, rel)
    print(f"update: KL {st['kl']:.6e} vs {kl64:.6e}, loss {st['loss']:.6e} vs {loss64:.6e}, "
          f"worst relative parameter-step error {worst:.2e}")
    b_step, b_kl, b_loss = UPDATE_BOUNDS[matmul]
    assert not st["aborted"]
    assert worst <= b_step
    assert abs(st["kl"] - kl64) <= b_kl * max(abs(kl64), 1e-6)
    assert abs(st["loss"] - loss64) <= b_loss * max(abs(loss64), 1e-6)
    assert st["lr"] == lr64


def test_ppo_update_aborts_on_non_finite_loss():
    """a non-finite loss restores the snapshot and halves the
    learning rate (checked once after the epochs, no per-minibatch sync)."""
    torch.manual_seed(1)
    model = ActorCritic(12, 4, (16, 16, 8)).cuda()
    learner = PPOLearner(model, PPOConfig(frames_per_iter=32, epochs=3, minibatch_per_agent=16, lr=1e-3))
    before = [p.detach().clone() for p in model.parameters()]
    ret = torch.zeros(64, device="cuda")
    ret[5] = float("nan")
    st = learner.update(torch.randn(64, 12, device="cuda"), torch.randn(64, 4, device="cuda"), None,
                        torch.randn(64, device="cuda"), ret)
    assert st["aborted"] and st["lr"] == 5e-4
    for p, q in zip(model.parameters(), before):
        assert torch.equal(p.detach(), q)
