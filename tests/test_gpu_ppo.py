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


@pytest.mark.parametrize("matmul,mb_per_agent", [("fp32", 16), ("tf32", 16), ("fp32", 32)])
def test_ppo_update_matches_fp64_restatement(matmul, mb_per_agent):
    """mb_per_agent 16: 2 shuffled minibatches per epoch; 32: one minibatch =
    the whole batch (the C5 config), which the GPU learner takes in row order."""
    torch.manual_seed(0)
    O, A, B = 76, 21, 512
    model = ActorCritic(O, A).cuda()
    params0 = {k: v.detach().cpu().double() for k, v in model.named_parameters()}
    cfg = PPOConfig(frames_per_iter=32, epochs=4, minibatch_per_agent=mb_per_agent, lr=3e-4, matmul=matmul)
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


@pytest.mark.parametrize("mb,A,use_idx", [(1000, 21, True), (257, 8, False), (4096, 17, True), (1, 3, True)])
def test_ppo_surrogate_kernel_matches_autograd_fp64(mb, A, use_idx):
    """stp_ppo_surrogate (the learner's loss head) against autograd of the
    same loss in float64 on the fp32 inputs: ratios inside and outside the
    clip range, advantages of both signs, exact ties (ratio 1).  Bounds: loss
    terms 1e-5 relative; d/dmu, d/dV elementwise 1e-5 of the largest entry;
    d/dlog_std 1e-5 relative (fixed-order double reductions)."""
    from paper_1810_05762_b200.ppo import surrogate_grad
    g = torch.Generator().manual_seed(mb * 7 + A)
    Bfull = mb + 37
    f = lambda *s, sc=1.0: (torch.randn(*s, generator=g) * sc).float()
    actions, mu_full = f(Bfull, A), f(Bfull, A, sc=0.5)
    log_std = f(A, sc=0.3) - 0.5
    value, ret = f(mb), f(Bfull, sc=2.0)
    adv = f(Bfull, sc=3.0) + 0.4
    idx = torch.randperm(Bfull, generator=g)[:mb] if use_idx else torch.arange(mb)
    mu = mu_full[idx]
    # old log-probs: the current ones shifted so ratios land on both sides of the clip range; some exact ties
    lp_now = (-0.5 * ((actions[idx] - mu) / torch.exp(log_std)) ** 2 - log_std - 0.5 * math.log(2 * math.pi)).sum(-1)
    old = torch.empty(Bfull)
    old[idx] = lp_now + (torch.rand(mb, generator=g) - 0.5) * 0.8
    old[idx[: mb // 10]] = lp_now[: mb // 10]  # ratio ~1
    stats = torch.tensor([float(Bfull), adv.double().sum().item(), (adv.double() ** 2).sum().item()],
                         dtype=torch.float64)
    clip, vf_coef = 0.2, 0.5
    cu = lambda t: t.cuda()
    bad = torch.zeros((), device="cuda")
    dmu, dv, dls, loss = surrogate_grad(cu(mu), cu(log_std), cu(value), cu(actions), cu(old), cu(adv), cu(ret),
                                        cu(idx) if use_idx else cu(torch.arange(mb)), cu(stats), clip, vf_coef, bad)
    # fp64 autograd of the same loss
    M, LS, V = (t.double().requires_grad_(True) for t in (mu, log_std, value))
    n, sm, sq = stats
    mean = sm / n
    an = (adv.double() - mean) / (torch.sqrt(torch.clamp(sq / n - mean * mean, min=0)) + 1e-8)
    k = idx
    lp = (-0.5 * ((actions[k].double() - M) / torch.exp(LS)) ** 2 - LS - 0.5 * math.log(2 * math.pi)).sum(-1)
    r = torch.exp(lp - old[k].double())
    a = an[k]
    pg = -torch.min(r * a, torch.clamp(r, 1 - clip, 1 + clip) * a).mean()
    vf = ((V - ret[k].double()) ** 2).mean()
    L = pg + vf_coef * vf
    gM, gLS, gV = torch.autograd.grad(L, [M, LS, V])
    assert float(bad) == 0.0
    assert abs(float(loss) - float(L)) <= 1e-5 * (1 + abs(float(L)))
    tol = lambda ref: 5e-5 * float(ref.abs().max()) + 1e-12
    # samples whose ratio sits within fp32 rounding of a clip bound may legitimately take the other branch
    rr = r.detach()
    edge = ((rr - (1 - clip)).abs() < 1e-5) | ((rr - (1 + clip)).abs() < 1e-5)
    keep = ~edge
    assert (dmu.cpu().double()[keep] - gM[keep]).abs().max() <= tol(gM)
    assert (dv.cpu().double() - gV).abs().max() <= tol(gV)
    if not bool(edge.any()):
        assert (dls.cpu().double() - gLS).abs().max() <= 1e-5 * (float(gLS.abs().max()) + 1e-12)


def test_ppo_surrogate_flags_non_finite_loss():
    from paper_1810_05762_b200.ppo import surrogate_grad
    mb, A = 64, 4
    z = lambda *s: torch.zeros(*s, device="cuda")
    mu = z(mb, A)
    mu[3, 1] = float("nan")
    bad = torch.zeros((), device="cuda")
    stats = torch.tensor([float(mb), 0.0, float(mb)], dtype=torch.float64, device="cuda")
    surrogate_grad(mu, z(A), z(mb), z(mb, A), z(mb), torch.ones(mb, device="cuda"), z(mb),
                   torch.arange(mb, device="cuda"), stats, 0.2, 0.5, bad)
    assert float(bad) == 1.0


@pytest.mark.parametrize("rows,H", [(131072 // 64, 256), (1000, 128), (513, 64), (7, 32), (0, 64)])
def test_selu_backward_bias_kernel(rows, H):
    """stp_selu_backward_bias against torch's SELU backward (result form) and
    the column sum; bounds 1e-6 relative (fp32, fixed-order sums)."""
    import ctypes as C
    from paper_1810_05762_b200 import abi
    g = torch.Generator().manual_seed(rows + H)
    z = torch.randn(rows, H, generator=g).cuda()
    y = torch.selu(z)
    dy = torch.randn(rows, H, generator=g).cuda()
    ref = torch.where(y > 0, dy * 1.0507009873554805, dy * (y + 1.0507009873554805 * 1.6732632423543772))
    gx = dy.clone()
    db = torch.full((H,), float("nan"), device="cuda")
    scratch = torch.empty(592 * H, device="cuda")
    rc = abi.load().stp_selu_backward_bias(C.c_void_p(gx.data_ptr()), C.c_void_p(y.data_ptr()), rows, H,
                                           C.c_void_p(db.data_ptr()), C.c_void_p(scratch.data_ptr()), C.c_void_p(1))
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.allclose(gx, ref, rtol=1e-6, atol=0)
    colsum = ref.double().sum(0)
    assert (db.double() - colsum).abs().max() <= 1e-5 * (1 + colsum.abs().max())


def test_explicit_learner_backward_matches_autograd():
    """The learner's explicit minibatch gradient (mlp_forward, stp_ppo_surrogate,
    mlp_backward: every parameter's .grad written by GEMMs / kernels) equals
    autograd of the same fp32 loss; bound 1e-4 of each tensor's largest entry."""
    from paper_1810_05762_b200.ppo import mlp_backward, mlp_forward, surrogate_grad
    torch.manual_seed(1)
    O, A, mb = 77, 21, 3000
    model = ActorCritic(O, A).cuda()
    x = torch.randn(mb + 11, O, device="cuda")
    act = torch.randn(mb + 11, A, device="cuda") * 0.5
    adv = torch.randn(mb + 11, device="cuda")
    ret = torch.randn(mb + 11, device="cuda")
    idx = torch.randperm(mb + 11, device="cuda")[:mb]
    with torch.no_grad():
        old = (-0.5 * ((act - model.pi(x)) / torch.exp(model.log_std)) ** 2 - model.log_std
               - 0.5 * math.log(2 * math.pi)).sum(-1) + 0.1 * torch.randn(mb + 11, device="cuda")
    stats = torch.stack([torch.tensor(float(mb + 11), dtype=torch.float64, device="cuda"), adv.double().sum(),
                         (adv.double() ** 2).sum()])
    # autograd reference
    n, sm, sq = stats
    an = ((adv.double() - sm / n) / (torch.sqrt(sq / n - (sm / n) ** 2) + 1e-8)).float()
    xi = x[idx]
    lp = model.log_prob(xi, act[idx])
    r = torch.exp(lp - old[idx])
    pg = -torch.min(r * an[idx], torch.clamp(r, 0.8, 1.2) * an[idx]).mean()
    L = pg + 0.5 * ((model.v(xi).squeeze(-1) - ret[idx]) ** 2).mean()
    ref = torch.autograd.grad(L, list(model.parameters()))
    for p in model.parameters():
        p.grad = torch.full_like(p, float("nan"))
    bad = torch.zeros((), device="cuda")
    pi_l, v_l = model.pi.layers, model.v.layers
    a_pi, a_v = mlp_forward(pi_l, xi), mlp_forward(v_l, xi)
    dmu, dv, dls, loss = surrogate_grad(a_pi[-1], model.log_std.detach(), a_v[-1].view(-1), act, old, adv, ret, idx,
                                        stats, 0.2, 0.5, bad, d_mu_bias=pi_l[-1].bias.grad,
                                        d_value_bias=v_l[-1].bias.grad)
    model.log_std.grad.copy_(dls)
    scratch = torch.empty(592 * 256, device="cuda")
    mlp_backward(pi_l, a_pi, dmu, scratch)
    mlp_backward(v_l, a_v, dv.view(-1, 1), scratch)
    torch.cuda.synchronize()
    assert abs(float(loss) - float(L)) <= 1e-5 * (1 + abs(float(L)))
    for (name, p), gref in zip(model.named_parameters(), ref):
        err = float((p.grad - gref).abs().max())
        assert err <= 1e-4 * float(gref.abs().max()) + 1e-9, (name, err)


@pytest.mark.parametrize("rows,H,selu", [(4099, 256, 1), (100, 64, 1), (33, 32, 0), (0, 128, 1)])
def test_bias_selu_kernel(rows, H, selu):
    """stp_bias_selu (the learner's forward epilogue) against torch.selu(z + b): 2 ulp-level (rtol 1e-6)."""
    import ctypes as C
    from paper_1810_05762_b200 import abi
    g = torch.Generator().manual_seed(rows * 3 + H)
    z = (torch.randn(rows, H, generator=g) * 3).cuda()
    b = torch.randn(H, generator=g).cuda()
    ref = torch.selu(z + b) if selu else z + b
    out = z.clone()
    rc = abi.load().stp_bias_selu(C.c_void_p(out.data_ptr()), C.c_void_p(b.data_ptr()), rows, H, selu, C.c_void_p(1))
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.allclose(out, ref, rtol=1e-6, atol=1e-7)


def test_captured_minibatch_step_equals_eager(monkeypatch):
    """The learner's minibatch step replayed from its CUDA graph gives the same
    update as the eager launches (same kernels, same GEMM calls): parameters
    after a 4-epoch, 2-minibatch update agree to 1e-6 of each tensor's scale,
    and a second update (graph reused with new rollout columns) too."""
    import copy as _copy
    torch.manual_seed(3)
    O, A, B = 77, 21, 4096
    base = ActorCritic(O, A).cuda()
    cfg = PPOConfig(frames_per_iter=8, epochs=4, minibatch_per_agent=4)
    results = []
    for flag in ("0", "1"):
        monkeypatch.setenv("STP_LEARNER_GRAPH", flag)
        model = _copy.deepcopy(base)
        learner = PPOLearner(model, cfg)
        stats = []
        for it in range(2):
            g = torch.Generator().manual_seed(10 + it)
            xw = torch.randn(B, O, generator=g).cuda()
            act = torch.randn(B, A, generator=g).cuda()
            adv = torch.randn(B, generator=g).cuda()
            ret = torch.randn(B, generator=g).cuda()
            stats.append(learner.update(xw, act, None, adv, ret, generator=torch.Generator().manual_seed(it)))
        assert isinstance(learner._mbs[next(iter(learner._mbs))].graph, torch.cuda.CUDAGraph) == (flag == "1")
        results.append(([p.detach().clone() for p in model.parameters()], stats))
    (pe, se), (pg, sg) = results
    for a, b in zip(pe, pg):
        assert (a - b).abs().max() <= 1e-6 * (a.abs().max() + 1e-12)
    for a, b in zip(se, sg):
        assert abs(a["kl"] - b["kl"]) <= 1e-5 * (abs(a["kl"]) + 1e-12) and a["lr"] == b["lr"]


@pytest.mark.parametrize("B,A", [(4096, 21), (300, 8), (1, 3)])
def test_ppo_kl_kernel(B, A):
    """stp_ppo_kl against the fp64 KL of diagonal Gaussians: 1e-5 relative."""
    from paper_1810_05762_b200.ppo import gaussian_kl, policy_kl
    g = torch.Generator().manual_seed(B + A)
    mu0, mu1 = torch.randn(B, A, generator=g), torch.randn(B, A, generator=g) * 0.1
    mu1 = mu0 + mu1
    ls0, ls1 = torch.randn(A, generator=g) * 0.2 - 0.5, torch.randn(A, generator=g) * 0.2 - 0.5
    ref = float(gaussian_kl(mu0.double(), ls0.double(), mu1.double(), ls1.double()).mean())
    got = float(policy_kl(mu0.cuda(), ls0.cuda(), mu1.cuda(), ls1.cuda()))
    assert abs(got - ref) <= 1e-5 * abs(ref) + 1e-7
