"""Config C5 host logic on CPU with gloo (world size 2): gradient allreduce,
global advantage normalisation, observation-statistics merge and parameter
broadcast keep both ranks bit-identical, and equal a single-process update
over the union of the shards."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_05762_b200.policy import ActorCritic, RunningStat
from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner, gae

B, O, A = 64, 12, 4


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(seed=0):
    g = torch.Generator().manual_seed(seed)
    xw = torch.randn(2 * B, O, generator=g)
    act = torch.randn(2 * B, A, generator=g)
    old = torch.randn(2 * B, generator=g) * 0.1 - 5.0
    adv = torch.randn(2 * B, generator=g)
    ret = torch.randn(2 * B, generator=g)
    return xw, act, old, adv, ret


def _cfg():
    # one full-batch minibatch per epoch so the 2-rank gradient average equals the union gradient
    return PPOConfig(frames_per_iter=1, epochs=3, minibatch_per_agent=1, lr=1e-3)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(1000 + rank)  # different init per rank: broadcast must fix it
    model = ActorCritic(O, A, hidden=(16, 16, 8))
    learner = PPOLearner(model, _cfg())
    xw, act, old, adv, ret = _data()
    sl = slice(rank * B, (rank + 1) * B)
    # identity permutation on every epoch keeps ranks comparable to the single run
    gen = torch.Generator().manual_seed(7)
    learner.update(xw[sl], act[sl], old[sl], adv[sl], ret[sl], generator=gen)
    # observation statistics merge
    st_local = RunningStat(O)
    st_local.push(xw[sl] * (rank + 1))
    st = RunningStat(O)
    st.merge_allreduce(st_local)
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
    gathered = [torch.zeros_like(flat) for _ in range(world)]
    dist.all_gather(gathered, flat)
    if rank == 0:
        q.put((torch.stack(gathered).numpy(), st.mean.numpy(), st.std.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_ppo_update_matches_union():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    params, mean2, std2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(params[0], params[1])  # ranks identical
    # single process on the union; rank-0 init is what the broadcast distributed
    torch.manual_seed(1000)
    model = ActorCritic(O, A, hidden=(16, 16, 8))
    learner = PPOLearner(model, _cfg())
    xw, act, old, adv, ret = _data()
    # the union minibatch gradient = mean of the two shard gradients (equal sizes)
    cfg = learner.cfg
    from paper_1810_05762_b200.ppo import gaussian_kl, gaussian_logp, global_normalize
    advn = global_normalize(adv)
    del old  # ppo_update snapshots the old policy on the whitened batch
    with torch.no_grad():
        mu_old, ls_old = model.pi(xw), model.log_std.detach().clone()
        old = gaussian_logp(act, mu_old, ls_old)
    for epoch in range(cfg.epochs):
        grads = None
        for r in range(2):
            sl = slice(r * B, (r + 1) * B)
            logp = model.log_prob(xw[sl], act[sl])
            ratio = torch.exp(logp - old[sl])
            a = advn[sl]
            pg = -torch.min(ratio * a, torch.clamp(ratio, 1 - cfg.clip, 1 + cfg.clip) * a).mean()
            vf = ((model.v(xw[sl]).squeeze(-1) - ret[sl]) ** 2).mean()
            learner.opt.zero_grad(set_to_none=False)
            (pg + cfg.vf_coef * vf).backward()
            g = [p.grad.clone() for p in model.parameters()]
            grads = g if grads is None else [x + y for x, y in zip(grads, g)]
        for p, g in zip(model.parameters(), grads):
            p.grad.copy_(g / 2)
        learner.opt.step()
    with torch.no_grad():  # one learning-rate adaptation after the update (:468-475)
        kl = gaussian_kl(mu_old, ls_old, model.pi(xw), model.log_std).mean()
        assert kl >= 0
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).numpy()
    np.testing.assert_allclose(params[0], flat, rtol=1e-5, atol=1e-6)
    # RunningStat merge == statistics of the concatenated stream
    ref = RunningStat(O)
    ref.push(torch.cat([xw[:B], xw[B:] * 2]))
    np.testing.assert_allclose(mean2, ref.mean.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(std2, ref.std.numpy(), rtol=1e-10)


def test_gae_matches_recursion():
    T, N = 7, 3
    g = torch.Generator().manual_seed(3)
    r, v = torch.randn(T, N, generator=g), torch.randn(T, N, generator=g)
    d = torch.zeros(T, N, dtype=torch.uint8)
    d[3, 1] = 1
    lv = torch.randn(N, generator=g)
    adv, ret = gae(r, v, d, lv, 0.99, 0.95)
    for n in range(N):
        a = 0.0
        for t in reversed(range(T)):
            nv = lv[n] if t == T - 1 else v[t + 1, n]
            nt = 1.0 - float(d[t, n])
            delta = r[t, n] + 0.99 * nv * nt - v[t, n]
            a = delta + 0.99 * 0.95 * nt * a
            assert abs(float(adv[t, n]) - float(a)) < 1e-5


def test_adapt_learning_rate_spec_examples():
    """SPEC.md:471-474 with desired KL 0.01."""
    from paper_1810_05762_b200.ppo import adapt_learning_rate
    assert abs(adapt_learning_rate(3e-4, 0.05, 0.01) - 3e-4 / 1.5) < 1e-15
    assert abs(adapt_learning_rate(3e-4, 0.001, 0.01) - 3e-4 * 1.5) < 1e-15
    assert adapt_learning_rate(3e-4, 0.01, 0.01) == 3e-4
    assert adapt_learning_rate(1e-2, 0.0, 0.01) == 1e-2 and adapt_learning_rate(1e-6, 9.0, 0.01) == 1e-6


def test_zero_advantages_leave_the_policy_unchanged_and_kl_nonnegative():
    """zero advantages -> the policy loss term has zero
    gradient (only the value net moves); the reported KL is >= 0."""
    torch.manual_seed(3)
    model = ActorCritic(O, A, hidden=(16, 16, 8))
    learner = PPOLearner(model, _cfg())
    xw, act, old, adv, ret = _data()
    pi0 = [p.detach().clone() for p in model.pi.parameters()] + [model.log_std.detach().clone()]
    v0 = [p.detach().clone() for p in model.v.parameters()]
    st = learner.update(xw, act, old, torch.zeros_like(adv), ret)
    assert st["kl"] >= 0.0 and not st["aborted"]
    for p, q in zip(list(model.pi.parameters()) + [model.log_std], pi0):
        assert torch.equal(p.detach(), q)
    assert any(not torch.equal(p.detach(), q) for p, q in zip(model.v.parameters(), v0))
