"""K4 (tcgen05 policy forward) against the plain PyTorch fp32 reference of the
same op.  Tolerance: bf16 operands with fp32 accumulation through 4 layers,
|err| <= 0.03 + 0.03 |ref| on the mean and value; the sampled action equals
mean + exp(log_std) * eps with eps restated from the counter-based RNG to 1e-4."""
import numpy as np
import pytest
import torch

from paper_1810_05762_b200.policy import HIDDEN, ActorCritic, PolicyKernel, RunningStat, kernel_noise

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,obs_dim,act_dim,n", [("humanoid", 76, 21, 4096), ("ant", 39, 8, 300), ("hfh", 241, 21, 1000),
                                                    ("humanoid", 76, 21, 77)])
def test_policy_kernel_matches_torch_fp32(name, obs_dim, act_dim, n):
    torch.manual_seed(0)
    dev = torch.device("cuda:0")
    model = ActorCritic(obs_dim, act_dim, HIDDEN[name]).to(dev)
    kern = PolicyKernel(model, dev)
    obs = torch.randn(n, obs_dim, device=dev) * 3 + 1
    stat = RunningStat(obs_dim, device=dev)
    stat.push(obs)
    mean, std = stat.mean.float(), stat.std.float()
    mu, act, logp, val = kern.forward(obs, mean, std, seed=9, step=5)
    torch.cuda.synchronize()
    with torch.no_grad():
        xw = torch.clamp((obs - mean) / std, -10, 10)
        mu_ref, v_ref = model.forward_ref(xw)
    assert (mu - mu_ref).abs().max() <= 0.03 + 0.03 * mu_ref.abs().max()
    assert ((mu - mu_ref).abs() <= 0.03 + 0.03 * mu_ref.abs()).all()
    assert ((val - v_ref).abs() <= 0.03 + 0.03 * v_ref.abs()).all()
    sd = torch.exp(model.log_std.detach())
    for e in [0, 1, n // 2, n - 1]:
        eps = torch.from_numpy(kernel_noise(9, e, 5, act_dim)).to(dev)
        np.testing.assert_allclose((mu[e] + sd * eps).cpu().numpy(), act[e].cpu().numpy(), rtol=1e-4, atol=1e-4)
    lp_ref = model.log_prob(xw, act).detach()
    # log-prob of the sample under the kernel's own mean
    assert (logp - lp_ref).abs().max() <= 0.05 + 0.05 * lp_ref.abs().max()


def test_train_loop_runs(capsys):
    """Config C5 on one GPU (paper_1810_05762_b200.train): rollout on the fused
    step kernel + tcgen05 policy forward, GAE, whitening, PPO update; every
    iteration finite, not aborted, KL >= 0."""
    import json
    from paper_1810_05762_b200 import train
    train.main(["--iters", "2", "--envs", "256", "--epochs", "2", "--frames", "8"])
    rows = [json.loads(l) for l in capsys.readouterr().out.splitlines() if l.startswith("{")]
    assert len(rows) == 2
    for r in rows:
        assert not r["aborted"] and r["kl"] >= 0 and np.isfinite(r["loss"]) and np.isfinite(r["mean_reward"])
