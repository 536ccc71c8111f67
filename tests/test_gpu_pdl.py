"""Programmatic dependent launch (sim_launch.h launch_pdl, K4, the step kernel,
the inter-agent pre-step chain) changes only when grids are scheduled, never
what they compute: a Humanoid rollout (step kernel <-> K4 policy forward, both
launched early behind each other) and an HFH run with inter-agent islands
(reset -> shapes -> env query -> narrow slots -> islands -> step chain) give
bit-identical observations, rewards, dones and actions with STP_PDL=1 (the
default) and STP_PDL=0 (plain launches).  Each setting runs in its own process
(the switch is read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import hashlib, sys, torch
sys.path.insert(0, {root!r})
from paper_1810_05762_b200.policy import ActorCritic, PolicyKernel
from paper_1810_05762_b200.sim import VecEnv
h = hashlib.sha256()
torch.manual_seed(0)
env = VecEnv("humanoid", n_envs=1024, seed=5)
obs = env.reset()
kern = PolicyKernel(ActorCritic(env.obs_dim, env.action_dim).to("cuda"), "cuda:0")
m, s = torch.zeros(env.obs_dim, device="cuda"), torch.ones(env.obs_dim, device="cuda")
for t in range(40):
    mu, act, logp, val = kern.forward(obs, m, s, seed=3, step=t)
    obs, rew, done = env.step(act)
    for x in (act, logp, val, obs, rew, done):
        h.update(x.cpu().numpy().tobytes())
hfh = VecEnv("hfh", n_envs=256, seed=9)
hfh.reset()
for t in range(120):
    o, r, d = hfh.step(hfh.random_actions(t))
    for x in (o, r, d):
        h.update(x.cpu().numpy().tobytes())
h.update(hfh.get_state().tobytes())
print("HASH", h.hexdigest())
'''


def _run(pdl):
    env = dict(os.environ, STP_PDL=str(pdl))
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT)], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.startswith("HASH")][0]


def test_pdl_does_not_change_results():
    assert _run(1) == _run(0)
