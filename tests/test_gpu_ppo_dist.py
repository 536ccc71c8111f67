"""The GPU learner's distributed logic (config C5) on the
fused path: two ranks on one device, gloo (host transport, so no rank's
kernels wait on the other's).  Global advantage statistics, per-minibatch
gradient averaging, the KL average and the parameter broadcast must keep both
ranks identical and equal one process updating on the union of the shards
(one full-batch minibatch per epoch, equal shards: the average of the rank
means is the union mean).  Bound: 1e-5 of each parameter's scale (different
summation order), ranks bit-identical."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_05762_b200.policy import ActorCritic
from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner

pytestmark = pytest.mark.gpu

B, O, A = 512, 20, 6


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    g = torch.Generator().manual_seed(3)
    xw = torch.randn(2 * B, O, generator=g)
    act = torch.randn(2 * B, A, generator=g) * 0.5
    adv = torch.randn(2 * B, generator=g) + 0.2
    ret = torch.randn(2 * B, generator=g)
    return xw, act, adv, ret


def _cfg():
    return PPOConfig(frames_per_iter=1, epochs=3, minibatch_per_agent=1, lr=1e-3)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(1000 + rank)  # different init per rank: the broadcast must fix it
    model = ActorCritic(O, A, hidden=(16, 16, 8)).cuda()
    learner = PPOLearner(model, _cfg())
    xw, act, adv, ret = _data()
    sl = slice(rank * B, (rank + 1) * B)
    st = learner.update(xw[sl].cuda(), act[sl].cuda(), None, adv[sl].cuda(), ret[sl].cuda())
    flat = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).cpu()
    gathered = [torch.zeros_like(flat) for _ in range(world)]
    dist.all_gather(gathered, flat)
    if rank == 0:
        q.put((torch.stack(gathered).numpy(), st["kl"], st["lr"]))
    dist.barrier()
    dist.destroy_process_group()


def test_gpu_learner_two_ranks_match_union():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    params, kl2, lr2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(params[0], params[1])  # ranks identical
    torch.manual_seed(1000)  # rank 0's init is what the broadcast distributed
    model = ActorCritic(O, A, hidden=(16, 16, 8)).cuda()
    learner = PPOLearner(model, _cfg())
    xw, act, adv, ret = _data()
    st = learner.update(xw.cuda(), act.cuda(), None, adv.cuda(), ret.cuda())
    off = 0
    for p in model.parameters():
        n = p.numel()
        ref = p.detach().reshape(-1).cpu().numpy()
        got = params[0][off:off + n]
        assert np.abs(got - ref).max() <= 1e-5 * (np.abs(ref).max() + 1e-12)
        off += n
    assert abs(kl2 - st["kl"]) <= 1e-4 * abs(st["kl"]) + 1e-9
    assert lr2 == st["lr"]
