"""The multi-GPU data path through the CUDA kernels: two
ranks (gloo, world size 2) each own a handle of 2048 Humanoid envs with
env_offset = rank * 2048 and step them on their own stream with no data-path
collective; the gathered observations, rewards, dones and states equal one
4096-env handle bit-for-bit (every draw is keyed by the global env index,
SURVEY §8(e)).  The box has one GPU, so both ranks use cuda:0; their kernels
never wait on each other (the gather happens on host tensors after the
rollout)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
N, STEPS = 4096, 30


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rollout(n, offset, task):
    from paper_1810_05762_b200.sim import VecEnv
    env = VecEnv(task, n_envs=n, seed=77, env_offset=offset)
    obs, rew, done = [], [], []
    for t in range(STEPS):
        o, r, d = env.step(env.random_actions(t))
        obs.append(o.cpu())
        rew.append(r.cpu())
        done.append(d.cpu())
    torch.cuda.synchronize()
    state = torch.from_numpy(env.get_state())
    env.close()
    return torch.stack(obs), torch.stack(rew), torch.stack(done), state


def _worker(rank, world, port, task, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_local = N // world
    outs = _rollout(n_local, rank * n_local, task)
    gathered = []
    for x in outs:
        g = [torch.zeros_like(x) for _ in range(world)]
        dist.all_gather(g, x.contiguous())
        gathered.append(g)
    if rank == 0:
        q.put([torch.cat(g, dim=1 if k < 3 else 0).numpy() for k, g in enumerate(gathered)])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("task", ["humanoid", "ant"])
def test_two_rank_cuda_shards_equal_single_handle(task):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, task, q)) for r in range(2)]
    for p in procs:
        p.start()
    sharded = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = [x.numpy() for x in _rollout(N, 0, task)]
    for a, b, name in zip(single, sharded, ["obs", "reward", "done", "state"]):
        np.testing.assert_array_equal(a, b, err_msg=name)
