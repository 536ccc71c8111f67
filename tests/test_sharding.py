"""Multi-GPU data path on CPU (gloo, world_size 2): envs shard by contiguous
global index (env_offset = rank * N_local) with NO data-path collective; every
random draw is keyed by the global env index, so the 2-rank run must equal
the 1-rank run bit-for-bit."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, STEPS = 8, 12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rollout(n, offset):
    import oracle
    from paper_1810_05762_b200 import abi
    env = oracle.OracleEnv(abi.builtin_model("humanoid"), abi.default_task(abi.TASK_HFH), abi.default_step_config(),
                           n, seed=5, env_offset=offset)
    rews, states = [], []
    for t in range(STEPS):
        _, r, _ = env.step(env.random_actions(t))
        rews.append(r)
    states = env.get_state()
    return np.array(rews), states


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_local = N // world
    rews, states = _rollout(n_local, rank * n_local)
    r = torch.from_numpy(rews)
    s = torch.from_numpy(states)
    rg = [torch.zeros_like(r) for _ in range(world)]
    sg = [torch.zeros_like(s) for _ in range(world)]
    dist.all_gather(rg, r)
    dist.all_gather(sg, s)
    if rank == 0:
        q.put((torch.cat(rg, dim=1).numpy(), torch.cat(sg, dim=0).numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rews2, states2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rews1, states1 = _rollout(N, 0)
    np.testing.assert_array_equal(rews1, rews2)
    np.testing.assert_array_equal(states1, states2)
