"""Config C5: Humanoid PPO rollout + update with envs sharded over G GPUs.

    torchrun --nproc-per-node G -m paper_1810_05762_b200.train --iters 5

Each rank steps its own env shard (env_offset = rank * N) with the fused
sm_100a kernel, samples actions with the tcgen05 policy forward, merges the
observation statistics (one allreduce), normalises advantages globally and
averages every minibatch gradient with one NCCL allreduce.
Prints one JSON line per iteration on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import time

import torch
import torch.distributed as dist

from .policy import HIDDEN, ActorCritic, PolicyKernel, RunningStat
from .ppo import PPOConfig, PPOLearner, gae, rollout
from .sim import VecEnv


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--task", default="humanoid")
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--frames", type=int, default=32)
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--matmul", choices=["fp32", "tf32"], default="fp32",
                    help="update GEMM precision (PPOConfig.matmul; tf32 is ~1.8x faster, not fp32-exact)")
    args = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    env = VecEnv(args.task, n_envs=args.envs, device=local, seed=args.seed, env_offset=rank * args.envs)
    torch.manual_seed(args.seed)
    model = ActorCritic(env.obs_dim, env.action_dim, HIDDEN.get(args.task, (256, 128, 64))).to(dev)
    cfg = PPOConfig(frames_per_iter=args.frames, epochs=args.epochs, matmul=args.matmul)
    learner = PPOLearner(model, cfg)  # broadcasts rank 0's parameters
    kern = PolicyKernel(model, dev)
    stat = RunningStat(env.obs_dim, device=dev)
    # the initial observations enter the statistics like every later batch:
    # pushed locally, then merged over ranks (one allreduce), so every rank
    # whitens with the same global statistics
    env.last_obs = env.reset()
    first = RunningStat(env.obs_dim, device=dev)
    first.push(env.last_obs)
    if world > 1:
        stat.merge_allreduce(first)
    else:
        stat._merge(first.n, first.mean, first.m2)
    step = 0
    for it in range(args.iters):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        data, last_val = rollout(env, kern, stat, args.frames, args.seed, step, env_offset=rank * args.envs)
        step += args.frames
        torch.cuda.synchronize()
        t_roll = time.perf_counter() - t0
        local_stat = RunningStat(env.obs_dim, device=dev)
        local_stat.push(data["obs"].reshape(-1, env.obs_dim))
        if world > 1:
            stat.merge_allreduce(local_stat)  # observation-statistics allreduce
        else:
            stat._merge(local_stat.n, local_stat.mean, local_stat.m2)
        adv_stats = torch.zeros(3, dtype=torch.float64, device=dev)  # count, sum, sum of squares (GAE kernel)
        adv, ret = gae(data["rew"], data["val"], data["done"], last_val, cfg.gamma, cfg.lam, stats=adv_stats)
        xw = stat.whiten(data["obs"].reshape(-1, env.obs_dim))
        stats = learner.update(xw, data["act"].reshape(-1, env.action_dim), data["logp"].reshape(-1),
                               adv.reshape(-1), ret.reshape(-1), adv_stats=adv_stats)
        kern.refresh()
        torch.cuda.synchronize()
        t_it = time.perf_counter() - t0
        if rank == 0:
            print(json.dumps({"iter": it, "world": world, "envs_per_gpu": args.envs,
                              "frames": args.frames * args.envs * world, "rollout_s": t_roll, "iter_s": t_it,
                              "rollout_env_steps_per_s": args.frames * args.envs * world / t_roll,
                              "mean_reward": float(data["rew"].mean()), **stats}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
