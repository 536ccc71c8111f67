#!/usr/bin/env python3
"""Benchmark: env-steps/s of Humanoid random-action rollouts, 4096 envs per GPU.

Metric (BASELINE.json): "env-steps/sec (Humanoid, 4096 envs/GPU) at 1/2/4/8
B200; % of HBM/FP32 roofline".  One *step* = one env_step of all 4096
environments of this rank (actuation, contacts, 4 x Newton/PCR solve,
integration, reward, termination, auto-reset, observation) = one launch of
the fused sm_100a kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 outside torchrun the script re-launches itself as N ranks
(torch.distributed.run, 127.0.0.1); each rank steps its own 4096 envs
(env_offset = rank * 4096) with no collective in the timed region.

Timing: K steps, each bracketed by CUDA events on the launching stream with
an L2 flush (a 256 MiB write, outside the events) between steps; a barrier +
synchronize brackets the whole timed loop; the per-rank device time is the
sum of the K event intervals; the job time is the MAX over ranks.  `value` is
total env-steps of all ranks / that time.  `e2e` repeats the measurement
through the host-buffer C-ABI call stp_step_host (pinned H2D actions, kernel,
D2H obs/reward/done, synchronise) and is timed on the host clock.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ENVS = 4096
TASK = "humanoid"
SEED = 1234

# BASELINE.json configs as workloads (the default is the metric's: Humanoid,
# 4096 envs per GPU).  flop = algorithmic FLOPs per env-step of the reference
# algorithm (0.93 M Humanoid-size, 0.37 M Ant-size; terrain
# contact work on top is not counted).  Terrain: boxes over the env grid.
WORKLOADS = {
    "humanoid4096": dict(task="humanoid", n=4096, flop=929_813.0,
                         name="humanoid_run_flat_4096envs_random_actions", config="metric (configs[2] size)"),
    "ant64": dict(task="ant", n=64, flop=369_122.0, name="ant_run_flat_64envs_random_actions", config="configs[0]"),
    "humanoid1024": dict(task="humanoid", n=1024, flop=929_813.0, name="humanoid_run_flat_1024envs_random_actions",
                         config="configs[1]"),
    "hfh4096": dict(task="hfh", n=4096, flop=929_813.0,
                    name="hfh_flagrun_4096envs_random_actions_interagent", config="configs[2]"),
    "hfh_terrain4096": dict(task="hfh_terrain", n=4096, flop=929_813.0, boxes=2048, extent=131.0,
                            name="hfh_terrain_4096envs_2048boxes_random_actions", config="configs[3]"),
}


def terrain_boxes(n_boxes, extent, seed=3):
    """generate_terrain over the env grid: dims U[0.2, 1] m,
    yaw U[0, pi) (counter-based RNG, fixed seed).  The oracle's restatement
    (oracle/model_text.py) draws the same boxes as the device library's
    stp_generate_terrain (tests/test_model_format.py), and keeps the CPU arms
    off the product library."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import model_text
    return model_text.generate_terrain(n_boxes, 0.2, 1.0, -3.0, extent, -3.0, extent, 0.0, 3.141592653589793, seed)


# Algorithmic work of the reference algorithm per Humanoid env-step (FP32
# roofline numerator): 0.93 MFLOP measured with a
# counting-scalar build of the unmodified reference on a 22-body / 21-hinge
# humanoid under random actions; one 16-iteration PCR solve = 179,114 FLOP.
# The PCR share is rescaled by the live Krylov iteration count the kernel
# reports.
F_ENV_STEP = 929_813.0
F_PCR_SOLVE16 = 179_114.0
F_PCR_ITER = F_PCR_SOLVE16 / 16.0


def _traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture (profiles/traffic.json, written by
    tools/ncu_traffic.py); null when no capture is recorded."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)[kernel]
        return {"bytes_per_launch": t["dram_read_bytes"] + t["dram_write_bytes"],
                "read": t["dram_read_bytes"], "write": t["dram_write_bytes"], "source": t["capture"]}
    except (OSError, KeyError, ValueError):
        return None


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region.

    Polls NVML every ~2 ms from a thread (nvidia-smi -lms is too coarse for a
    sub-second region); falls back to nvidia-smi when NVML is unavailable."""

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.err = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis else self.device
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as ex:  # reported, never fatal
            self.err = repr(ex)
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                     int(get_reasons(self.h))))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if self.err is not None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self._stop.set()
        self.t.join(timeout=1)
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        reasons = sorted({k for _, r in self.samples for k, b in bits.items() if r & b})
        mhz = [m for m, _ in self.samples]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(mhz)}


def _cpu_info():
    """lscpu model name, logical CPUs and physical cores of this host."""
    model, sockets, cores_per = None, 1, None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            v = v.strip()
            if k.strip() == "Model name":
                model = v
            elif k.strip() == "Socket(s)":
                sockets = int(v)
            elif k.strip() == "Core(s) per socket":
                cores_per = int(v)
    except (OSError, ValueError, subprocess.SubprocessError):
        pass
    logical = os.cpu_count() or 1
    try:
        logical = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    return {"cpu_model": model, "logical_cpus": logical,
            "physical_cores": sockets * cores_per if cores_per else None}


def cpu_reference_rate(n_envs: int, steps: int, warmup: int, threads: int, budget_s: float = 20.0,
                       single_thread_s: float = 0.0, workload: str = "humanoid4096"):
    """Reference stampede::physics::step + restated env layer on host cores.

    Runs oracle/_ref (the compiled, unmodified reference, its Release flags)
    when it was built, else the restated oracle port.  The model, task and
    step config come from the oracle's own reader of assets/humanoid.model
    (oracle/model_text.py), so this arm never loads the product library.
    Bounded sample: the env count is cut so the timed part stays within
    ~budget_s.  With single_thread_s > 0 the same workload is also timed on
    one thread (n = all cores and n = 1).
    """
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import OracleEnv, available
    import model_text
    from paper_1810_05762_b200 import abi  # ctypes struct layouts only (no library load)
    kind = "reference_fast" if available("reference_fast") else "restatement"
    wl = WORKLOADS[workload]
    kinds = {"ant": abi.TASK_ANT, "humanoid": abi.TASK_HUMANOID, "hfh": abi.TASK_HFH,
             "hfh_terrain": abi.TASK_HFH_TERRAIN}
    model = model_text.load_model("ant" if wl["task"] == "ant" else "humanoid")
    task = model_text.default_task(kinds[wl["task"]])
    cfg = model_text.default_step_config()
    boxes = terrain_boxes(wl["boxes"], wl["extent"]) if wl.get("boxes") else None

    def measure(nthreads, budget, n_steps, n_warm):
        probe_n = min(n_envs, 64 * nthreads)
        env = OracleEnv(model, task, cfg, probe_n, seed=SEED, nthreads=nthreads, kind=kind, terrain=boxes)
        for s in range(2):
            env.step(env.random_actions(s))
        t0 = time.perf_counter()
        env.step(env.random_actions(2))
        rate = probe_n / max(time.perf_counter() - t0, 1e-6)
        env.close()
        n_sample = int(max(16, min(n_envs, rate * budget / max(1, n_steps))))
        env = OracleEnv(model, task, cfg, n_sample, seed=SEED, nthreads=nthreads, kind=kind, terrain=boxes)
        acts = [env.random_actions(s) for s in range(n_warm + n_steps)]
        for s in range(n_warm):
            env.step(acts[s])
        t0 = time.perf_counter()
        for s in range(n_steps):
            env.step(acts[n_warm + s])
        dt = time.perf_counter() - t0
        env.close()
        return n_sample * n_steps / dt, n_sample

    value, n_sample = measure(threads, budget_s, steps, warmup)
    info = _cpu_info()
    out = {"value": value, "unit": "env-steps/s", "cores": threads,
           "kind": "reference" if kind.startswith("reference") else "port",
           "sample": f"{n_sample} of {n_envs} {wl['task']} envs x {steps} env_steps (random actions, auto-reset), "
                     f"{'oracle/_ref/libstampede_ref_fast.so: unmodified stampede::physics::step, -O3 -march=native, util::ThreadPool(' + str(threads) + ')' if kind.startswith('reference') else 'oracle/liboracle.so restatement'}"
                     f" + restated env layer; model from assets/*.model via oracle/model_text.py",
           **info}
    if single_thread_s > 0:
        v1, n1 = measure(1, single_thread_s, 2, 1)
        out["value_1_thread"] = v1
        out["sample_1_thread"] = f"{n1} envs x 2 env_steps on 1 thread"
    return out


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args) -> None:
    """`--gpus N` (N > 1) outside torchrun: re-run this script as N ranks of
    one node through torch.distributed.run on 127.0.0.1 (the driver's own
    launch sets WORLD_SIZE and skips this).  Rank 0 prints the line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    sys.exit(subprocess.run(cmd, env=env).returncode)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch
            if torch.cuda.device_count() < world:
                raise SystemExit(f"bench.py --gpus {world}: only {torch.cuda.device_count()} GPU(s) visible")
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def bench_config(world: int, workload: str = "humanoid4096") -> dict:
    """The workload description, identical in both arms."""
    wl = WORKLOADS[workload]
    c = {"workload": wl["name"], "envs_per_gpu": wl["n"], "task": wl["task"], "baseline_config": wl["config"],
         "parallelism": f"dp{world} (env shards, no collective)",
         "l2": "flushed between timed steps (256 MiB write)", "auto_reset": True}
    if wl.get("boxes"):
        c["terrain"] = f"{wl['boxes']} static yaw boxes over [-3, {wl['extent']:.0f}] m^2 (generate_terrain, seed 3)"
    return c


def metric_name(workload: str) -> str:
    return ("env-steps/sec (Humanoid, 4096 envs/GPU)" if workload == "humanoid4096"
            else f"env-steps/sec ({WORKLOADS[workload]['name']})")


def run_reference(args, world, rank):
    if rank != 0:
        return
    threads = _cpu_info()["logical_cpus"]
    budget = float(os.environ.get("STP_BENCH_CPU_BUDGET_S", "90"))
    n_envs = WORKLOADS[args.workload]["n"]
    r = cpu_reference_rate(n_envs, max(1, args.steps), max(0, args.warmup), threads, budget_s=budget,
                           single_thread_s=min(10.0, budget / 6), workload=args.workload)
    line = {"metric": metric_name(args.workload), "value": r["value"], "unit": "env-steps/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * n_envs / r["value"] if r["value"] else None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(world, args.workload),
            "cpu_baseline": r,
            "e2e": {"value": r["value"], "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "CPU reference on the host cores of rank 0 only (one sample of the per-GPU workload)",
            "repo_libraries_loaded": _repo_libraries_loaded()}
    print(json.dumps(line), flush=True)


def _repo_libraries_loaded():
    """Shared objects under this repo mapped into the process (the reference
    arm must show only oracle/_ref/*.so)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in paths if os.path.realpath(p).startswith(os.path.realpath(ROOT)))


def run_ours(args, world, rank, local):
    global N_ENVS, TASK
    wl = WORKLOADS[args.workload]
    N_ENVS, TASK = wl["n"], wl["task"]
    boxes = terrain_boxes(wl["boxes"], wl["extent"]) if wl.get("boxes") else None
    import torch
    from paper_1810_05762_b200.sim import VecEnv
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    assert torch.cuda.is_available(), "bench.py --impl ours needs a CUDA device (no CPU fallback)"
    env = VecEnv(TASK, n_envs=N_ENVS, device=local, seed=SEED, env_offset=rank * N_ENVS, terrain=boxes)
    K, Wm = args.steps, args.warmup
    # synthetic inputs resident in HBM before timing: one action batch per step
    acts = [env.random_actions(s) for s in range(Wm + K)]
    obs = torch.empty((N_ENVS, env.obs_dim), device=dev)
    rew = torch.empty((N_ENVS,), device=dev)
    done = torch.empty((N_ENVS,), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    for s in range(Wm):
        env.step(acts[s], obs, rew, done)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for s in range(K):
        flush.fill_(float(s))
        ev[s][0].record()
        env.step(acts[Wm + s], obs, rew, done)
        ev[s][1].record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    rep = env.report()
    kry_mean = float(rep["krylov_iterations"].mean())
    failed = int(rep["failed"].sum())
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    per_rank_ms = [dev_ms]
    if world > 1:
        allt = [torch.zeros_like(t) for _ in range(world)]
        torch.distributed.all_gather(allt, t)
        per_rank_ms = [float(x.item()) for x in allt]
    job_ms = max(per_rank_ms)
    value = world * N_ENVS * K / (job_ms / 1e3)
    ms_per_step = job_ms / K

    # ---- rollout: env_step + tcgen05 policy forward (K4) per step, device-timed
    rollout = None
    try:
        from paper_1810_05762_b200.policy import HIDDEN, ActorCritic, PolicyKernel, RunningStat
        torch.manual_seed(0)
        model = ActorCritic(env.obs_dim, env.action_dim, HIDDEN.get(TASK, HIDDEN["hfh"])).to(dev)
        kern = PolicyKernel(model, dev)
        st = RunningStat(env.obs_dim, device=dev)
        st.push(obs)
        m_, s_ = st.mean.float(), st.std.float()
        for s in range(3):
            _, a, _, _ = kern.forward(obs, m_, s_, seed=SEED, step=s)
            env.step(a.clamp(-1, 1), obs, rew, done)
        torch.cuda.synchronize()
        r0, r1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        r0.record()
        for s in range(K):
            _, a, _, _ = kern.forward(obs, m_, s_, seed=SEED, step=3 + s)
            env.step(a.clamp(-1, 1), obs, rew, done)
        r1.record()
        torch.cuda.synchronize()
        roll_ms = r0.elapsed_time(r1) / K
        # K4 alone: one CUDA graph of K forwards, so the device time is not
        # bounded by the host's per-call Python / ctypes overhead
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                for s in range(K):
                    kern.forward(obs, m_, s_, seed=SEED, step=3 + s)
        torch.cuda.current_stream(dev).wait_stream(cs)
        g.replay()
        torch.cuda.synchronize()
        q0, q1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        q0.record()
        g.replay()
        q1.record()
        torch.cuda.synchronize()
        pol_ms = q0.elapsed_time(q1) / K
        rollout = {"env_steps_per_s": N_ENVS / (roll_ms / 1e3), "ms_per_step": roll_ms,
                   "policy_forward_ms": pol_ms, "policy_forward_timing": "CUDA graph of K forwards, device",
                   "policy": f"tcgen05 SELU MLP pi+V {HIDDEN.get(TASK, HIDDEN["hfh"])} bf16",
                   "l2": "not flushed"}
    except Exception as ex:
        rollout = {"error": repr(ex)}

    # ---- config C5: PPO iterations (rollout + 20-epoch update with the
    # per-minibatch gradient allreduce), host-timed after one warm-up
    # iteration; informational (the metric above is the env step).  Frames per
    # iteration per GPU stay the paper's 32 x 1024 = 32768 (PAPER.md:256-258,
    # SPEC.md:379-381): 8 frames per agent at 4096 envs
    ppo = None
    try:
        if args.workload != "humanoid4096":
            raise RuntimeError("PPO iteration timed for the metric workload only")
        from paper_1810_05762_b200.ppo import PPOConfig, PPOLearner, gae
        from paper_1810_05762_b200.ppo import rollout as ppo_rollout
        torch.manual_seed(0)
        pmodel = ActorCritic(env.obs_dim, env.action_dim, HIDDEN.get(TASK, HIDDEN["hfh"])).to(dev)
        pcfg = PPOConfig(frames_per_iter=max(1, 32768 // N_ENVS))
        learner = PPOLearner(pmodel, pcfg)
        pkern = PolicyKernel(pmodel, dev)
        pst = RunningStat(env.obs_dim, device=dev)
        env.last_obs = env.reset()
        first = RunningStat(env.obs_dim, device=dev)
        first.push(env.last_obs)
        if world > 1:
            pst.merge_allreduce(first)  # same global statistics on every rank
        else:
            pst._merge(first.n, first.mean, first.m2)
        times, upd = [], []
        for it in range(5):
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            data, last_val = ppo_rollout(env, pkern, pst, pcfg.frames_per_iter, SEED, 1000 + it * pcfg.frames_per_iter,
                                         env_offset=rank * N_ENVS)
            loc = RunningStat(env.obs_dim, device=dev)
            loc.push(data["obs"].reshape(-1, env.obs_dim))
            if world > 1:
                pst.merge_allreduce(loc)
            else:
                pst._merge(loc.n, loc.mean, loc.m2)
            ast = torch.zeros(3, dtype=torch.float64, device=dev)
            adv, ret = gae(data["rew"], data["val"], data["done"], last_val, pcfg.gamma, pcfg.lam, stats=ast)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            stats = learner.update(pst.whiten(data["obs"].reshape(-1, env.obs_dim)),
                                   data["act"].reshape(-1, env.action_dim), None, adv.reshape(-1), ret.reshape(-1),
                                   adv_stats=ast)
            pkern.refresh()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            times.append(t2 - t0)
            upd.append(t2 - t1)
        it_s = statistics.median(times[1:])
        frames = pcfg.frames_per_iter * N_ENVS * world
        ppo = {"iteration_s": it_s, "update_s": statistics.median(upd[1:]), "frames_per_iteration": frames,
               "frames_per_agent": pcfg.frames_per_iter, "env_steps_per_s_with_update": frames / it_s,
               "epochs": pcfg.epochs, "kl": stats["kl"], "aborted": stats["aborted"], "clock": "host, median of 4",
               "update_gemms": pcfg.matmul,
               "learner": "explicit fwd/bwd: cuBLAS fp32 GEMMs + stp_ppo_surrogate / stp_selu_backward_bias / "
                          "stp_bias_selu kernels, fused Adam"}
    except Exception as ex:
        ppo = {"error": repr(ex)}

    # ---- e2e through the reference-facing C-ABI call with pinned host buffers:
    # each step's actions sit in their own pinned buffer (as a policy writing
    # into host memory would leave them), and stp_step_host is called with raw
    # pointers - the H2D copy, the kernel, the D2H copies and the synchronise
    # are all inside the call and inside the timed region
    import ctypes
    n_buf = min(K, 64)
    h_acts = [acts[Wm + s].cpu().pin_memory() for s in range(n_buf)]
    h_obs = torch.empty((N_ENVS, env.obs_dim), dtype=torch.float32, pin_memory=True)
    h_rew = torch.empty((N_ENVS,), dtype=torch.float32, pin_memory=True)
    h_done = torch.empty((N_ENVS,), dtype=torch.uint8, pin_memory=True)
    p_acts = [ctypes.c_void_p(t.data_ptr()) for t in h_acts]
    p_out = [ctypes.c_void_p(t.data_ptr()) for t in (h_obs, h_rew, h_done)]
    step_host = env.lib.stp_step_host
    for s in range(min(Wm, 3)):
        rc = step_host(env._h, p_acts[s % n_buf], *p_out)
        assert rc == 0, rc
    if world > 1:
        torch.distributed.barrier()
    rcs = 0
    e0 = time.perf_counter()
    for s in range(K):
        rcs |= step_host(env._h, p_acts[s % n_buf], *p_out)
    e2e_s = time.perf_counter() - e0
    assert rcs == 0, rcs
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_value = world * N_ENVS * K / float(te.item())
    h2d = N_ENVS * env.action_dim * 4
    d2h = N_ENVS * (env.obs_dim * 4 + 4 + 1)

    peaks, src = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s
    f_pcr_iter = F_PCR_ITER if TASK != "ant" else 71_617.0 / 16.0  # one PCR iteration
    f_env = wl["flop"] - f_pcr_iter * (64.0 - kry_mean)  # live Krylov count
    achieved = N_ENVS * f_env / (ms_per_step / 1e3) / 1e12
    roof = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": achieved / fp32_peak, "traffic": _traffic("k_env_step<float,32,2>"),
            "kernel": f"k_env_step<float,32,{4 if wl.get('boxes') else 2}>",
            "flop_per_env_step": f_env, "krylov_iters_per_env_step": kry_mean,
            "peak_source": f"148 SM x 128 FP32 lanes x 2 x sm_max_mhz {sm_max:.0f} ({src})",
            "hbm_gbs_achieved": N_ENVS * 2700 / (ms_per_step / 1e3) / 1e9,
            "hbm_peak_gbs": float(peaks.get("hbm_gbs", 6650.0))}
    if clocks.get("sm_mhz"):
        roof["frac_at_measured_clock"] = achieved / (148 * 128 * 2 * clocks["sm_mhz"] * 1e6 / 1e12)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(N_ENVS, 5, 1, _cpu_info()["logical_cpus"], budget_s=20.0,
                                     single_thread_s=6.0, workload=args.workload)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "env-steps/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"unavailable: {ex!r}"}
    per_rank = [N_ENVS * K / (ms / 1e3) for ms in per_rank_ms]
    if rank == 0:
        line = {"metric": metric_name(args.workload), "value": value, "unit": "env-steps/s",
                "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": bench_config(world, args.workload),
                "per_rank_env_steps_per_s": per_rank,
                "weak_scaling_fraction_of_ideal": value / sum(per_rank),
                "e2e": {"value": e2e_value, "unit": "env-steps/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "path": "stp_step_host (pinned host buffers)"},
                "gpu_launches": K, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks, "rollout": rollout, "ppo": ppo,
                "wall_s_timed_region": wall, "failed_envs_last_step": failed}
        print(json.dumps(line), flush=True)
    env.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="humanoid4096",
                    help="BASELINE config (default: the metric's Humanoid, 4096 envs per GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    self_launch(args)
    world, rank, local = dist_setup(args)
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}; reporting n_gpus = {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
