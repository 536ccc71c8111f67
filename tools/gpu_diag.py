"""First-light diagnostics on a B200: GPU vs oracle on a few envs, timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_05762_b200 import abi
from paper_1810_05762_b200.sim import VecEnv
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from oracle import OracleEnv

def teacher_forced(task, prec, N=16, steps=40, tmax_scale=1.0):
    env = VecEnv(task, n_envs=N, precision=prec, seed=7)
    orc = OracleEnv(env.model, env.task, env.cfg, N, seed=7)
    s0 = orc.get_state(); g0 = env.get_state()
    print(task, prec, "reset state max diff", np.abs(s0 - g0).max())
    tm = np.array([env.model.joints[j].max_torque for j in range(env.action_dim)])
    errs = []; cnt_mis = 0; cnt_tot = 0
    for t in range(steps):
        a = orc.random_actions(t) * tmax_scale
        tq = a * tm
        st = orc.get_state()
        env.set_state(st)
        orc.physics_step(tq); env.physics_step(tq)
        so, sg = orc.get_state(), env.get_state()
        dx = np.abs(so[..., 0:3] - sg[..., 0:3]).max(axis=(1, 2))
        dv = (np.abs(so[..., 7:13] - sg[..., 7:13]).max(axis=(1, 2)) / np.maximum(1, np.abs(so[..., 7:13]).max(axis=(1, 2))))
        co, cg = orc.contact_arrays(), env.contact_arrays()
        mis = (co["count"] != cg["count"]).sum()
        cnt_mis += mis; cnt_tot += N
        errs.append((dx, dv))
        if t < 3 or t == steps - 1:
            rg = env.report(); ro = orc.report()
            print(f"  t={t} dx max {dx.max():.3e} relv max {dv.max():.3e} contacts gpu {cg['count'][:4]} orc {co['count'][:4]} mis {mis} kry g{rg['krylov_iterations'][:3]} o{ro['krylov_iterations'][:3]} failed {rg['failed'].sum()} ovf {rg['overflow'].sum()}")
    dx = np.concatenate([e[0] for e in errs]); dv = np.concatenate([e[1] for e in errs])
    print(f"  SUMMARY {task} {prec}: dx p50 {np.median(dx):.2e} p99 {np.percentile(dx,99):.2e} max {dx.max():.2e}; relv p50 {np.median(dv):.2e} p99 {np.percentile(dv,99):.2e} max {dv.max():.2e}; contact count mismatches {cnt_mis}/{cnt_tot}")

def env_compare(task, prec, N=8, steps=30):
    env = VecEnv(task, n_envs=N, precision=prec, seed=3)
    orc = OracleEnv(env.model, env.task, env.cfg, N, seed=3)
    for t in range(steps):
        a = orc.random_actions(t)
        st = orc.get_state(); ts = orc.task_state()
        env.set_state(st); env.set_task_state(ts["target"], ts["counters"], ts["last_tau"])
        oo, ro, do = orc.step(a)
        og, rg, dg = env.step_host(a.astype(np.float32))
        if t < 3 or t == steps - 1:
            print(f"  env {task} {prec} t={t} obs maxdiff {np.abs(oo-og).max():.3e} at {np.unravel_index(np.abs(oo-og).argmax(), oo.shape)} rew diff {np.abs(ro-rg).max():.3e} done o{do.sum()} g{dg.sum()} rew {ro[:3]} {rg[:3]}")

def bench(task, N, steps=50):
    env = VecEnv(task, n_envs=N, precision="f32", seed=1)
    acts = [env.random_actions(i) for i in range(8)]
    for i in range(5): env.step(acts[i % 8])
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(steps): env.step(acts[i % 8])
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    print(f"BENCH {task} N={N}: {ms:.3f} ms/step, {N/ms*1e3:.3e} env-steps/s")

if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    for task in ["humanoid", "ant"]:
        for prec in ["f64", "f32"]:
            try:
                teacher_forced(task, prec)
            except Exception as ex:
                print("ERR teacher_forced", task, prec, repr(ex))
        for prec in ["f64", "f32"]:
            try:
                env_compare(task, prec)
            except Exception as ex:
                print("ERR env_compare", task, prec, repr(ex))
    for task, N in [("humanoid", 1024), ("humanoid", 4096), ("ant", 4096)]:
        try:
            bench(task, N)
        except Exception as ex:
            print("ERR bench", task, N, repr(ex))
