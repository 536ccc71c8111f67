"""K4 phase timeline (experiment): build a copy of the library with
-DSTP_K4_PHASES (policy_mlp.cu only; the other objects come from the normal
build), run the rollout policy forward at 4096 envs, and print per-phase
durations (median / max over CTAs) from %globaltimer stamps.
`build REV` also builds tools/exp/_k4old.so from REV's policy_mlp.cu; `run`
then checks the two kernels' outputs for bit identity and times both.
usage: python tools/exp/k4_phases.py build [REV]  (here)  |  python tools/exp/k4_phases.py run  (GPU)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
SO = os.environ.get("K4SO", os.path.join(ROOT, "tools", "exp", "_k4phase.so"))
OLD = os.path.join(ROOT, "tools", "exp", "_k4old.so")
NAMES = {0: "start", 1: "prologue sync", 11: "obs landed", 2: "obs prologue", 3: "weights landed", 4: "mma L0",
         5: "epi L0", 6: "mma L1", 7: "epi L1", 8: "mma L2", 9: "epi L2", 10: "mma L3", 12: "head + end"}
for _l in range(4):
    NAMES[13 + _l] = f"sync L{_l}"
    NAMES[17 + _l] = f"issued L{_l}"
    NAMES[21 + _l] = f"noise L{_l}"
NAMES.update({25: "head tile", 26: "head sync", 27: "head rows", 28: "L0 first tmem ld"})
ORDER = [1, 11, 2, 3, 13, 17, 21, 4, 28, 5, 14, 18, 22, 6, 7, 15, 19, 23, 8, 9, 16, 20, 24, 10, 25, 26, 27, 12]
KP = 32
CLK_GHZ = float(os.environ.get("CLK_GHZ", "1.965"))


def build():
    from paper_1810_05762_b200 import build as B
    B.build()
    obj = os.path.join(B.BUILD, "policy_mlp_phases.o")
    cmd = [B.NVCC] + B.ARCH + B.FLAGS + ["-DSTP_K4_PHASES", "-c", os.path.join(B.CSRC, "policy_mlp.cu"), "-o", obj]
    subprocess.run(cmd, check=True, capture_output=True)
    objs = [os.path.join(B.BUILD, s + ".o") for s in B.SOURCES if s != "policy_mlp.cu"] + [obj]
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", SO] + objs + ["-lcudart"], check=True)
    print("built", SO)
    if len(sys.argv) > 2:
        src = os.path.join(B.BUILD, "policy_mlp_old.cu")
        with open(src, "w") as f:
            f.write(subprocess.run(["git", "show", f"{sys.argv[2]}:paper_1810_05762_b200/csrc/policy_mlp.cu"],
                                   cwd=ROOT, check=True, capture_output=True, text=True).stdout)
        obj = os.path.join(B.BUILD, "policy_mlp_old.o")
        subprocess.run([B.NVCC] + B.ARCH + B.FLAGS + ["-c", src, "-o", obj], check=True, capture_output=True)
        objs[-1] = obj
        subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", OLD] + objs + ["-lcudart"], check=True)
        print("built", OLD)


def run():
    import ctypes as C

    import numpy as np
    import torch

    from paper_1810_05762_b200 import abi
    abi.LIB_PATH = SO
    from paper_1810_05762_b200.policy import ActorCritic, PolicyKernel
    from paper_1810_05762_b200.sim import VecEnv
    n = int(os.environ.get("N", "4096"))
    env = VecEnv("humanoid", n_envs=n)
    obs = env.reset()
    kern = PolicyKernel(ActorCritic(env.obs_dim, env.action_dim).to("cuda"), "cuda:0")
    m_ = torch.zeros(env.obs_dim, device="cuda")
    s_ = torch.ones(env.obs_dim, device="cuda")
    lib = abi.load()
    lib.stp_k4_phases.argtypes = [C.c_void_p, C.c_int]
    for it in range(30):
        _, a, _, _ = kern.forward(obs, m_, s_, step=it)
        obs, _, _ = env.step(a)
    torch.cuda.synchronize()
    for _ in range(int(os.environ.get("REPS", "1"))):  # REPS=2: the recorded forward follows a forward (warm code)
        kern.forward(obs, m_, s_, step=99)
    torch.cuda.synchronize()
    nt = 64 if (n + 63) // 64 * 2 >= 120 else 32 if (n + 31) // 32 * 2 >= 120 else 16  # stp_policy_forward's NT
    ctas = 2 * ((n + nt - 1) // nt)
    buf = np.zeros(ctas * KP, dtype=np.uint64)
    lib.stp_k4_phases(buf.ctypes.data, buf.size)
    t = buf.reshape(ctas, KP).astype(np.int64)
    g0 = t[:, 31].min()
    span = (t[:, 12] - t[:, 0]) / CLK_GHZ / 1e3 + (t[:, 31] - g0) / 1e3
    print(f"{ctas} CTAs; launch spread {(t[:, 31].max() - g0) / 1e3:.2f} us; "
          f"kernel span {span.max():.2f} us (SM clock at {CLK_GHZ} GHz; CTA body median "
          f"{np.median((t[:, 12] - t[:, 0]) / CLK_GHZ / 1e3):.2f} us)")
    prev = 0
    for i in ORDER:
        if i in (17, 18, 19, 20):  # thread 0 only; others wait at the mma barrier
            pass
        d = (t[:, i] - t[:, prev]) / CLK_GHZ / 1e3
        print(f"  {NAMES[prev]:>15} -> {NAMES[i]:<15} median {np.median(d):7.2f} us  max {d.max():7.2f} us"
              f"   (policy {np.median(d[: ctas // 2]):6.2f}, value {np.median(d[ctas // 2:]):6.2f})")
        prev = i

    def timed(k, reps=50):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(5):
            k.forward(obs, m_, s_, step=1)
        ev[0].record()
        for _ in range(reps):
            k.forward(obs, m_, s_, step=1)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps * 1e3

    print(f"forward: {timed(kern):.2f} us / call (instrumented build)")
    if os.path.exists(OLD):
        old = PolicyKernel(kern.model, "cuda:0")
        old.lib = abi.load(OLD)
        m_ = torch.rand(env.obs_dim, device="cuda") - 0.5
        s_ = torch.rand(env.obs_dim, device="cuda") + 0.5
        a = kern.forward(obs, m_, s_, seed=3, step=7)
        b = old.forward(obs, m_, s_, seed=3, step=7)
        for name, x, y in zip(["mean", "action", "logp", "value"], a, b):
            print(f"  {name}: bit-identical {bool(torch.equal(x, y))}  max|d| {(x - y).abs().max().item():.3g}")
        print(f"old forward: {timed(old):.2f} us / call")


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
