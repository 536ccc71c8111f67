"""For the saved outliers: GPU f64 instrument, GPU f32 under 1e-7 input
perturbations, Krylov counts (GPU vs oracle)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np, oracle
from paper_1810_05762_b200.sim import VecEnv
d = np.load(os.path.join(ROOT, "tools", "exp", "data", "outliers.npz"))
K = 64
g64 = VecEnv("humanoid", n_envs=1, precision="f64", seed=7)
gp = VecEnv("humanoid", n_envs=K, precision="f32", seed=7)
o = oracle.OracleEnv(g64.model, g64.task, g64.cfg, 1, seed=7)
rng = np.random.default_rng(0)
for k in range(8):
    pre, tq, po = d["pre"][k], d["tq"][k], d["post_o"][k]
    o.set_state(pre[None]); o.physics_step(tq[None]); ko = o.report()["krylov_iterations"][0]
    g64.set_state(pre[None]); g64.physics_step(tq[None])
    e64 = np.abs(g64.get_state()[0][..., :3] - po[..., :3]).max()
    P = np.repeat(pre[None], K, 0)
    P[1:, :, :3] += rng.uniform(-1, 1, P[1:, :, :3].shape) * 1e-7
    gp.set_state(P); gp.physics_step(np.repeat(tq[None], K, 0))
    gs = gp.get_state(); kg = gp.report()["krylov_iterations"]
    dx = np.abs(gs[..., :3] - po[None, :, :3]).max(axis=(1, 2))
    print(f"case {k} gpu dx {d['dx'][k]:.2e}: f64 kernel dx {e64:.1e}; f32 exact input dx {dx[0]:.2e}; "
          f"f32 perturbed dx p50 {np.median(dx[1:]):.2e} min {dx[1:].min():.2e} max {dx[1:].max():.2e}; "
          f"krylov oracle {ko} gpu {kg[0]} (perturbed {sorted(set(kg.tolist()))})", flush=True)
