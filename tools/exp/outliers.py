"""Find the worst teacher-forced fp32 step errors (physics) over a long
Humanoid protocol and save the pre-states / torques for offline analysis."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np, oracle
from paper_1810_05762_b200.sim import VecEnv
n, steps, seed = 32, 1000, 7
g = VecEnv("humanoid", n_envs=n, precision="f32", seed=seed)
o = oracle.OracleEnv(g.model, g.task, g.cfg, n, seed=seed)
tm = np.array([g.model.joints[j].max_torque for j in range(g.action_dim)])
rec = []
for t in range(steps):
    tq = o.random_actions(t) * tm
    s = o.get_state()
    g.set_state(s)
    o.physics_step(tq); g.physics_step(tq)
    a, b = o.get_state(), g.get_state()
    dx = np.abs(a[..., :3] - b[..., :3]).max(axis=(1, 2))
    for e in np.argsort(dx)[-3:]:
        rec.append((dx[e], t, e, s[e].copy(), tq[e].copy(), a[e].copy(), b[e].copy()))
rec.sort(key=lambda r: -r[0])
rec = rec[:20]
np.savez(os.path.join(ROOT, "gpurun_out", "outliers.npz"), dx=np.array([r[0] for r in rec]),
         t=np.array([r[1] for r in rec]), e=np.array([r[2] for r in rec]), pre=np.array([r[3] for r in rec]),
         tq=np.array([r[4] for r in rec]), post_o=np.array([r[5] for r in rec]), post_g=np.array([r[6] for r in rec]))
print([(float(r[0]), r[1], r[2]) for r in rec[:10]])
