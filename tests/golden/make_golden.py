"""Generate golden fixtures from the compiled, unmodified reference physics
(oracle/_ref/libstampede_ref.so, built from /root/reference by oracle/Makefile).

For Ant and Humanoid: 2 envs x 40 env_steps of the SPEC env layer with
counter-based random actions; every pre-step state, action, post-step state,
reward, done, obs and the ordered contact list (body, separation).  Run here
(where /root/reference exists); the .npz travels with the repo.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle  # noqa: E402
from paper_1810_05762_b200 import abi  # noqa: E402

N, STEPS, SEED = 2, 40, 20261018


def make(task_name, kind_id):
    model = abi.builtin_model("ant" if task_name == "ant" else "humanoid")
    task = abi.default_task(kind_id)
    cfg = abi.default_step_config()
    env = oracle.OracleEnv(model, task, cfg, N, seed=SEED, kind="reference")
    pre, post, acts, rews, dones, obs, ccount, cbody, csep, tgt, cnt = ([] for _ in range(11))
    for t in range(STEPS):
        a = env.random_actions(t)
        pre.append(env.get_state())
        ts = env.task_state()
        tgt.append(ts["target"])
        cnt.append(ts["counters"])
        o, r, d = env.step(a)
        post.append(env.get_state())
        acts.append(a)
        rews.append(r)
        dones.append(d)
        obs.append(o)
        c = env.contact_arrays(64)
        ccount.append(c["count"])
        cbody.append(c["body_a"])
        csep.append(c["separation"])
    np.savez_compressed(os.path.join(HERE, f"golden_{task_name}.npz"), pre=np.array(pre), post=np.array(post),
                        actions=np.array(acts), reward=np.array(rews), done=np.array(dones), obs=np.array(obs),
                        contact_count=np.array(ccount), contact_body=np.array(cbody),
                        contact_sep=np.array(csep), target=np.array(tgt), counters=np.array(cnt),
                        seed=SEED, n=N, steps=STEPS, backend=env.backend)


if __name__ == "__main__":
    if not oracle.available("reference"):
        oracle.build(reference=True)
    make("ant", abi.TASK_ANT)
    make("humanoid", abi.TASK_HUMANOID)
    print("written", os.listdir(HERE))
