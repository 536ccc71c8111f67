"""Generate golden fixtures from the compiled, unmodified reference physics
(oracle/_ref/libstampede_ref.so, built from /root/reference by oracle/Makefile).

For Ant, Humanoid and HFH: 4 envs x 240 env_steps (Ant 200) of the SPEC env
layer (auto-reset on) with counter-based random actions.  Humanoids fall
under random torques, so the Humanoid and HFH fixtures contain terminations,
auto-resets and (HFH) the 160-frame fall grace and flagrun target redraws.  Stored per step: the state BEFORE the step
(``states[t]``; ``states[t + 1]`` is the state after it, i.e. the reset state
for a done env), actions, reward, done, obs, target / counters before the
step and the ordered contact list (count, body_a, separation).  Run here
(where /root/reference exists); the .npz files travel with the repo.

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

N, SEED = 4, 20261018
STEPS = {"ant": 200, "humanoid": 240, "hfh": 240}
CAPACITY = 64


def make(task_name, kind_id):
    model = abi.builtin_model("ant" if task_name == "ant" else "humanoid")
    task = abi.default_task(kind_id)
    cfg = abi.default_step_config()
    env = oracle.OracleEnv(model, task, cfg, N, seed=SEED, kind="reference")
    states, acts, rews, dones, obs, ccount, cbody, csep, tgt, cnt = ([] for _ in range(10))
    for t in range(STEPS[task_name]):
        a = env.random_actions(t)
        states.append(env.get_state())
        ts = env.task_state()
        tgt.append(ts["target"])
        cnt.append(ts["counters"])
        o, r, d = env.step(a)
        acts.append(a)
        rews.append(r)
        dones.append(d)
        obs.append(o.astype(np.float32))
        c = env.contact_arrays(CAPACITY)
        ccount.append(c["count"])
        cbody.append(c["body_a"].astype(np.int8))
        csep.append(c["separation"].astype(np.float32))
    states.append(env.get_state())
    np.savez_compressed(os.path.join(HERE, f"golden_{task_name}.npz"), states=np.array(states),
                        actions=np.array(acts), reward=np.array(rews), done=np.array(dones), obs=np.array(obs),
                        contact_count=np.array(ccount), contact_body=np.array(cbody),
                        contact_sep=np.array(csep), target=np.array(tgt), counters=np.array(cnt),
                        seed=SEED, n=N, steps=STEPS[task_name], task=task_name, backend=env.backend)
    print(task_name, "done events", int(np.array(dones).sum()))


if __name__ == "__main__":
    if not oracle.available("reference"):
        oracle.build(reference=True)
    make("ant", abi.TASK_ANT)
    make("humanoid", abi.TASK_HUMANOID)
    make("hfh", abi.TASK_HFH)
    print("written", sorted(os.listdir(HERE)))
