"""Write the round's profile summaries under profiles/ from the captures of
tools/gpu_profile_round.sh TAG (gpurun_out/prof_TAG, prof_pol_TAG, launches_TAG.csv)
and, if present, gpurun_out/launches_hfh_TAG.csv.
usage: python tools/write_profiles.py TAG"""
import csv
import io
import os
import shutil
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def sh(*cmd):
    return subprocess.run(list(cmd), capture_output=True, text=True, cwd=ROOT).stdout


def pcr_block(rep):
    raw = sh("ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    R = rows[2:]
    ia = h.index("Instructions Executed")
    nw = int(R[0][ia])
    tot_all = sum(int(r[ia]) for r in R)
    c = Counter()
    tot = 0
    for r in R:
        n = int(r[ia])
        if n < 40 * nw:
            continue
        op = r[1].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        c[op.split()[0]] += n
        tot += n
    trips = 60 * nw
    return (f"PCR loop: {tot / nw:.0f} of {tot_all / nw:.0f} instructions per warp-step "
            f"({tot / tot_all * 100:.0f} %); 60 trips per env-step, {tot / trips:.0f} instructions per trip\n  "
            + ", ".join(f"{k} {v / trips:.1f}" for k, v in c.most_common(14)))


def launches(path):
    return sh(sys.executable, "tools/launch_summary.py", path).strip().splitlines()[:8]


rep = os.path.join(G, f"prof_{TAG}.ncu-rep")
lines = [f"# Round 1 — ncu evidence for k_env_step {TAG} (B200, sm_100a)", "",
         "Command: `python bench.py --steps 20 --warmup 5 --no-cpu-baseline` (4096 Humanoid envs, flat ground, random actions).",
         f"Launch list (`profiles/r01_launches_{TAG}.csv`): `ncu --metrics gpu__time_duration.sum --clock-control none -c 200` "
         "of the same command (cold-cache, serialised: shares, not absolutes).", "", "```"]
lines += launches(os.path.join(G, f"launches_{TAG}.csv"))
lines += ["```", "",
          "Full capture: `ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 8 -c 1` "
          f"(`tools/gpu_profile_round.sh {TAG}`).", "", "```"]
lines += sh(sys.executable, "tools/ncu_summary.py", rep).rstrip().splitlines()
lines += ["```", "", "Hot PCR loop (SASS rows executed >= 40x per warp):", "", "```", pcr_block(rep), "```", ""]
sh("bash", "tools/spills.sh")
lines += ["Execution-weighted source lines (whole kernel, per warp-step; `tools/line_profile.py`):", "", "```"]
lines += sh(sys.executable, "tools/line_profile.py", rep, "25").rstrip().splitlines()
lines += ["```", ""]
hfh = os.path.join(G, f"launches_hfh_{TAG}.csv")
if os.path.exists(hfh):
    lines += ["HFH with inter-agent collisions, 4096 envs (`tools/exp/hfh_run.py`, launch list "
              f"`profiles/r01_launches_hfh_{TAG}.csv`): the detection / island kernels beside the step.", "", "```"]
    lines += launches(hfh)
    lines += ["```", ""]
    shutil.copy(hfh, os.path.join(P, f"r01_launches_hfh_{TAG}.csv"))
with open(os.path.join(P, f"r01_k_env_step_{TAG}.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
shutil.copy(os.path.join(G, f"launches_{TAG}.csv"), os.path.join(P, f"r01_launches_{TAG}.csv"))

pol = os.path.join(G, f"prof_pol_{TAG}.ncu-rep")
if os.path.exists(pol):
    pl = [f"# Round 1 — ncu evidence for k_policy_mlp {TAG} (K4, tcgen05 policy/value forward)", "",
          "Command: `python -m pytest tests/test_gpu_policy.py -q -x -k 4096` (4096 envs, Humanoid nets "
          "76-256-128-64-{21,1}, bf16 operands, fp32 TMEM accumulators).",
          "Capture: `ncu --set full --clock-control none --import-source on -k regex:k_policy_mlp -c 1`.",
          "Grid: 32 env tiles x {pi, V} = 64 CTAs of 256 threads; weights by one TMA bulk copy each, issued before "
          "the coalesced observation prologue (nets too large for shared memory stream K-block chunks).", "", "```"]
    pl += sh(sys.executable, "tools/ncu_summary.py", pol, "--lines", "8").rstrip().splitlines()
    pl += ["```", ""]
    with open(os.path.join(P, f"r01_k_policy_mlp_{TAG}.md"), "w") as f:
        f.write("\n".join(pl) + "\n")
print("\n".join(lines[:40]))
