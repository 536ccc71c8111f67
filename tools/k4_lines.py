"""Stall samples / instructions of k_policy_mlp per policy_mlp.cu source line
from an `ncu --set full --import-source on` report, SASS rows aligned with
`nvdisasm -gi` of the same build (instructions inlined from helpers are
attributed to the policy_mlp.cu line they are inlined at).

usage: python tools/k4_lines.py REPORT.ncu-rep [--sass /tmp/k4_gi.sass]
(nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cubin
 -I include -I paper_1810_05762_b200/csrc paper_1810_05762_b200/csrc/policy_mlp.cu
 -o /tmp/k4.cubin && nvdisasm -gi /tmp/k4.cubin > /tmp/k4_gi.sass)"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
sass = sys.argv[sys.argv.index("--sass") + 1] if "--sass" in sys.argv else "/tmp/k4_gi.sass"
SRC = "/root/repo/paper_1810_05762_b200/csrc/policy_mlp.cu"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:k_policy"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
R = rows[2:]
ia = h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
fn = [p for p in re.split(r"//-+ \.text\.", open(sass).read()) if "k_policy_mlp" in p.split("\n", 1)[0]][0]
ins, cur, fresh = [], None, True
for ln in fn.splitlines():
    # nvdisasm -gi prints the inline chain innermost first: keep the first
    # policy_mlp.cu line of each group
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        f, l, fi, li = m.group(1), int(m.group(2)), m.group(3), m.group(4)
        if fresh:
            cur = l if f.endswith("policy_mlp.cu") else (int(li) if fi and fi.endswith("policy_mlp.cu") else -1)
            fresh = False
        continue
    fresh = True
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((cur, m.group(2).strip()))
assert len(ins) == len(R), (len(ins), len(R))
src = open(SRC).read().splitlines()
byl, bys, reasons = Counter(), Counter(), {}
for i, r in enumerate(R):
    l = ins[i][0]
    byl[l] += int(r[ia] or 0)
    bys[l] += int(r[ist] or 0)
    rc = reasons.setdefault(l, Counter())
    for c in cols:
        rc[h[c][6:]] += int(r[c] or 0)
tot = sum(bys.values())
print(f"stall samples {tot}")
for l, s in bys.most_common(int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30):
    why = ", ".join(f"{k} {v}" for k, v in reasons[l].most_common(2))
    txt = src[l - 1].strip()[:70] if l and l > 0 else ""
    print(f"{100 * s / tot:5.1f}% instr {byl[l]:>7}  L{l}: {txt}   [{why}]")
