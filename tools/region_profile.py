"""Per-phase instruction and stall-sample breakdown of the f32 W=32 CPB=2 step
kernel from an `ncu --set full --import-source on` report.  SASS rows of the
report are aligned with `nvdisasm -gi` of the same build; each instruction is
attributed to the sim_step.cuh line it was inlined at (else its own line), and
lines to the kernel phases marked by "// ---- ..." comments in sim_step.cuh.

usage: python tools/region_profile.py REPORT.ncu-rep [--sass /tmp/step_gi.sass]
(build the sass: nvcc ... -cubin sim_step_f32.cu -o step.cubin; nvdisasm -gi step.cubin)"""
import csv
import io
import os
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
sass = sys.argv[sys.argv.index("--sass") + 1] if "--sass" in sys.argv else "/tmp/step_gi.sass"
KERNEL = os.environ.get("KERNEL", "_ZN3stp10k_env_stepIfLi32ELi2ELb0ELb0E")  # Lb1: the island instantiation
SRC = "/root/repo/paper_1810_05762_b200/csrc/sim_step.cuh"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:k_env_step"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# one section per captured launch ("Kernel Name" row, header row, SASS rows): NCU_SECTION picks one
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sec = int(os.environ.get("NCU_SECTION", "0"))
h = rows[starts[sec] + 1]
R = [r for r in rows[starts[sec] + 2:starts[sec + 1]] if r]
ia = h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
txt = open(sass).read()
fn = [p for p in re.split(r"//-+ \.text\.", txt) if p.startswith(KERNEL)][0]
INNER = "--inner" in sys.argv  # the innermost sim_step.cuh line of the inline chain (lambdas), not the outermost
ins, cur, fresh = [], None, True
for ln in fn.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        f, l, fi, li = m.group(1), int(m.group(2)), m.group(3), m.group(4)
        if INNER and not fresh:
            continue
        fresh = False
        if f.endswith("sim_step.cuh"):
            cur = l  # the step body is one inlined function: its own line is the useful one
        elif fi and fi.endswith("sim_step.cuh"):
            cur = int(li)
        else:
            cur = -1
        continue
    fresh = True
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((cur, m.group(2).strip()))
assert len(ins) == len(R), (len(ins), len(R))
src = open(SRC).read().splitlines()
marks = [(i + 1, re.sub(r"\s*[-=]{3,}.*", "", ln.split("// ----------------")[-1]).strip(" -"))
         for i, ln in enumerate(src) if "// ----------------" in ln or "// ---- " in ln]


def region(line):
    if line is None or line < 0:
        return "(other files / not inlined)"
    name = "(kernel prologue / helpers)"
    for l, nm in marks:
        if l <= line:
            name = f"{l}: {nm[:60]}"
    return name


nw = int(R[0][ia])
inst, stall, tot, tst = Counter(), Counter(), 0, 0
for i, r in enumerate(R):
    n, st = int(r[ia]), int(r[ist])
    g = region(ins[i][0])
    inst[g] += n
    stall[g] += st
    tot += n
    tst += st
print(f"warps {nw}  instructions/warp {tot / nw:.0f}  stall samples {tst}")
for g, n in sorted(inst.items(), key=lambda kv: -kv[1]):
    print(f"{n / nw:8.0f} instr/warp {100 * n / tot:5.1f}%  stalls {100 * stall[g] / max(1, tst):5.1f}%  {g}")

if "--lines" in sys.argv:
    lo, hi = map(int, sys.argv[sys.argv.index("--lines") + 1].split(":"))
    byl, bys = Counter(), Counter()
    for i, r in enumerate(R):
        l = ins[i][0]
        if l is not None and lo <= l <= hi:
            byl[l] += int(r[ia])
            bys[l] += int(r[ist])
    for l, n in sorted(byl.items()):
        if n / nw >= 20:
            print(f"{n / nw:8.0f} {100 * bys[l] / max(1, tst):5.1f}%  {l}: {src[l - 1].strip()[:90]}")

if "--stalls" in sys.argv:
    # stall reasons of the instructions executed >= 40x per warp (the PCR loop)
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    acc = Counter()
    loop_inst = 0
    for i, r in enumerate(R):
        if int(r[ia]) >= 40 * nw:
            loop_inst += int(r[ia])
            for c in cols:
                acc[h[c]] += int(r[c] or 0)
    tot_s = sum(acc.values())
    print(f"hot loop: {loop_inst / nw:.0f} instr/warp; stall samples {tot_s}")
    for k, v in acc.most_common(12):
        print(f"  {k:24s} {100 * v / tot_s:5.1f}%  ({v / max(1, loop_inst / nw * 0 + 1):.0f})")
    # and per opcode class in the loop
    byop = Counter()
    for i, r in enumerate(R):
        if int(r[ia]) >= 40 * nw:
            op = ins[i][1].split()[0]
            if op.startswith("@"):
                op = ins[i][1].split()[1]
            byop[op.split(".")[0]] += int(r[ist])
    print("  stall samples by opcode (of the stalled instruction):",
          ", ".join(f"{k} {100 * v / max(1, sum(byop.values())):.0f}%" for k, v in byop.most_common(10)))

if "--spills" in sys.argv:
    # executed local-memory instructions (LDL / STL) per source line
    byl = Counter()
    for i, r in enumerate(R):
        op = ins[i][1]
        if "LDL" in op or "STL" in op:
            byl[ins[i][0]] += int(r[ia])
    tot_sp = sum(byl.values())
    print(f"spill instructions executed per warp: {tot_sp / nw:.0f}")
    for l, n in byl.most_common(25):
        txt = src[l - 1].strip()[:80] if l and l > 0 else ""
        print(f"{n / nw:8.1f}  {l}: {txt}  [{region(l)}]")
