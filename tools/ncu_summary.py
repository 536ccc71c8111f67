"""Summarise an ncu report: key metrics, opcode mix, top source lines."""
import csv, io, re, subprocess, sys
from collections import Counter

rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep] + list(a), capture_output=True, text=True).stdout

KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Waves Per SM", "DRAM Throughput", "L1/TEX Hit Rate", "Block Limit Registers",
        "Block Limit Shared Mem", "Dynamic Shared Memory Per Block", "Compute (SM) Throughput"]
r = csv.reader(io.StringIO(run("--page", "details", "--csv")))
h = next(r)
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for row in r:
    if row[mi] in KEYS:
        print(f"  {row[mi]:40s} {row[vi]} {row[ui]}")
raw = run("--page", "raw", "--csv")
r = list(csv.reader(io.StringIO(raw)))
if len(r) >= 3:
    names, vals = r[0], r[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_pipe_fma.sum",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
              "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"):
        if k in names:
            print(f"  {k:60s} {vals[names.index(k)]}")
    # warp stall reasons (cycles per issued instruction, largest first)
    pre = "smsp__average_warps_issue_stalled_"
    st = []
    for i, n in enumerate(names):
        if n.startswith(pre) and n.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(vals[i]), n[len(pre):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    if st:
        print("  stall reasons (cycles/issue): " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
if "--lines" in sys.argv:
    rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
    cur = None; hdr = None; agg = {}
    for row in rows:
        if row and row[0] == "File Path":
            cur = row[1].split("/")[-1]; continue
        if row and row[0] == "Line No":
            hdr = row; continue
        if hdr is None or not row or not row[0]:
            continue
        try:  # rows whose source text holds commas/quotes (inline asm) may not split cleanly
            ln = int(row[0])
            ie = int(float(row[hdr.index("Instructions Executed")] or 0))
            ws = int(float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
        except (ValueError, IndexError):
            continue
        agg[(cur, ln)] = (ie, ws, row[1].strip()[:80])
    tot = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[sys.argv.index("--lines") + 1])]:
        print(f"  {k[0]:16s}:{k[1]:4d} instr {v[0] / tot * 100:5.1f}% stall {v[1] / ts * 100:5.1f}%  {v[2]}")
