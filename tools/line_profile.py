"""Execution-weighted instruction / stall counts per source line of the f32 W=32 CPB=2
step kernel: aligns `ncu --page source --print-source sass` rows of a report with
`nvdisasm -g` of the same build (tools/spills.sh writes /tmp/spill.sass).
usage: python tools/line_profile.py REPORT.ncu-rep [N] [--min-exec X] [--max-exec Y]"""
import csv, io, re, subprocess, sys
from collections import Counter
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
def opt(name, d):
    return float(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else d
lo, hi = opt("--min-exec", 0), opt("--max-exec", 1e30)
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]; R = rows[2:]
ia = h.index("Instructions Executed"); ist = h.index("Warp Stall Sampling (All Samples)")
txt = open('/tmp/spill.sass').read()
KERNEL = sys.argv[sys.argv.index('--kernel') + 1] if '--kernel' in sys.argv else '_ZN3stp10k_env_stepIfLi32ELi2ELb0E'
fn = [p for p in re.split(r'//-+ \.text\.', txt) if p.startswith(KERNEL)][0]
ins = []; cur = None
for ln in fn.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
    if m:
        ins.append((cur, m.group(2).strip()))
assert len(ins) == len(R), (len(ins), len(R))
nw = int(R[0][ia])  # first instruction runs once per warp
byline = Counter(); stl = Counter(); tot = 0
for i in range(len(R)):
    n = int(R[i][ia])
    tot += n
    if not (lo * nw <= n <= hi * nw):
        continue
    byline[ins[i][0]] += n; stl[ins[i][0]] += int(R[i][ist])
print(f"warps {nw}  instr/warp {tot / nw:.0f}  selected/warp {sum(byline.values()) / nw:.0f}")
root = '/root/repo/paper_1810_05762_b200/csrc/'
srcs = {}
for k, v in byline.most_common(N):
    f = k[0] if k else None
    if f and f not in srcs:
        try:
            srcs[f] = open(root + f).read().splitlines()
        except OSError:
            srcs[f] = []
    s = srcs[f][k[1] - 1].strip()[:80] if f and len(srcs[f]) >= k[1] else ''
    print(f"{v / nw:7.1f} {stl[k]:5d} {f}:{k[1] if k else 0}  {s}")
