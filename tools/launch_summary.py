"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:60]
    v = float(r[vi].replace(",", ""))
    unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "ns"
    if unit in ("usecond", "us"):
        v *= 1e3
    elif unit in ("msecond", "ms"):
        v *= 1e6
    tot[name] += v; cnt[name] += 1
all_t = sum(tot.values())
print(f"{'kernel':62s} {'launches':>8s} {'mean us':>9s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:62s} {cnt[k]:8d} {tot[k] / cnt[k] / 1e3:9.2f} {tot[k] / all_t * 100:6.1f}%")
