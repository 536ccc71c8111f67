"""Record per-launch DRAM traffic of a kernel from an `ncu --set full` capture
into profiles/traffic.json (bench.py reports it as roofline.traffic).
usage: python tools/ncu_traffic.py REPORT.ncu-rep KERNEL_KEY CAPTURE_NOTE"""
import csv, io, json, os, subprocess, sys

rep, key, note = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
names, units, vals = r[0], r[1], r[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def get(m):
    i = names.index(m)
    return float(vals[i].replace(",", "")) * scale[units[i]]
def dur():
    i = names.index("gpu__time_duration.sum")
    return float(vals[i].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
                                               "msecond": 1e3}[units[i]]
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
d = json.load(open(out_path)) if os.path.exists(out_path) else {}
d[key] = {"dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum"),
          "duration_us": dur(),
          "capture": note}
json.dump(d, open(out_path, "w"), indent=1)
print(key, d[key])
