#!/usr/bin/env python3
"""Print a compact table of a parity report JSON (tools/parity_report.py)."""
import json
import sys


def fmt(s):
    return " ".join(f"{k}={v:.2e}" if isinstance(v, float) else f"{k}={v}" for k, v in s.items())


def main(path):
    d = json.load(open(path))
    for name, v in d["protocols"].items():
        print("==", name)
        for k, vv in v.items():
            if isinstance(vv, dict) and "gpu" in vv and isinstance(vv["gpu"], dict):
                print(f"  {k:12s} gpu: {fmt(vv['gpu'])}")
                if vv.get("f32", {}).get("n"):
                    print(f"  {'':12s} f32: {fmt(vv['f32'])}")
            else:
                print(f"  {k}: {vv}")


if __name__ == "__main__":
    main(sys.argv[1])
