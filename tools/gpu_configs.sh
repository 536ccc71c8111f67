#!/bin/bash
# every BASELINE config through bench.py (same methodology), one JSON line each
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for w in humanoid4096 ant64 humanoid1024 hfh4096 hfh_terrain4096; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 10 2>gpurun_out/cfg_$w.err >> gpurun_out/configs.jsonl; echo "$w rc=$?"
done
