#!/bin/bash
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 8 -c 1 -o gpurun_out/prof_${1:-x} $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
