#!/bin/bash
# plain bench, then ncu --set full on one k_env_step launch (1 GPU)
TAG=${1:-cur}
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 8 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
