#!/bin/bash
TAG=${1:-split}
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_solve -s 8 -c 1 -o gpurun_out/prof_${TAG}_solve $CMD > /dev/null 2>&1; echo "solve rc=$?"
