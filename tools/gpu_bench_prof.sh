#!/bin/bash
# bench (plain) -> ncu launch list -> ncu --set full on the step kernel
set -x
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
python bench.py --steps 200 --warmup 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 8 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
