#!/bin/bash
# Round profile evidence (1 GPU): plain bench -> ncu launch list of the same
# command -> ncu --set full on one k_env_step launch -> ncu --set full on one
# k_policy_mlp launch (4096-env policy test).  Each ncu pass only after the same
# command exited 0 without ncu.
TAG=${1:-cur}
CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 8 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full rc=$?"
PCMD="python -m pytest tests/test_gpu_policy.py -q -x -k 4096"
$PCMD > gpurun_out/plain_pol_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_policy_mlp -c 1 -o gpurun_out/prof_pol_$TAG $PCMD > gpurun_out/ncu_pol_$TAG.log 2>&1; echo "policy rc=$?"
