#!/bin/bash
CMD="python -m pytest tests/test_gpu_policy.py -q -x -k 4096"
$CMD > gpurun_out/plain_pol.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_policy_mlp -c 1 -o gpurun_out/prof_policy $CMD > gpurun_out/ncu_pol.log 2>&1; echo "ncu rc=$?"
