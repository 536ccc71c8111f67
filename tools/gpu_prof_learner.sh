#!/bin/bash
# PPO learner kernels: tests, update timing / kernel table, one ncu --set full
# capture of each learner kernel (k_ppo_head, k_ppo_finish, k_selu_bwd_bias,
# k_bias_selu) at 4096 envs x 32 frames (131 K-row minibatch).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ppo.py -q > gpurun_out/ppo_t.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ppo_t.log
timeout 600 python tools/exp/ppo_prof.py > gpurun_out/ppo_prof_final.log 2>&1; echo "prof rc=$?"
for k in k_ppo_head k_selu_bwd_bias k_bias_selu k_colsum_finish k_ppo_finish; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 \
    -o gpurun_out/prof_$k -f python tools/exp/ppo_prof.py > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
