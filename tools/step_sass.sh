#!/bin/bash
# nvdisasm -gi of the fp32 step TU as build.py compiles it (for tools/region_profile.py)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -cubin -ftz=true -prec-div=false -prec-sqrt=false \
  -I/root/repo/include -I/root/repo/paper_1810_05762_b200/csrc /root/repo/paper_1810_05762_b200/csrc/sim_step_f32.cu \
  -o /tmp/step.cubin && nvdisasm -gi /tmp/step.cubin > /tmp/step_gi.sass && echo "/tmp/step_gi.sass"
