#!/bin/bash
# end-of-round GPU cycle: smoke, GPU tests, bench (+ reference arm), launch list,
# every BASELINE config, fp32 parity report.  usage: STP_BUILD=<sha> bash tools/final_cycle.sh
mkdir -p gpurun_out
bash tools/gpu_round_cycle.sh
bash tools/gpu_configs.sh
timeout 1500 python tools/parity_report.py --out gpurun_out/r02_parity.json > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/parity.log
