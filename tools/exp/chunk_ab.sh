#!/bin/bash
# e2e A/B of the host-path chunk size (STP_HOST_MIN_CHUNK) on the configs below 4096 envs
for rep in 1 2; do for v in mc1024 mc512 mc256; do
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  for w in humanoid1024 humanoid4096; do
    python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', '$w', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,2))"
  done
done; done
cp tools/exp/lib_mc1024.so paper_1810_05762_b200/libstampede_b200.so
