#!/bin/bash
# A/B of the e2e figure for alternative library builds
for v in ${VARIANTS:-c1 c4}; do
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,3), 'M/s', 'e2e ms', round(4096/d['e2e']['value']*1e3,4))"
done
