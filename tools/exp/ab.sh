#!/bin/bash
# A/B: run bench with alternative builds of the library
for v in ${VARIANTS:-classic pipe}; do
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
done
