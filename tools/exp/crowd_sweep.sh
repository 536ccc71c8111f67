# HFH: island side-stream priority threshold (STP_ISL_CROWD) vs bench step and rollout
for c in 0 24 64 1000000; do for w in hfh4096 hfh_terrain4096; do
  STP_ISL_CROWD=$c timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('rollout',{});print('crowd=$c $w', round(d['ms_per_step'],4), round(d['value']/1e6,2), 'rollout', round(r.get('ms_per_step'),4))"
done; done
