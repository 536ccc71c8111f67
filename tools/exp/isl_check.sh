# island launch changes: interagent tests, HFH bench + rollout (uncrowded 50 steps, crowded 100 steps)
timeout 900 python -m pytest tests/test_gpu_interagent.py -x -q > gpurun_out/isl_t.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/isl_t.log
for st in 50 100; do for w in hfh4096 hfh_terrain4096; do
  timeout 600 python bench.py --workload $w --steps $st --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('rollout',{});print('steps=$st $w', round(d['ms_per_step'],4), 'rollout', round(r.get('ms_per_step'),4))"
done; done
