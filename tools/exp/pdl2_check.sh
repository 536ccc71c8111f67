mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_pdl2.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_pdl2.log
python tools/exp/hfh_timeline.py 2>&1 | tail -22
for w in hfh4096 humanoid4096 hfh_terrain4096; do for p in 1 0; do
  STP_PDL=$p timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('rollout',{});print('$w PDL=$p', round(d['ms_per_step'],4), round(d['value']/1e6,2), 'rollout', r.get('ms_per_step'))"
done; done
