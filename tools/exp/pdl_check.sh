mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_pdl.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_pdl.log
for p in 1 0; do
  STP_PDL=$p timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/pdl_$p.json 2>gpurun_out/pdl.err
  python -c "import json;d=json.load(open('gpurun_out/pdl_$p.json'));r=d.get('rollout',{});print('PDL=$p step ms',round(d['ms_per_step'],4),'K4 us',round(1e3*r.get('policy_forward_ms',0),2),'rollout ms',r.get('ms_per_step'))"
done
K4SO=tools/exp/_k4phase.so python tools/exp/k4_phases.py run 2>&1 | tail -26 | head -25
