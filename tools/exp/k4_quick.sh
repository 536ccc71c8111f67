# K4 quick loop: policy tests, phases, bench (rollout + K4)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_policy.py tests/test_gpu_ppo.py -x -q 2>&1 | tail -2
K4SO=tools/exp/_k4phase.so python tools/exp/k4_phases.py run 2>&1 | tail -26 | head -25
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/k4q.json 2>gpurun_out/k4q.err
python -c "import json;d=json.load(open('gpurun_out/k4q.json'));r=d.get('rollout',{});print('step ms',round(d['ms_per_step'],4),'K4 us',round(1e3*r.get('policy_forward_ms',0),2),'rollout ms',r.get('ms_per_step'))"
