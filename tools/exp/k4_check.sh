# K4 iteration: phase timelines of the variants in $K4V (tools/exp/_k4ph_<v>.so),
# then for each library in $K4LIBS (tools/exp/lib_<v>.so): policy tests + bench K4 / rollout timing
mkdir -p gpurun_out
for v in ${K4V:-s0}; do echo "== phases $v"; K4SO=tools/exp/_k4ph_$v.so python tools/exp/k4_phases.py run 2>&1 | tail -26 | head -25; done
cp paper_1810_05762_b200/libstampede_b200.so /tmp/lib_default.so
for v in ${K4LIBS:-}; do
  echo "== lib $v"
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  timeout 600 python -m pytest tests/test_gpu_policy.py -x -q 2>&1 | tail -2
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/k4_bench_$v.json 2>gpurun_out/k4_bench.err
  python -c "import json;d=json.load(open('gpurun_out/k4_bench_$v.json'));r=d.get('rollout',{});print('step ms',round(d['ms_per_step'],4),'K4 us',round(1e3*r.get('policy_forward_ms',0),2),'rollout ms',r.get('ms_per_step'))"
done
cp /tmp/lib_default.so paper_1810_05762_b200/libstampede_b200.so
