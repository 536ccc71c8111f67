for rep in 1 2; do for v in head new; do
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  python bench.py --workload hfh4096 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,2))"
done; done
cp tools/exp/lib_new.so paper_1810_05762_b200/libstampede_b200.so
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_interagent.py -x -q -k "host or inter or island" > gpurun_out/e2e_t.log 2>&1; tail -1 gpurun_out/e2e_t.log
