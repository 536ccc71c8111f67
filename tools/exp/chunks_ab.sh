# host-path chunk count with direct obs writes: e2e of the default bench
for rep in 1 2; do for v in c1 c2 c4; do
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v e2e', round(d['e2e']['value']/1e6,2))"
done; done
cp tools/exp/lib_c4.so paper_1810_05762_b200/libstampede_b200.so
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "host" 2>&1 | tail -1
