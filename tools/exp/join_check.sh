# the accessor-ordering test on the build without the caller-stream join (expected to fail), then the fixed build
cp tools/exp/lib_sc.so paper_1810_05762_b200/libstampede_b200.so
timeout 300 python -m pytest tests/test_gpu.py -q -k accessors_order -p no:cacheprovider > gpurun_out/join_old.log 2>&1; echo "old build rc=$?"; tail -1 gpurun_out/join_old.log
cp tools/exp/lib_join.so paper_1810_05762_b200/libstampede_b200.so
for i in 1; do timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/join_full_$i.log 2>&1; echo "fixed full run $i rc=$?"; tail -1 gpurun_out/join_full_$i.log; grep FAILED gpurun_out/join_full_$i.log; done
timeout 600 python bench.py > gpurun_out/bench_join.json 2> gpurun_out/bench_join.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_join.json'));print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
