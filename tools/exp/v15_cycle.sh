timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_v15.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_v15.json 2> gpurun_out/bench_v15.err; echo "bench rc=$?"; cat gpurun_out/bench_v15.json
bash tools/gpu_profile_round.sh v15
