timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_v16.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_v16.json 2> gpurun_out/bench_v16.err; echo "bench rc=$?"; cat gpurun_out/bench_v16.json
bash tools/gpu_profile_round.sh v16
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_v16.json 2>/dev/null; echo "ref rc=$?"
