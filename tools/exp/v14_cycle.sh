timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v14a.log 2>&1; echo "pytest a rc=$?"; tail -2 gpurun_out/pytest_v14a.log
timeout 900 python -m pytest tests/test_gpu.py -q -k "rolled_back or parity" > gpurun_out/pytest_v14b.log 2>&1; echo "pytest b rc=$?"; tail -2 gpurun_out/pytest_v14b.log
timeout 600 python bench.py > gpurun_out/bench_v14.json 2> gpurun_out/bench_v14.err; echo "bench rc=$?"; cat gpurun_out/bench_v14.json
bash tools/gpu_profile_round.sh v14
