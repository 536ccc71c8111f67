#!/bin/bash
# one GPU iteration: parity tests, then the bench line
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_cycle.json 2> gpurun_out/bench_cycle.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cycle.json'));print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],'kry',d['roofline']['krylov_iters_per_env_step'])"
