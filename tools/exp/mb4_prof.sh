cp tools/exp/lib_mb4.so paper_1810_05762_b200/libstampede_b200.so
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_env_step -s 8 -c 1 -o gpurun_out/prof_mb4 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_mb4.log 2>&1; echo rc=$?
