# repeat the GPU suite on the current build, then the sincospi build (where the rollback test failed once)
for i in 1 2 3; do timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/stress_cur_$i.log 2>&1; echo "cur run $i rc=$?"; tail -1 gpurun_out/stress_cur_$i.log; done
cp tools/exp/lib_scpi.so paper_1810_05762_b200/libstampede_b200.so
for i in 1 2; do timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/stress_scpi_$i.log 2>&1; echo "scpi run $i rc=$?"; tail -1 gpurun_out/stress_scpi_$i.log; grep FAILED gpurun_out/stress_scpi_$i.log; done
