# compute-sanitizer on the rollback test, current build and the sincospi build where it failed
T="tests/test_gpu.py -q -x -k rolled_back -p no:cacheprovider"
for tool in initcheck racecheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $T > gpurun_out/san_${tool}_cur.log 2>&1; echo "cur $tool rc=$?"; grep -m5 "ERROR SUMMARY\|Uninitialized\|hazard\|Invalid" gpurun_out/san_${tool}_cur.log
done
cp tools/exp/lib_scpi.so paper_1810_05762_b200/libstampede_b200.so
python -m pytest $T > gpurun_out/scpi_plain.log 2>&1; echo "scpi plain rc=$?"
for tool in initcheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $T > gpurun_out/san_${tool}_scpi.log 2>&1; echo "scpi $tool rc=$?"; grep -m5 "ERROR SUMMARY\|Uninitialized\|hazard\|Invalid" gpurun_out/san_${tool}_scpi.log
done
