# A/B of step-kernel builds (tools/exp/lib_*.so), then the GPU tests and the config sweep on the last
VARIANTS="${VARIANTS:-v13 sc}" bash tools/exp/ab.sh
cp tools/exp/lib_${LAST:-sc}.so paper_1810_05762_b200/libstampede_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${LAST:-sc}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${LAST:-sc}.log
timeout 300 python tools/exp/configs.py > gpurun_out/configs_${LAST:-sc}.log 2>&1; tail -12 gpurun_out/configs_${LAST:-sc}.log
