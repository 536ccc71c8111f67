mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_inline.log 2>&1; echo tests rc=$? 
tail -3 gpurun_out/t_inline.log
VARIANTS="base mb4" bash tools/exp/ab.sh
bash tools/exp/mb4_prof.sh
cp tools/exp/lib_base.so paper_1810_05762_b200/libstampede_b200.so
