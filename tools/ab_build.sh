#!/bin/bash
# Build variant libraries for A/B timing: tools/ab_build.sh name "-DFLAG=1 ..." [name2 "flags2" ...]
# -> tools/exp/lib_<name>.so (then: VARIANTS="a b" bash tools/exp/ab.sh on the GPU box)
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  STP_NVCC_EXTRA="$2" python paper_1810_05762_b200/build.py > /dev/null
  cp paper_1810_05762_b200/libstampede_b200.so tools/exp/lib_$1.so
  echo "built tools/exp/lib_$1.so ($2)"
  shift 2
done
python paper_1810_05762_b200/build.py > /dev/null  # restore the default build
