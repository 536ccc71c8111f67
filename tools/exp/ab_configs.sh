#!/bin/bash
# A/B of tools/exp/configs.py for alternative library builds
for v in ${VARIANTS:-a b}; do
  cp tools/exp/lib_$v.so paper_1810_05762_b200/libstampede_b200.so
  python tools/exp/configs.py 2>&1 | grep -E "n  |n [0-9]" | sed "s/^/$v /"
done
