#!/bin/bash
# Render-only library A/B on one box: tools/render_bench.py for each ab/*.so, three rounds
# interleaved.  Usage: gpu_render_lib_ab.sh [configs] [steps]
cd "$GRAFT_REPO_ROOT"
for rep in 1 2 3; do
  for so in ab/*.so; do
    for c in ${1:-c3 c5}; do
      BS_LIB_PATH=$PWD/$so timeout 300 python tools/render_bench.py $c 1024 ${2:-30} 200 2>&1 | tail -1
    done
  done
done
