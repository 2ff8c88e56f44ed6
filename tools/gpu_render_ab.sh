#!/bin/bash
# Rasterizer A/B: C3 / C5 bench lines under the launch knobs (tile, threads, smem budget).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-ab}
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c3} --steps 30 --warmup 3 --no-cpu --secondary "" > gpurun_out/${TAG}_${name}.json 2>> gpurun_out/${TAG}.err
  python - "$name" gpurun_out/${TAG}_${name}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    k = d["roofline"]["kernels"]
    print(sys.argv[1], {n: round(v["us_per_launch"], 1) for n, v in k.items()}, "value=%.3g" % d["value"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
}
run base X=1
run b110_t512 BS_RENDER_BUDGET=112000 BS_RENDER_THREADS=512
run b72_t512 BS_RENDER_BUDGET=74000 BS_RENDER_THREADS=512
run b110_t512_tile64 BS_RENDER_BUDGET=112000 BS_RENDER_THREADS=512 BS_RENDER_TILE=64
CFG=c5 run c5_base X=1
CFG=c5 run c5_b110_t512 BS_RENDER_BUDGET=112000 BS_RENDER_THREADS=512
