#!/bin/bash
# Library A/B on one box: C2 / C4 bench lines for each ab/*.so (BS_LIB_PATH), interleaved
# twice so box drift shows up.  Usage: gpu_lib_ab.sh TAG [configs]
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-lab}; CFGS=${2:-c2 c4}
for rep in 1 2; do
  for so in ab/*.so; do
    n=$(basename $so .so)
    for c in $CFGS; do
      BS_LIB_PATH=$PWD/$so timeout 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-cpu --secondary "" > gpurun_out/${TAG}_${n}_${c}_$rep.json 2>> gpurun_out/${TAG}.err
      python - "$n $c #$rep" gpurun_out/${TAG}_${n}_${c}_$rep.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], {k: round(v["us_per_launch"], 1) for k, v in d["roofline"]["kernels"].items()}, "value=%.4g" % d["value"], "e2e=%.4g" % (d.get("e2e") or {}).get("value", 0))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
    done
  done
done
