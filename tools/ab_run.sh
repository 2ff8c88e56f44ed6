#!/bin/bash
# Same-box library A/B: for each "lib:configs" argument, bench lines with BS_LIB_PATH=ab/<lib>.so,
# the whole list repeated REPS times (interleaved, so box drift shows up).
# Usage (under gpurun): STEPS=200 REPS=2 bash tools/ab_run.sh TAG lib1:c2,c3 lib2:c3 ...
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=$1; shift
for rep in $(seq 1 ${REPS:-2}); do
  for spec in "$@"; do
    n=${spec%%:*}; cfgs=${spec#*:}
    for c in ${cfgs//,/ }; do
      out=gpurun_out/${TAG}_${n}_${c}_$rep.json
      BS_LIB_PATH=$PWD/ab/$n.so timeout 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-cpu --secondary "" > $out 2>> gpurun_out/${TAG}.err
      python - "$n $c #$rep" $out <<'PY'
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
