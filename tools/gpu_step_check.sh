#!/bin/bash
# Step-kernel change check: parity tests, then C2 / C4 timing.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-sc}
timeout 900 python -m pytest -q -x tests/test_step_gpu.py tests/test_scale_parity_gpu.py tests/test_controllers_gpu.py tests/test_cabinet_gpu.py tests/test_hetero_gpu.py > gpurun_out/${TAG}_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/${TAG}_tests.log
for c in c2 c4; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --secondary "" > gpurun_out/${TAG}_$c.json 2>> gpurun_out/${TAG}.err
  python - $c gpurun_out/${TAG}_$c.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], {n: round(v["us_per_launch"], 1) for n, v in d["roofline"]["kernels"].items()}, "value=%.4g" % d["value"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
