#!/bin/bash
# compute-sanitizer racecheck (shared-memory hazards, incl. warp-level) and memcheck over the step
# and render kernels.  Usage (under gpurun): bash tools/sanitize.sh [tag]
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-san}
summ() { grep -o "[A-Za-z_]*\.cu[h]*:[0-9]*\|RACECHECK SUMMARY.*\|ERROR SUMMARY.*\|Potential [A-Z]* hazard" | sort | uniq -c | sort -rn; }
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 \
  python tools/sanitize_probe.py PickCube OpenCabinet PickHetero CartpoleBalance 2>&1 | summ > gpurun_out/${TAG}_racecheck.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/raster_probe.py 1 0 2>&1 | summ >> gpurun_out/${TAG}_racecheck.txt
# benchmark scale: >= 3 frames per persistent rasterizer CTA, a full 4096-env step wave
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_scale_probe.py 400 4096 2>&1 | summ > gpurun_out/${TAG}_racecheck_scale.txt
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_probe.py PickCube OpenCabinet PickHetero CartpoleBalance 2>&1 | summ > gpurun_out/${TAG}_memcheck.txt
timeout 900 compute-sanitizer --tool memcheck python tools/raster_probe.py 1 0 2>&1 | summ >> gpurun_out/${TAG}_memcheck.txt
timeout 1800 compute-sanitizer --tool memcheck python tools/sanitize_scale_probe.py 400 4096 2>&1 | summ > gpurun_out/${TAG}_memcheck_scale.txt
