#!/bin/bash
# Render-only GPU session: raster parity tests, C3/C4/C5 bench lines, A/B knobs (512-thread CTAs,
# 64-pixel tiles), one ncu capture of k_render.  Usage (under gpurun): bash tools/gpu_render.sh tag
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=$1
timeout 600 python -m pytest tests/test_raster_stress_gpu.py tests/test_render_gpu.py tests/test_hetero_gpu.py tests/test_cabinet_gpu.py -q -x > gpurun_out/${T}_rtests.log 2>&1; echo "exit $?" >> gpurun_out/${T}_rtests.log
for c in c3 c4 c5; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --secondary "" > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err
done
BS_RENDER_THREADS=512 timeout 300 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu --secondary "" > gpurun_out/${T}_bench_c3_rt512.json 2>> gpurun_out/${T}_bench.err
BS_RENDER_TILE=64 timeout 300 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu --secondary "" > gpurun_out/${T}_bench_c3_t64.json 2>> gpurun_out/${T}_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render -s 3 -c 1 -o gpurun_out/${T}_prof_render python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --secondary "" > /dev/null 2>> gpurun_out/${T}_ncu.err
echo done
