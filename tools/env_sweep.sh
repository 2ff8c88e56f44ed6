#!/bin/bash
# Throughput against envs per GPU (one B200): bench lines of C2 (state) and C3 (rgb+depth 128^2)
# at several env counts, device `value` and e2e.  Usage (under gpurun): bash tools/env_sweep.sh TAG
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-sweep}
for n in 1024 2048 4096 8192 16384 32768 65536; do
  timeout 300 python bench.py --config c2 --envs $n --steps 100 --warmup 5 --no-cpu --secondary "" | tail -1 >> gpurun_out/${TAG}_c2.jsonl 2>> gpurun_out/${TAG}.err
done
for n in 256 512 1024 2048 4096 8192; do
  timeout 300 python bench.py --config c3 --envs $n --steps 30 --warmup 5 --no-cpu --secondary "" | tail -1 >> gpurun_out/${TAG}_c3.jsonl 2>> gpurun_out/${TAG}.err
done
