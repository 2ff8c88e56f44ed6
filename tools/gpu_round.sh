#!/bin/bash
# One GPU session: GPU tests, bench (ours + reference arms), launch list, ncu captures of the
# step and render kernels.  Usage (under gpurun): bash tools/gpu_round.sh [tag] [skip-ref|run] [phase|full] [full]
# ("phase": k_step phase split; "full": also racecheck/memcheck and smoke())
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-run}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "$2" != "skip-ref" ]; then
  timeout 300 python bench.py --steps 50 --warmup 5 --impl reference > gpurun_out/${TAG}_bench_ref.json 2>> gpurun_out/${TAG}_bench.err
  for c in c3 c4 c5; do
    timeout 300 python bench.py --steps 5 --warmup 3 --impl reference --config $c > gpurun_out/${TAG}_bench_ref_$c.json 2>> gpurun_out/${TAG}_bench.err
  done
fi
for c in c4 c5; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --secondary "" > gpurun_out/${TAG}_bench_$c.json 2>> gpurun_out/${TAG}_bench.err
done
# multi-rank code path (2 ranks sharing this one GPU, gloo for the statistics collectives)
BENCH_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --secondary "" > gpurun_out/${TAG}_bench_2rank.json 2>> gpurun_out/${TAG}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --secondary c3 > /dev/null 2>> gpurun_out/${TAG}_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/${TAG}_prof_step python bench.py --steps 3 --warmup 3 --no-cpu --secondary "" > /dev/null 2>> gpurun_out/${TAG}_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render -s 3 -c 1 -o gpurun_out/${TAG}_prof_render python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --secondary "" > /dev/null 2>> gpurun_out/${TAG}_ncu.err
# issue / fp64 counters of the render kernel on C4 and C5 (tools/ncu_issue.py -> profiles/issue.json)
M=smsp__inst_executed.sum,smsp__cycles_elapsed.avg,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed
for c in c4 c5; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_render -s 3 -c 1 -o gpurun_out/${TAG}_issue_render_$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu --secondary "" > /dev/null 2>> gpurun_out/${TAG}_ncu.err
done
if [ "$3" == "phase" ]; then
  timeout 600 python tools/phase_timing.py 4096 50 > gpurun_out/${TAG}_phase.txt 2>&1
fi
if [ "$3" == "full" ] || [ "$4" == "full" ]; then
  bash tools/sanitize.sh ${TAG}
  python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.txt 2>&1
fi
echo done
