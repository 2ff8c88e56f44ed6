# A/B of the k_step lanes per env (BS_STEP_G) over workloads.  Usage (gpurun): bash tools/ab_g.sh "c4 c5"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for c in ${1:-c4}; do
  for g in 8 16 32; do
    BS_STEP_G=$g timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --secondary "" > gpurun_out/abg_${g}_${c}.json 2>>gpurun_out/abg.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/abg_${g}_${c}.json').read().strip().splitlines()[-1]); print('G=$g $c', {k: round(v['us_per_launch'],1) for k,v in d['roofline']['kernels'].items()}, 'value=%.4g'%d['value'])"
  done
done
done
