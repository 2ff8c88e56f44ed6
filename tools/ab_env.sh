# A/B of an env-var knob on the C2/C3 bench lines, interleaved.  Usage (gpurun): bash tools/ab_env.sh VAR "v1 v2" "c2 c3"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for c in ${3:-c2}; do
  for v in $2; do
    env $1=$v timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --secondary "" > gpurun_out/abe_${v}_${c}.json 2>>gpurun_out/abe.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/abe_${v}_${c}.json').read().strip().splitlines()[-1]); print('$1=$v $c', {k: round(v['us_per_launch'],1) for k,v in d['roofline']['kernels'].items()}, 'value=%.4g'%d['value'], 'e2e=%.4g'%d['e2e']['value'])"
  done
done
done
