cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for g in 0 2048; do
  for c in c3 c4; do
    BS_STEP_G16_MAX_ENVS=$g timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --secondary "" > gpurun_out/g16_${g}_${c}.json 2>>gpurun_out/g16.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/g16_${g}_${c}.json').read().strip().splitlines()[-1]); print('g16max=$g $c', {k: round(v['us_per_launch'],1) for k,v in d['roofline']['kernels'].items()}, 'value=%.4g'%d['value'])"
  done
done
done
BS_STEP_G16_MAX_ENVS=100000 timeout 600 python -m pytest -q -x tests/test_step_gpu.py tests/test_scale_parity_gpu.py 2>&1 | tail -3
