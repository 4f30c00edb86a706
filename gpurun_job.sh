mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_gpu.log
for c in cfg1 cfg2 cfg3; do
timeout 400 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_$c.log 2>&1; echo "bench $c exit $?"
python -c "
import json
for l in open('gpurun_out/bench_$c.log'):
  if l.startswith('{'):
    d=json.loads(l); print('$c us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, 'budget', d['config']['tc_sm_budget'], min(d['config']['autotune_ms'].values()), 'e2e', round(d['e2e']['value']))
"
tail -2 gpurun_out/bench_$c.log | grep -i error
done
