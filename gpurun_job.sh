mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?"
python -c "
import json
for l in open('gpurun_out/bench.log'):
  if l.startswith('{'):
    d=json.loads(l); print('us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'], 'e2e', d['e2e'])
"
tail -3 gpurun_out/bench.log | grep -i error
