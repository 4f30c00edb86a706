mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?"
python -c "
import json
for l in open('gpurun_out/bench.log'):
  if l.startswith('{'):
    d=json.loads(l); print('us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, d['kernels_window_ms_per_step'], d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value']))
"
tail -2 gpurun_out/bench.log | grep -i error
