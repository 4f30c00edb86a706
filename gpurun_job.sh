set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/trace_tc.py > gpurun_out/trace.log 2>&1; tail -4 gpurun_out/trace.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --serial --no-cpu-baseline > gpurun_out/bench_serial.log 2>&1; echo "bench serial exit $?"
for f in gpurun_out/bench_full.log gpurun_out/bench_serial.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
  if l.startswith('{'):
    d=json.loads(l); print('us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, d['clocks'], d['config']['planner'], d['config'].get('tc_sm_budget'), d['config'].get('autotune_ms'))
  elif 'Error' in l or 'error' in l: print(l[:300])
"; done
