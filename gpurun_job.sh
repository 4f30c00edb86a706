mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python tools/ctalog.py 148 4096 > gpurun_out/ctalog_fused.log 2>&1; echo "ctalog exit $?"
timeout 300 python bench.py --serial --no-cpu-baseline --steps 10 > gpurun_out/bench_serial.log 2>&1; echo "bench exit $?"
for f in gpurun_out/bench_serial.log; do python -c "
import json,sys
for l in open('$f'):
  if l.startswith('{'):
    d=json.loads(l); print('us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, d['clocks'], d['config'].get('tc_sm_budget'), d['config'].get('autotune_ms'))
"; tail -2 $f | grep -i error; done
