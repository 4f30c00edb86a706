timeout 100 python -m pytest tests -m gpu -x -q -k "tc or Tc or TC or smoke" 2>&1 | tail -2
for fl in 0; do echo "== dbg $fl"; timeout 100 python tools/trace_tc.py $fl > gpurun_out/trace_$fl.log 2>&1; grep -A2 "period\|X (saw\|saw S -> S\|S freed -> m\|m settled ->" gpurun_out/trace_$fl.log | cut -c1-200; done
timeout 200 python bench.py --serial --no-cpu-baseline > gpurun_out/bench_serial.log 2>&1; echo "bench serial exit $?"
for f in gpurun_out/bench_serial.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
  if l.startswith('{'):
    d=json.loads(l); print('us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, d['clocks'], d['config']['planner'], d['config'].get('tc_sm_budget'), d['config'].get('autotune_ms'))
  elif 'Error' in l or 'error' in l: print(l[:300])
"; done
