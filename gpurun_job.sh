set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -25 gpurun_out/pytest_gpu.log
for m in 18 37; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks $m > gpurun_out/bench_m$m.log 2>&1; echo "bench m=$m exit $?"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 37 --serial > gpurun_out/bench_serial37.log 2>&1; echo "bench serial exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_pac -s 2 -c 1 -o gpurun_out/prof_tc8 python bench.py --quick --serial --steps 2 --warmup 3 --blocks 37 > gpurun_out/ncu_tc.log 2>&1; echo "ncu tc exit $?"
for f in gpurun_out/bench_*.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
  if l.startswith('{'):
    d=json.loads(l); print('us/step %.1f GB/s %.0f'%(d['us_per_step'],d['value']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, d['clocks'], d['config']['planner'], d['config'].get('tc_sm_budget'), d['config'].get('autotune_ms'))
  elif 'Error' in l or 'error' in l: print(l[:300])
"; done
