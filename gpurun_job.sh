mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_gpu.log; grep -E "^E  " gpurun_out/pytest_gpu.log | head -3
for fl in 0 768; do
timeout 300 python bench.py --quick --no-graph --steps 10 --flags $fl > gpurun_out/bench_fl$fl.log 2>&1
python -c "
import json
for l in open('gpurun_out/bench_fl$fl.log'):
  if l.startswith('{'):
    d=json.loads(l); print('flags $fl us/step %.1f'%(d['us_per_step']), {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()})
"
tail -2 gpurun_out/bench_fl$fl.log | grep -i error
done
