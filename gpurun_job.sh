mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
CMD="python bench.py --quick --steps 4 --warmup 3"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_pac -s 2 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1; echo "tc exit $?"
