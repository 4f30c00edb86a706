mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 400 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
CMD="python bench.py --quick --steps 4 --warmup 3"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_pac -s 2 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1; echo "tc exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mma_pac -s 2 -c 1 -o gpurun_out/prof_mma $CMD > gpurun_out/ncu_mma.log 2>&1; echo "mma exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge -s 2 -c 1 -o gpurun_out/prof_merge $CMD > gpurun_out/ncu_merge.log 2>&1; echo "merge exit $?"
timeout 300 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_gpu.log
