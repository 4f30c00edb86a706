#!/usr/bin/env bash
# Round-end measurement on one B200 (run from the repo root under gpurun):
# bench lines for every config, the reference arm, the ncu launch list of
# the cfg2 bench command and per-kernel ncu --set full captures at each
# config's benchmarked tensor-core SM budget (-> profiles/ncu_summary*).
set -u
OUT=gpurun_out/measure
mkdir -p $OUT
for c in cfg2 cfg3 cfg5 cfg1 cfg4; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv \
  python bench.py --quick --steps 2 --warmup 1 > $OUT/launches_bench.log 2>&1
echo "launches rc=$?"
for c in cfg2 cfg3 cfg5 cfg4; do
  b=$(python -c "import json;print(json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1])['config']['tc_sm_budget'])" 2>/dev/null || echo 96)
  f=$(python -c "import json;print(0 if json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1])['config']['lightly_shared'].startswith('transposed') else 4194304)" 2>/dev/null || echo 0)
  timeout 900 ncu --set full --profile-from-start off --clock-control none --import-source on \
    -o $OUT/ncu_$c python tools/ncu_step.py $c $b $f > $OUT/ncu_$c.log 2>&1
  echo "ncu $c budget $b rc=$?"
  echo "$b" > $OUT/budget_$c.txt
done
