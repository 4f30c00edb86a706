"""A/B of library variants with alternation: each round runs every variant
once (subprocess: tensor-core kernel alone at a fixed SM budget, 200 calls,
and the full step at that budget), medians over rounds.

    python tools/ab_rounds.py rounds budget tag1 tag2 ...   (tag '-' = default library;
    tag@N also sets CODEC_TC_UNIT_COST=N)
"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import math, sys, json, torch
sys.path.insert(0, %r)
import bench
budget = %d
ns = bench.prepare("cfg2", torch.device("cuda", 0), budgets=[budget])
def t(step, n=200):
    for _ in range(5): step(ns.q_dev, ns.kp, ns.vp, out=ns.out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): step(ns.q_dev, ns.kp, ns.vp, out=ns.out)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
tc = ns.step.with_budget(budget, flags=8 | 32 | 64)
print(json.dumps({"tc_us": t(tc), "step_us": t(ns.step)}))
'''
rounds, budget, tags = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3:]
res = {t: [] for t in tags}
for r in range(rounds):
    for tag in tags:
        env = dict(os.environ)
        lib, _, cost = tag.partition("@")
        if cost:
            env["CODEC_TC_UNIT_COST"] = cost
        if lib != '-':
            env["CODEC_B200_LIB"] = os.path.join(ROOT, "paper_2505_17694_b200", f"_codec_b200_{lib}.so")
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, budget)], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        res[tag].append(json.loads(line[-1]) if line else {"err": out.stderr[-300:]})
for tag in tags:
    ok = [x for x in res[tag] if "tc_us" in x]
    if not ok:
        print(tag, res[tag]); continue
    print(f"{tag:10s} tc {statistics.median(x['tc_us'] for x in ok):7.1f} us  step {statistics.median(x['step_us'] for x in ok):7.1f} us  "
          f"(tc {[round(x['tc_us'],1) for x in ok]}, step {[round(x['step_us'],1) for x in ok]})")
