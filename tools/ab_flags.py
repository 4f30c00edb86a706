"""A/B of launch flags on a config's prepared step (the bench's plan and
autotuned budget), alternating variants over rounds, medians.

    python tools/ab_flags.py config rounds flagsA flagsB ...
"""
import os, statistics, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

config, rounds, variants = sys.argv[1], int(sys.argv[2]), [int(x) for x in sys.argv[3:]]
ns = bench.prepare(config, torch.device("cuda", 0))
steps = {f: ns.step.with_budget(ns.budget, flags=ns.step.flags | f) for f in variants}
res = {f: [] for f in variants}
for rnd in range(rounds):
    for f in variants:
        st = steps[f]
        g = st.capture(ns.q_dev, ns.kp, ns.vp, ns.out) if rnd == 0 else st._replay
        st._replay = g
        for _ in range(5):
            g()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            g()
        e1.record()
        torch.cuda.synchronize()
        res[f].append(e0.elapsed_time(e1) / 200 * 1e3)
print(config, "budget", ns.budget)
for f in variants:
    print(f"  flags {f:8d}: {statistics.median(res[f]):7.1f} us  {[round(x, 1) for x in res[f]]}")
