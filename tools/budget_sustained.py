"""cfg2 step time per tensor-core SM budget in sustained (power-capped)
conditions: >= `seconds` of back-to-back graph replays per budget, median
of 20-step windows, nvidia-smi SM clock sampled meanwhile.

    python tools/budget_sustained.py [config] [seconds] budget ...
"""
import os, statistics, subprocess, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

config = sys.argv[1]
secs = float(sys.argv[2])
budgets = [int(x) for x in sys.argv[3:]]
ns = bench.prepare(config, torch.device("cuda", 0), budgets=[budgets[0]])
for rnd in range(2):
    for b in budgets:
        st = ns.step.with_budget(b, plan=None)
        if b != ns.budget:
            import paper_2505_17694_b200 as P
            pl = P.plan_device(ns.forest, ns.g, ns.table, ns.h_local, ns.sms, b)
            st = ns.step.with_budget(b, plan=pl)
        g = st.capture(ns.q_dev, ns.kp, ns.vp, ns.out)
        clk = bench.ClockSampler(0)
        wins, t0 = [], time.perf_counter()
        while time.perf_counter() - t0 < secs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g()
            e1.record()
            torch.cuda.synchronize()
            wins.append(e0.elapsed_time(e1) / 20 * 1e3)
        c = clk.stop()
        print(f"round {rnd} budget {b}: {statistics.median(wins):7.1f} us (windows {len(wins)}), sm {c['sm_mhz']} MHz, "
              f"{c['reasons']}", flush=True)
