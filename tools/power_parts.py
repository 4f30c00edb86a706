"""Power and clock of the step's parts in sustained windows: the full
step, the tensor-core kernel alone, the suffix kernel alone (same budget,
graph replay, >= `seconds` each), with nvidia-smi sampling meanwhile.

    python tools/power_parts.py [config] [seconds]
"""
import os, statistics, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

config = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
ns = bench.prepare(config, torch.device("cuda", 0), budgets=[96] if config == "cfg2" else None)
for name, fl in (("full step", 0), ("TC only", 8 | 32 | 64), ("suffix only", 8 | 16 | 64), ("full step", 0)):
    st = ns.step if fl == 0 else ns.step.with_budget(ns.budget, flags=ns.step.flags | fl)
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
    print(f"{name:12s} {statistics.median(wins):8.1f} us  sm {c['sm_mhz']} MHz  power {c['power_w_median']} W  "
          f"{c['reasons']}", flush=True)
