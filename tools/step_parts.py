"""Where the cfg2 step's time goes: the overlapped step at a fixed SM
budget with one kernel skipped at a time (timing only; wrong outputs).

    python tools/step_parts.py [config] [budget]
"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

config = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 96
ns = bench.prepare(config, torch.device("cuda", 0), budgets=[budget])
cases = [("full step", 0), ("no merge", 64), ("no suffix", 32), ("no TC", 16), ("TC only", 32 | 64 | 8),
         ("suffix only", 16 | 64 | 8)]
res = {}
for rnd in range(3):
    for name, fl in cases:
        st = ns.step if fl == 0 else ns.step.with_budget(budget, flags=ns.step.flags | fl)
        for _ in range(5):
            st(ns.q_dev, ns.kp, ns.vp, out=ns.out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            st(ns.q_dev, ns.kp, ns.vp, out=ns.out)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(name, []).append(e0.elapsed_time(e1) / 100 * 1e3)
for name, _ in cases:
    v = sorted(res[name])
    print(f"{name:12s} {v[1]:7.1f} us  {[round(x, 1) for x in res[name]]}")
