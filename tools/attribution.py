"""Step time with parts of the step switched off (SKIP flags), cfg at a fixed
tensor-core SM budget: how much each kernel adds to the overlapped step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 96
ns = bench.prepare(cfg, torch.device("cuda", 0), budgets=[budget])


def t(step, n=50):
    for _ in range(5):
        step(ns.q_dev, ns.kp, ns.vp, out=ns.out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        step(ns.q_dev, ns.kp, ns.vp, out=ns.out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for name, fl in (("full", 0), ("no merge", 64), ("TC + merge (no suffix)", 32), ("suffix + merge (no TC)", 16),
                 ("TC only", 32 | 64), ("suffix only", 16 | 64)):
    print(f"{cfg} budget {budget}: {name:28s} {t(ns.step.with_budget(budget, flags=fl)):8.1f} us", flush=True)
