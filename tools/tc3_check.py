"""TC3 (three-group shared-node kernel, CODEC_FLAG_TC3) against the default
kernel and the float64 device reference on the bench's cfg2 step and a few
random forests; then times both (TC alone and the full step)."""
import math, os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2505_17694_b200 as P
from paper_2505_17694_b200.executor import DecodeStep
TC3 = 4194304
for cfg in ("cfg2", "cfg3"):
    ns = bench.prepare(cfg, torch.device("cuda", 0), budgets=[96])
    a = ns.step(ns.q_dev, ns.kp, ns.vp).clone()
    st3 = ns.step.with_budget(ns.budget, flags=ns.step.flags | TC3)
    b = st3(ns.q_dev, ns.kp, ns.vp)
    torch.cuda.synchronize()
    d = float((a - b).abs().max())
    worst = 0.0
    for r in [0, 1, ns.forest.bs // 2, ns.forest.bs - 1]:
        ref = bench.path_reference(ns.forest, ns.kp, ns.vp, ns.q_dev, r)
        worst = max(worst, float((b[r].double() - ref).abs().max()))
    rep = all(torch.equal(b, st3(ns.q_dev, ns.kp, ns.vp)) for _ in range(3))
    print(f"{cfg}: max |tc3 - default| {d:.2e}, max err vs fp64 {worst:.2e}, repeatable {rep}", flush=True)
    for name, fl in (("default TC alone", 8 | 32 | 64), ("tc3 TC alone", 8 | 32 | 64 | TC3), ("default step", 0),
                     ("tc3 step", TC3)):
        st = ns.step.with_budget(ns.budget, flags=ns.step.flags | fl)
        g = st.capture(ns.q_dev, ns.kp, ns.vp, ns.out)
        for _ in range(5):
            g()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(100):
                g()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 100 * 1e3)
        print(f"  {name:18s} {sorted(ts)[1]:8.1f} us", flush=True)
