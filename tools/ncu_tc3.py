import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
ns = bench.prepare("cfg2", torch.device("cuda", 0), budgets=[96])
st = ns.step.with_budget(96, flags=8 | 32 | 64 | 4194304)
st(ns.q_dev, ns.kp, ns.vp, out=ns.out)
torch.cuda.synchronize()
torch.cuda.profiler.start()
st(ns.q_dev, ns.kp, ns.vp, out=ns.out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
