"""One decode step of the bench's prepared step, bracketed by
cudaProfilerStart/Stop for ncu --profile-from-start off.

    ncu --set full --profile-from-start off --clock-control none --import-source on \\
        -o gpurun_out/ncu_cfg2 python tools/ncu_step.py cfg2 96 [flags]

(flags: the bench's routing choice, e.g. 4194304 = CODEC_FLAG_NO_TCT)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 148
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ns = bench.prepare(cfg, torch.device("cuda", 0), flags=flags, budgets=[budget])
torch.cuda.synchronize()
torch.cuda.profiler.start()
ns.step(ns.q_dev, ns.kp, ns.vp, out=ns.out)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, "budget", budget, "launches", ns.step.launches)
