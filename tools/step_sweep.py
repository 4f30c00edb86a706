"""Debug: cfg2 step time (concurrent TC + suffix kernels) over SM budgets,
plus the suffix kernel alone, for comparing kernel variants
(CODEC_B200_LIB=...).

    python tools/step_sweep.py [budget ...]
"""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.executor import DecodeStep

budgets = [int(x) for x in sys.argv[1:]] or [148, 104, 96, 88, 80]
dev = torch.device('cuda')
spec = W.two_level(32768, 512, 256, h_q=32, h_kv=8, d=128, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((256, 32, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)


def timeit(step, n=20, reps=5):
    for _ in range(3):
        step(q, kp, vp)
    torch.cuda.synchronize()
    best = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            step(q, kp, vp)
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1) / n * 1e3)
    best.sort()
    return best[len(best) // 2]


plan = P.plan_device(f, 4, P.load_default_profile(), 8, 148, 148)
sfx = DecodeStep(f, plan, 32, 'bfloat16', flags=16 | 64, concurrent=False)  # SKIP_TC | SKIP_MERGE
print(f"suffix kernel alone: {timeit(sfx):7.1f} us", flush=True)
for b in budgets:
    plan = P.plan_device(f, 4, P.load_default_profile(), 8, 148, b)
    step = DecodeStep(f, plan, 32, 'bfloat16', tc_sm_budget=b, concurrent=True)
    print(f"budget {b:3d}: step {timeit(step):7.1f} us", flush=True)
