"""cfg2 step time over the contiguous pool vs paged pools (random page
permutation), same plan and SM budget.

    python tools/paged_bench.py [budget]
"""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.executor import DecodeStep
from paper_2505_17694_b200.paging import paged_pools, page_layout

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 96
dev = torch.device('cuda')
spec = W.two_level(32768, 512, 256, h_q=32, h_kv=8, d=128, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((256, 32, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)


def timeit(step, k, v, n=20, reps=5):
    for _ in range(3):
        step(q, k, v)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            step(q, k, v)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n * 1e3)
    return sorted(ts)[len(ts) // 2]


plan = P.plan_device(f, 4, P.load_default_profile(), 8, 148, budget, page_size=128)
base = DecodeStep(f, plan, 32, 'bfloat16', tc_sm_budget=budget)
ref = base(q, kp, vp)
print(f"contiguous: {timeit(base, kp, vp):7.1f} us", flush=True)
for page in (128, 256, 1024):
    gen = torch.Generator().manual_seed(page)
    kx, vx, pt = paged_pools(f, kp, vp, page, generator=gen)
    step = DecodeStep(f, plan, 32, 'bfloat16', tc_sm_budget=budget, page_size=page, page_table=pt,
                      pool_tokens=kx.shape[1])
    same = torch.equal(step(q, kx, vx), ref)
    print(f"paged P={page:5d}: {timeit(step, kx, vx):7.1f} us  (== contiguous: {same})", flush=True)
    del kx, vx
