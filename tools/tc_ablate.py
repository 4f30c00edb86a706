"""Debug: time the tensor-core kernel alone on cfg2 under the timing-only
ablation flags (wrong outputs), to see which part of the tile pipeline binds.

    python tools/tc_ablate.py [budget]
"""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.executor import DecodeStep

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 148
only = [int(x) for x in sys.argv[2:]]  # run just these flag sets
dev = torch.device('cuda')
spec = W.two_level(32768, 512, 256, h_q=32, h_kv=8, d=128, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((256, 32, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
plan = P.plan_device(f, 4, P.load_default_profile(), 8, 148, budget)
SKIP = 8 | 32 | 64
cases = [("full", 0), ("no TMEM S/P", 256), ("no exp", 512), ("no softmax (TMEM+exp)", 768),
         ("no loads", 32768), ("no softmax, no loads", 768 | 32768), ("issuer only", 131072)]
if only:
    cases = [(f"flags {x}", x) for x in only]
info = None
for name, fl in cases:
    step = DecodeStep(f, plan, 32, 'bfloat16', flags=SKIP | fl, tc_sm_budget=budget, concurrent=False)
    info = step.info
    for _ in range(3):
        step(q, kp, vp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        step(q, kp, vp)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"{name:34s} {us:8.1f} us", flush=True)
blob = step.blob_host
bp = blob[info.off_tc_block_ptr: info.off_tc_block_ptr + info.n_tc_blocks + 1]
recs = blob[info.off_tc: info.off_tc + 8 * info.n_tc_groups].reshape(-1, 8)
tiles = [int(sum((recs[j, 4] + 127) // 128 for j in range(bp[b], bp[b + 1]))) for b in range(info.n_tc_blocks)]
print("pairs", info.n_tc_blocks, "tiles/pair max", max(tiles), "-> clk/tile at 1.92 GHz = us *", round(1920 / max(tiles), 2))
