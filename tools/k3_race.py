"""Debug: repeat the no-TC step (suffix kernel only) and compare chosen
partial slots with float64 references each run.

    python tools/k3_race.py seed budget kv_head slot:tok:len ...
"""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200.executor import DecodeStep
from test_gpu_fuzz import _forest

seed, budget, kh = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pieces = [tuple(int(x) for x in a.split(":")) for a in sys.argv[4:]]
rng = np.random.default_rng(500 + seed)
parent, length, paths = _forest(rng)
f = P.forest_from_pool(parent[1:], length[1:], paths, 8, 128)
gen = torch.Generator(device="cuda").manual_seed(seed)
T = f.total_tokens
kp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
q = (torch.randn((f.bs, 32, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
plan = P.plan_device(f, 4, P.load_default_profile(), 8, 148, budget)
step = DecodeStep(f, plan, 32, "bfloat16", tc_sm_budget=budget, concurrent=False, flags=1 | 64)  # NO_TC, SKIP_MERGE
info = step.info
o_bytes = (info.n_slots * 32 * 128 * 4 + 255) // 256 * 256
req = int(os.environ.get("REQ", "0"))
refs = {}
for slot, t0, n in pieces:
    for qh in range(kh * 4, kh * 4 + 4):
        k = kp[kh, t0:t0 + n].double(); v = vp[kh, t0:t0 + n].double()
        s = (k @ q[req, qh].double()) / math.sqrt(128)
        m = s.max(); w = torch.exp(s - m)
        refs[(slot, qh)] = ((w @ v) / w.sum(), float(w.sum()), float(m))
for it in range(30):
    step.workspace.zero_()
    step(q, kp, vp)
    torch.cuda.synchronize()
    po = step.workspace[:info.n_slots * 32 * 128 * 4].view(torch.float32).view(info.n_slots, 32, 128)
    pml = step.workspace[o_bytes:o_bytes + info.n_slots * 32 * 8].view(torch.float32).view(info.n_slots, 32, 2)
    bad = []
    for (slot, qh), (o, l, m) in refs.items():
        err = float((po[slot, qh].double() - o).abs().max())
        if err > 1e-4:
            bad.append((slot, qh, f"err {err:.1e}", f"l {float(pml[slot, qh, 1]):.2f} vs {l * math.exp(m) / math.exp(float(pml[slot, qh, 0])) if False else l:.2f}",
                        f"m {float(pml[slot, qh, 0]):.4f} vs {m:.4f}"))
    if bad:
        print("run", it, bad[:4], flush=True)
print("done")
