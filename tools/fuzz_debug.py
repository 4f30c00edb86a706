"""Debug a failing fuzz case: per-request error at a given budget, with
variants (serial, SIMT suffix kernel) to localise the faulty kernel."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200.executor import DecodeStep
from test_gpu_fuzz import _forest, _reference

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 3
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = np.random.default_rng(500 + seed)
parent, length, paths = _forest(rng)
print("nodes", len(parent) - 1, "bs", len(paths), "lengths", length[:6], "...")
f = P.forest_from_pool(parent[1:], length[1:], paths, 8, 128)
gen = torch.Generator(device="cuda").manual_seed(seed)
T = f.total_tokens
kp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
q = (torch.randn((f.bs, 32, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
ref = torch.stack([_reference(f, kp, vp, q, r) for r in range(f.bs)])
table = P.load_default_profile()
plan = P.plan_device(f, 4, table, 8, 148, budget)
for name, kw in [("concurrent", dict(concurrent=True)), ("serial", dict(concurrent=False)),
                 ("simt", dict(concurrent=True, flags=2048)), ("no_tc", dict(concurrent=False, flags=1))]:
    step = DecodeStep(f, plan, 32, "bfloat16", tc_sm_budget=budget, **kw)
    out = step(q, kp, vp).double()
    torch.cuda.synchronize()
    e = (out - ref).abs().amax(dim=(1, 2))
    bad = torch.nonzero(e > 2e-3).flatten().tolist()
    eh = (out - ref).abs().amax(dim=2)
    print(f"{name:10s} max err {float(e.max()):.2e} bad requests {bad[:20]} ({len(bad)})")
    if bad:
        r = bad[0]
        print("   request", r, "path", f.paths[r], "bad heads", torch.nonzero(eh[r] > 2e-3).flatten().tolist())
info = DecodeStep(f, plan, 32, "bfloat16", tc_sm_budget=budget).info
print("tc groups", info.n_tc_groups, "tc blocks", info.n_tc_blocks, "gemv", info.n_gemv_groups, "merge", info.n_merge,
      "max_merge", info.max_merge, "slots", info.n_slots)

# per-piece partials of one (request, kv head) against float64 references
if len(sys.argv) > 4:
    r, kh = int(sys.argv[3]), int(sys.argv[4])
    pieces = [tuple(int(x) for x in a.split(":")) for a in sys.argv[5:]]  # slot:tok0:tok1
    step = DecodeStep(f, plan, 32, "bfloat16", tc_sm_budget=budget, concurrent=False)
    step(q, kp, vp)
    torch.cuda.synchronize()
    info = step.info
    hq = 32
    o_bytes = (info.n_slots * hq * 128 * 4 + 255) // 256 * 256
    po = step.workspace[:info.n_slots * hq * 128 * 4].view(torch.float32).view(info.n_slots, hq, 128)
    pml = step.workspace[o_bytes:o_bytes + info.n_slots * hq * 8].view(torch.float32).view(info.n_slots, hq, 2)
    for slot, t0, t1 in pieces:
        for qh in range(kh * 4, kh * 4 + 4):
            k = kp[kh, t0:t1].double(); v = vp[kh, t0:t1].double()
            s = (k @ q[r, qh].double()) / math.sqrt(128)
            m = s.max(); w = torch.exp(s - m); o = (w @ v) / w.sum()
            got = po[slot, qh].double()
            print(f"slot {slot} tokens [{t0},{t1}) qh {qh}: O err {float((got - o).abs().max()):.2e}  "
                  f"m {float(pml[slot, qh, 0]):.4f} vs {float(m):.4f}  l {float(pml[slot, qh, 1]):.3f} vs {float(w.sum()):.3f}")
