"""Repeatability check of one fuzz case: run the same step N times and
report how many distinct outputs appear (per flag set)."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200.executor import DecodeStep
from test_gpu_fuzz import _forest, _reference

seed, budget = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(500 + seed)
parent, length, paths = _forest(rng)
f = P.forest_from_pool(parent[1:], length[1:], paths, 8, 128)
gen = torch.Generator(device="cuda").manual_seed(seed)
T = f.total_tokens
kp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
q = (torch.randn((f.bs, 32, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
ref = torch.stack([_reference(f, kp, vp, q, r) for r in range(f.bs)])
plan = P.plan_device(f, 4, P.load_default_profile(), 8, 148, budget)
for name, kw in [("default", dict(concurrent=True)), ("serial", dict(concurrent=False)),
                 ("no_tc", dict(concurrent=False, flags=1)), ("tc_only", dict(concurrent=False, flags=32)),
                 ("sfx_only", dict(concurrent=False, flags=16))]:
    step = DecodeStep(f, plan, 32, "bfloat16", tc_sm_budget=budget, **kw)
    outs = []
    for _ in range(12):
        outs.append(step(q, kp, vp).clone())
    torch.cuda.synchronize()
    distinct = []
    for o in outs:
        if not any(torch.equal(o, d) for d in distinct):
            distinct.append(o)
    errs = [float((o.double() - ref).abs().max()) for o in distinct]
    print(f"{name:9s} distinct outputs {len(distinct)}  errs {['%.1e' % e for e in errs]}", flush=True)
    if len(distinct) > 1:
        d = (distinct[0] - distinct[1]).abs().amax(dim=2)
        idx = torch.nonzero(d > 0)
        print("   differing (request, head) pairs:", idx[:12].tolist(), "count", len(idx))
