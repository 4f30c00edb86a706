"""Debug: which kernel makes concurrent vs serial outputs differ?"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.executor import DecodeStep


def build(spec, dtype):
    tdt = torch.bfloat16
    specs = [(p, torch.from_numpy(np.ascontiguousarray(k)).to(tdt), torch.from_numpy(np.ascontiguousarray(v)).to(tdt), vis)
             for p, k, v, vis in spec.node_specs()]
    qb = P.QueryBatch(torch.from_numpy(np.ascontiguousarray(spec.queries)).to(tdt), spec.h_kv)
    return P.build_forest(specs, spec.paths, qb), qb
import io
table = P.load_profile(io.StringIO(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests/golden/a100_d128.csv')).read()))
spec = W.two_level(2048, 200, 96, h_q=32, h_kv=8, d=128, seed=4)
f, q = build(spec, "bfloat16")
plan = P.divide_and_schedule(P.device_tasks(f, group_size=4), table, 37)
kp, vp = f.device_pool("bfloat16")
qd = q.queries.cuda()
np_ = lambda t: t.double().cpu().numpy()
for flags in (0, 2048):
    ser = DecodeStep(f, plan, 32, "bfloat16", concurrent=False, flags=flags)
    outs = [np_(ser(qd, kp, vp)) for _ in range(3)]
    print([(s.node, s.start, s.stop, b) for s, b in zip(plan.subtasks, plan.assignment.block_of) if s.node == 1]); print("flags", flags, "serial repeat equal:", all(np.array_equal(o, outs[0]) for o in outs))
    for budget in (0, 120, 64):
        c = DecodeStep(f, plan, 32, "bfloat16", concurrent=True, tc_sm_budget=budget, flags=flags)
        co = [np_(c(qd, kp, vp)) for _ in range(3)]
        d = np.abs(co[0] - outs[0])
        bad = np.argwhere(d > 0)
        print(f"  budget {budget}: repeat equal {all(np.array_equal(o, co[0]) for o in co)}, "
              f"vs serial max diff {d.max():.3e}, n diff {len(bad)}, reqs {sorted(set(bad[:,0].tolist()))[:10]}, heads {sorted(set(bad[:,1].tolist()))[:10]}")
    s2 = DecodeStep(f, plan, 32, "bfloat16", concurrent=False, tc_sm_budget=64, flags=flags)
    d = np.abs(np_(s2(qd, kp, vp)) - outs[0])
    print(f"  serial budget 64 vs serial: max diff {d.max():.3e}")

# which partials differ? (merge skipped, workspace compared)
ser = DecodeStep(f, plan, 32, "bfloat16", concurrent=False, flags=64)
ser(qd, kp, vp)
torch.cuda.synchronize()
wref = ser.workspace.clone()
info = ser.info
print("slots", info.n_slots, "tc units", info.n_tc_groups, "gemv groups", info.n_gemv_groups)
blob = ser.blob_host
rows = blob[info.off_rows: info.off_rows + 4 * info.n_rows].reshape(-1, 4)
for trial in range(3):
    c = DecodeStep(f, plan, 32, "bfloat16", concurrent=True, tc_sm_budget=64, flags=64)
    c(qd, kp, vp)
    torch.cuda.synchronize()
    hq = 32
    o_bytes = ((info.n_slots * hq * 128 * 4 + 255) // 256) * 256
    a = wref[:o_bytes].view(torch.float32).view(info.n_slots, hq, 128).cpu().numpy()
    b = c.workspace[:o_bytes].view(torch.float32).view(info.n_slots, hq, 128).cpu().numpy()
    ml_a = wref[o_bytes:o_bytes + info.n_slots * hq * 8].view(torch.float32).view(info.n_slots, hq, 2).cpu().numpy()
    ml_b = c.workspace[o_bytes:o_bytes + info.n_slots * hq * 8].view(torch.float32).view(info.n_slots, hq, 2).cpu().numpy()
    bad = np.argwhere(np.abs(a - b).max(-1) > 0)
    badml = np.argwhere(np.abs(ml_a - ml_b).max(-1) > 0)
    print("trial", trial, "bad (slot, head):", bad[:8].tolist(), "ml bad:", badml[:8].tolist())
    for sl, h in bad[:4]:
        r = np.argwhere(rows[:, 2] == sl)
        print("   slot", sl, "row records", r.ravel().tolist(), "req", rows[r.ravel(), 0].tolist(), "vis", rows[r.ravel(), 1].tolist(),
              "ml ser", ml_a[sl, h], "conc", ml_b[sl, h])
