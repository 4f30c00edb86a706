"""Generate the golden fixtures under tests/golden/ by running the REAL
reference package (prefixdec, /root/reference/pkg/src) in the build
container. /root/reference does not exist on the GPU box, so everything
the tests need from it is frozen here:

    a100_d128.csv   the reference's bundled cost profile, re-emitted via
                    its own dump_profile (data the planner goldens use)
    planner.json    estimate / slicing / lower_bound / caps / LPT /
                    divide_and_schedule / plan_uniform_bk results, floats
                    stored as repr strings (bit-exact)
    index.json      forest indexing (query sets, preorder offsets, paths,
                    tasks) for random forests and configs 1-5 (structure)
    forests.npz     execute() and naive_attention() outputs (float64 and
                    float32) for seeded random forests; inputs are NOT
                    stored -- tests regenerate them with the same recipe
    pac.npz         pac()/por() outputs for seeded shapes
    workloads.json  sha256 of generator draws (pins our generator)
    traffic.json    traffic_report rows/bytes per config

Run:  python tests/golden/make_golden.py      (needs /root/reference)
"""
from __future__ import annotations

import hashlib
import io
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path(os.environ.get("PREFIXDEC_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parent))          # tests/ (recipes.py)
sys.path.insert(0, str(HERE.parent.parent))   # repo root

os.environ["PREFIXDEC_KERNEL"] = "python"     # deterministic numpy backend

import prefixdec as P                          # noqa: E402
from prefixdec.forest import QueryBatch, build_forest  # noqa: E402

from recipes import random_forest_spec, random_micro_tasks, pac_inputs, PAC_SHAPES  # noqa: E402
from paper_2505_17694_b200 import workloads as W  # noqa: E402


def r(x):
    return repr(float(x))


def ref_forest(spec):
    specs = []
    for i in range(1, spec.n_nodes):
        vis = spec.visible[i] if getattr(spec, "visible", None) else None
        specs.append((spec.parent[i], spec.keys[i], spec.values[i], vis))
    q = QueryBatch(spec.queries, spec.h_kv) if spec.queries is not None else None
    return build_forest(specs, spec.paths, q), q


def struct_forest(spec):
    """Reference Forest with 1x1 tensors: indexing and planning depend
    only on lengths and paths."""
    specs = [(spec.parent[i], np.zeros((spec.length[i], 1, 1)), np.zeros((spec.length[i], 1, 1)))
             for i in range(1, spec.n_nodes)]
    return build_forest(specs, spec.paths)


def plan_doc(plan):
    return {
        "b_k": list(plan.b_k),
        "subtasks": [[st.task_index, st.node, st.start, st.stop, r(st.cost_ms)] for st in plan.subtasks],
        "block_of": list(plan.assignment.block_of),
        "loads": [r(x) for x in plan.assignment.loads],
        "makespan": r(plan.makespan_ms),
        "cost_l": None if plan.cost_l_ms is None else r(plan.cost_l_ms),
        "truncated": bool(plan.search_truncated),
    }


def n_combos(tasks, table, m):
    """Grid-search size the reference would enumerate (scheduler.py:201-205)."""
    cost_l = P.lower_bound(tasks, table, m)
    caps = P.division_caps(tasks, table, cost_l)
    total = 1
    for t, cap in zip(tasks, caps):
        total *= len({P.scheduler.canonical_division(t.n, b) for b in range(1, max(1, min(cap, t.n)) + 1)})
    return total


def bounded_plan(tasks, table, m, budget=400):
    """divide_and_schedule with search_limit lowered to `budget` when the
    full grid would be slow in pure Python; the limit is recorded so the
    product planner is called with the same argument."""
    limit = P.scheduler.DEFAULT_SEARCH_LIMIT if n_combos(tasks, table, m) <= budget else budget
    return P.divide_and_schedule(tasks, table, m, search_limit=limit), limit


def tasks_doc(tasks):
    return [[t.node, t.n_q, t.n] for t in tasks]


def main():
    table = P.load_default_profile()
    buf = io.StringIO()
    P.dump_profile(table, buf)
    (HERE / "a100_d128.csv").write_text(buf.getvalue(), encoding="utf-8")
    proxy = P.profile_synthetic(0.004, 2.0e-6, 4.0e-8,
                                nq_knots=(1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024),
                                n_knots=(64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072))
    buf = io.StringIO()
    P.dump_profile(proxy, buf)
    (HERE / "proxy_b200.csv").write_text(buf.getvalue(), encoding="utf-8")
    tables = {"a100": table, "proxy": proxy}

    # ---------------- planner ----------------
    pl = {"estimate": [], "slices": [], "micro": [], "configs": [], "uniform": [], "greedy": [],
          "overflow": []}
    grid_nq = [1, 2, 3, 4, 5, 7, 10, 13, 20, 33, 50, 77, 100, 128, 200, 999, 1024, 4096]
    grid_n = [1, 3, 64, 100, 511, 512, 700, 1000, 1024, 2896, 4000, 8192, 12345, 16384, 20000, 65536, 131072, 10**6]
    for name, t in tables.items():
        for q in grid_nq:
            for n in grid_n:
                pl["estimate"].append([name, q, n, r(P.estimate(t, q, n))])
    for n in [1, 2, 7, 10, 13, 64, 100, 512, 1000, 32768]:
        for b in [0, 1, 2, 3, 5, 6, 7, 64, 99, 1000, 40000]:
            pl["slices"].append([n, b, [list(x) for x in P.scheduler.slice_ranges(n, b)],
                                 P.scheduler.canonical_division(n, b)])
    for seed in range(60):
        tasks, m = random_micro_tasks(seed)
        T = [P.Task(*t) for t in tasks]
        for name, t in tables.items():
            cost_l = P.lower_bound(T, t, m)
            caps = P.division_caps(T, t, cost_l)
            plan, limit = bounded_plan(T, t, m)
            pl["micro"].append({"seed": seed, "table": name, "tasks": tasks, "m": m, "cost_l": r(cost_l),
                                "caps": caps, "limit": limit, "plan": plan_doc(plan)})
    flag = [P.Task(1, 8, 16384)] + [P.Task(2 + i, 1, 512) for i in range(8)]
    pl["flagship"] = plan_doc(P.divide_and_schedule(flag, table, 8))
    pl["flagship_identity"] = plan_doc(P.plan_uniform_bk(flag, table, 8, 1))
    for bk in (1, 2, 3, 6, 64):
        pl["uniform"].append({"bk": bk, "plan": plan_doc(P.plan_uniform_bk(flag, table, 8, bk))})
    rng = np.random.default_rng(99)
    for trial in range(20):
        costs = [float(x) for x in rng.choice([0.5, 1.0, 1.5, 2.0, 0.25], size=int(rng.integers(1, 30)))]
        m = int(rng.integers(1, 9))
        a = P.greedy_assign(costs, m)
        pl["greedy"].append({"costs": [r(c) for c in costs], "m": m, "block_of": list(a.block_of),
                             "loads": [r(x) for x in a.loads]})
    over = [P.Task(j + 1, 4, 16384) for j in range(3)]
    pl["overflow"].append({"tasks": tasks_doc(over), "m": 4, "limit": 2,
                           "plan": plan_doc(P.divide_and_schedule(over, table, 4, search_limit=2))})
    # config-scale planning instances (node-level and g-multiplied tasks)
    for cname, hm_list, m_list in (("cfg1", (1, 1), (8, 148)), ("cfg2", (1, 4), (8, 18, 148)),
                                   ("cfg3", (1, 4), (8, 148)), ("cfg4", (1,), (148,))):
        spec = W.make_config(cname, tensors=False)
        forest = struct_forest(spec)
        for hm in sorted(set(hm_list)):
            tasks = P.tasks_from_forest(forest, head_multiplicity=hm)
            for m in m_list:
                for tname in ("a100", "proxy"):
                    plan, limit = bounded_plan(tasks, tables[tname], m)
                    pl["configs"].append({"config": cname, "hm": hm, "m": m, "table": tname, "limit": limit,
                                          "tasks": tasks_doc(tasks), "plan": plan_doc(plan)})
                    print(cname, hm, m, tname, limit, len(plan.subtasks), flush=True)
    (HERE / "planner.json").write_text(json.dumps(pl, sort_keys=True), encoding="utf-8")

    # ---------------- indexing ----------------
    idx = {"random": [], "configs": []}
    for seed in range(40):
        spec = random_forest_spec(seed, with_masks=(seed % 2 == 1))
        f, _ = ref_forest(spec)
        idx["random"].append({
            "seed": seed, "masks": seed % 2 == 1,
            "query_sets": [list(n.query_set) for n in f.nodes],
            "token_offset": list(f.token_offset),
            "paths": [list(p) for p in f.paths],
            "children": [list(c) for c in f.children],
            "tasks": tasks_doc(P.tasks_from_forest(f)),
            "request_len": [f.request_len(q) for q in range(f.bs)],
        })
    for cname in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        spec = W.make_config(cname, tensors=False)
        f = struct_forest(spec)
        off = f.token_offset
        idx["configs"].append({
            "config": cname,
            "n_nodes": len(f.nodes), "bs": f.bs,
            "token_offset_sha": hashlib.sha256(np.asarray(off, np.int64).tobytes()).hexdigest(),
            "qset_sha": hashlib.sha256(np.concatenate(
                [np.asarray(n.query_set, np.int64) for n in f.nodes[1:]]).tobytes()).hexdigest(),
            "tasks_sha": hashlib.sha256(np.asarray(tasks_doc(P.tasks_from_forest(f)), np.int64).tobytes()).hexdigest(),
            "total_tokens": f.total_tokens,
        })
    (HERE / "index.json").write_text(json.dumps(idx, sort_keys=True), encoding="utf-8")

    # ---------------- numerics ----------------
    arrs = {}
    meta = {"forests": []}
    for seed in range(48):
        masks = seed % 3 == 2
        spec = random_forest_spec(seed, with_masks=masks)
        f, q = ref_forest(spec)
        bk = 1 + seed % 3
        plan_u = P.plan_uniform_bk(P.tasks_from_forest(f), table, m=4, bk=bk)
        plan_a = P.divide_and_schedule(P.tasks_from_forest(f), table, m=4)
        arrs[f"naive_{seed}"] = P.naive_attention(q, f)
        arrs[f"exec_u_{seed}"] = P.execute(f, q, plan_u, P.BlockPool(worker_count=1))
        arrs[f"exec_a_{seed}"] = P.execute(f, q, plan_a, P.BlockPool(worker_count=1))
        f32, q32 = P.cast_workload(f, q, np.float32)
        plan32 = P.plan_uniform_bk(P.tasks_from_forest(f32), table, m=4, bk=bk)
        arrs[f"exec32_{seed}"] = P.execute(f32, q32, plan32, P.BlockPool(worker_count=1))
        meta["forests"].append({"seed": seed, "masks": masks, "bk": bk,
                                "plan_u": plan_doc(plan_u), "plan_a": plan_doc(plan_a)})
    for i, shape in enumerate(PAC_SHAPES):
        for masked in (False, True):
            qq, kk, vv, vis = pac_inputs(shape, masked=masked)
            p = P.pac(qq, kk, vv, visible=vis)
            tag = f"{i}_{int(masked)}"
            arrs[f"pac_out_{tag}"] = p.out
            arrs[f"pac_m_{tag}"] = p.max_score
            arrs[f"pac_s_{tag}"] = p.exp_sum
    np.savez_compressed(HERE / "forests.npz", **arrs)
    (HERE / "forests.json").write_text(json.dumps(meta, sort_keys=True), encoding="utf-8")

    # ---------------- generator pins ----------------
    wl = {}
    cases = {
        "two_level_small": (P.gen_two_level, W.two_level, dict(shared_len=100, leaf_len=7, batch=5), P.Dims(4, 2, 16), 0),
        "full_tree": (P.gen_full_tree, W.full_tree, dict(arity=3, depth=3, node_len=9), P.Dims(2, 1, 8), 5),
        "degenerate": (P.gen_degenerate, W.degenerate, dict(depth=5, node_len=6), P.Dims(2, 2, 4), 2),
        "shared_ratio": (P.gen_shared_ratio, W.shared_ratio, dict(total_len=257, ratio=0.7, batch=6), P.Dims(1, 1, 16), 9),
        "cfg1": (P.gen_two_level, W.two_level, dict(shared_len=1024, leaf_len=64, batch=16), P.Dims(8, 8, 128), 0),
    }
    for name, (ref_fn, _ours, kw, dims, seed) in cases.items():
        f, q = ref_fn(**kw, dims=dims, seed=seed)
        h = hashlib.sha256()
        for n in f.nodes[1:]:
            h.update(n.keys.tobytes())
            h.update(n.values.tobytes())
        h.update(q.queries.tobytes())
        wl[name] = {"kw": kw, "dims": [dims.h_q, dims.h_kv, dims.d], "seed": seed, "sha256": h.hexdigest(),
                    "paths": [list(p) for p in f.paths], "parents": [n.parent for n in f.nodes[1:]]}
    (HERE / "workloads.json").write_text(json.dumps(wl, sort_keys=True), encoding="utf-8")

    # ---------------- traffic ----------------
    tr = {}
    for cname in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        spec = W.make_config(cname, tensors=False)
        f = struct_forest(spec)
        rep = P.traffic_report(f, element_size=2)
        tr[cname] = {"rows_codec": rep.kv_rows_codec, "rows_baseline": rep.kv_rows_baseline,
                     "nq_bar": r(rep.nq_bar), "h_kv": spec.h_kv, "d": spec.d}
    (HERE / "traffic.json").write_text(json.dumps(tr, sort_keys=True), encoding="utf-8")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
