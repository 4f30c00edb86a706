"""Pin the CPU oracle (oracle/) against golden vectors recorded from the
real reference (tests/golden/make_golden.py). CPU only."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_json, golden_npz, golden_table_text, rel_err
from recipes import PAC_SHAPES, pac_inputs, random_forest_spec, random_micro_tasks
from oracle import attention as OA
from oracle import index as OI
from oracle import plan as OP
from paper_2505_17694_b200 import workloads as W


@pytest.fixture(scope="module")
def grids():
    return {"a100": OP.parse_profile(golden_table_text("a100_d128.csv")),
            "proxy": OP.parse_profile(golden_table_text("proxy_b200.csv"))}


def f(s):
    return float(s)


def check_plan(p: OP.Plan, doc):
    assert list(p.b_k) == doc["b_k"]
    assert [list(st[:4]) for st in p.subtasks] == [st[:4] for st in doc["subtasks"]]
    assert [st[4] for st in p.subtasks] == [f(st[4]) for st in doc["subtasks"]]
    assert list(p.block_of) == doc["block_of"]
    assert list(p.loads) == [f(x) for x in doc["loads"]]
    assert p.makespan == f(doc["makespan"])
    assert p.truncated == doc["truncated"]
    if doc["cost_l"] is not None:
        assert p.cost_l == f(doc["cost_l"])


class TestPlannerOracle:
    def test_estimates_bit_exact(self, grids):
        for name, q, n, val in golden_json("planner.json")["estimate"]:
            assert OP.estimate(grids[name], q, n) == f(val), (name, q, n)

    def test_slices(self):
        for n, b, ranges, count in golden_json("planner.json")["slices"]:
            assert [list(x) for x in OP.slices(n, b)] == ranges
            assert OP.n_slices(n, b) == count

    def test_micro_instances(self, grids):
        for doc in golden_json("planner.json")["micro"]:
            tasks, m = random_micro_tasks(doc["seed"])
            assert [list(t) for t in tasks] == doc["tasks"] and m == doc["m"]
            g = grids[doc["table"]]
            cl = OP.lower_bound(tasks, g, m)
            assert cl == f(doc["cost_l"])
            assert OP.caps(tasks, g, cl) == doc["caps"]
            check_plan(OP.divide_and_schedule(tasks, g, m, limit=doc["limit"]), doc["plan"])

    def test_flagship_and_uniform(self, grids):
        pl = golden_json("planner.json")
        flag = [(1, 8, 16384)] + [(2 + i, 1, 512) for i in range(8)]
        check_plan(OP.divide_and_schedule(flag, grids["a100"], 8), pl["flagship"])
        check_plan(OP.uniform(flag, grids["a100"], 8, 1), pl["flagship_identity"])
        for u in pl["uniform"]:
            check_plan(OP.uniform(flag, grids["a100"], 8, u["bk"]), u["plan"])
        # reference test_scheduler.py:163-175 worked numbers
        p = OP.divide_and_schedule(flag, grids["a100"], 8)
        assert p.b_k == (4,) + (1,) * 8 and p.makespan == pytest.approx(0.1128, rel=1e-12)

    def test_greedy(self):
        for doc in golden_json("planner.json")["greedy"]:
            owner, load = OP.lpt([f(c) for c in doc["costs"]], doc["m"])
            assert owner == doc["block_of"]
            assert load == [f(x) for x in doc["loads"]]

    def test_overflow_fallback(self, grids):
        doc = golden_json("planner.json")["overflow"][0]
        tasks = [tuple(t) for t in doc["tasks"]]
        check_plan(OP.divide_and_schedule(tasks, grids["a100"], doc["m"], limit=doc["limit"]), doc["plan"])

    def test_config_scale_plans(self, grids):
        for doc in golden_json("planner.json")["configs"]:
            tasks = [tuple(t) for t in doc["tasks"]]
            check_plan(OP.divide_and_schedule(tasks, grids[doc["table"]], doc["m"], limit=doc["limit"]),
                       doc["plan"])


class TestIndexOracle:
    def test_random_forests(self):
        for doc in golden_json("index.json")["random"]:
            spec = random_forest_spec(doc["seed"], with_masks=doc["masks"])
            ix = OI.forest_index(spec.parent, spec.length, spec.paths, spec.visible)
            qs = [list(ix["qset_idx"][ix["qset_ptr"][i]:ix["qset_ptr"][i + 1]]) for i in range(spec.n_nodes)]
            assert qs[1:] == doc["query_sets"][1:]
            assert list(ix["node_off"]) == doc["token_offset"]
            assert [list(p) for p in spec.paths] == doc["paths"]
            assert OI.children_lists(spec.parent, spec.n_nodes) == doc["children"]
            assert [list(t) for t in OP.node_tasks(OI.query_sets(spec.paths, spec.n_nodes), spec.length)] == doc["tasks"]

    def test_config_structures(self):
        for doc in golden_json("index.json")["configs"]:
            spec = W.make_config(doc["config"], tensors=False)
            ix = OI.forest_index(spec.parent, spec.length, spec.paths)
            assert hashlib.sha256(ix["node_off"].astype(np.int64).tobytes()).hexdigest() == doc["token_offset_sha"]
            assert hashlib.sha256(ix["qset_idx"][ix["qset_ptr"][1]:].astype(np.int64).tobytes()).hexdigest() == doc["qset_sha"]
            qs = OI.query_sets(spec.paths, spec.n_nodes)
            tasks = np.asarray(OP.node_tasks(qs, spec.length), np.int64)
            assert hashlib.sha256(tasks.tobytes()).hexdigest() == doc["tasks_sha"]
            assert sum(spec.length) == doc["total_tokens"]

    def test_traffic_rows(self):
        for cname, doc in golden_json("traffic.json").items():
            spec = W.make_config(cname, tensors=False)
            qs = OI.query_sets(spec.paths, spec.n_nodes)
            assert sum(spec.length[1:]) == doc["rows_codec"]
            assert sum(spec.length[i] * len(qs[i]) for i in range(1, spec.n_nodes)) == doc["rows_baseline"]


class TestGeneratorPins:
    @pytest.mark.parametrize("name", ["two_level_small", "full_tree", "degenerate", "shared_ratio", "cfg1"])
    def test_draws_bit_identical(self, name):
        doc = golden_json("workloads.json")[name]
        fn = {"two_level_small": W.two_level, "full_tree": W.full_tree, "degenerate": W.degenerate,
              "shared_ratio": W.shared_ratio, "cfg1": W.two_level}[name]
        h_q, h_kv, d = doc["dims"]
        spec = fn(**doc["kw"], h_q=h_q, h_kv=h_kv, d=d, seed=doc["seed"])
        h = hashlib.sha256()
        for i in range(1, spec.n_nodes):
            h.update(spec.keys[i].tobytes())
            h.update(spec.values[i].tobytes())
        h.update(spec.queries.tobytes())
        assert h.hexdigest() == doc["sha256"]
        assert [list(p) for p in spec.paths] == doc["paths"]
        assert spec.parent[1:] == doc["parents"]


def oracle_forest(spec):
    keys = [np.zeros((0, spec.h_kv, spec.d))] + spec.keys[1:]
    vals = [np.zeros((0, spec.h_kv, spec.d))] + spec.values[1:]
    return OA.ForestData(spec.parent, keys, vals, spec.paths, spec.visible)


class TestNumericOracle:
    def test_pac_goldens(self):
        z = golden_npz()
        for i, shape in enumerate(PAC_SHAPES):
            for masked in (False, True):
                q, k, v, vis = pac_inputs(shape, masked=masked)
                out, m, s = OA.pac(q, k, v, vis)
                tag = f"{i}_{int(masked)}"
                assert rel_err(out, z[f"pac_out_{tag}"]) <= 1e-12
                assert rel_err(m, z[f"pac_m_{tag}"]) <= 1e-12
                assert rel_err(s, z[f"pac_s_{tag}"]) <= 1e-12

    def test_known_answers(self):
        """test_attention.py:53-70 scalar goldens."""
        a = lambda *x: np.asarray(x, np.float64).reshape(-1, 1, 1)
        out, m, s = OA.pac(a(2.0), a(3.0), a(7.0))
        assert (out.item(), m.item(), s.item()) == (7.0, 6.0, 1.0)
        out, m, s = OA.pac(a(2.0), a(3.0, 5.0), a(7.0, 11.0))
        assert out.item() == pytest.approx(10.928055160152, rel=1e-12)
        assert m.item() == 10.0 and s.item() == pytest.approx(1.0183156388887, rel=1e-12)
        merged = OA.por(OA.pac(a(2.0), a(3.0), a(7.0)), OA.pac(a(2.0), a(5.0), a(11.0)))
        assert merged[0].item() == pytest.approx(10.928055160152, rel=1e-12)

    def test_merge_rounds(self):
        assert OA.merge_rounds([3, 2]) == [[(0, 1), (2, 3)], [(0, 2)], [(0, 4)]]
        assert OA.merge_rounds([1]) == []

    def test_execute_and_naive_goldens(self, grids):
        z = golden_npz()
        for doc in golden_json("forests.json")["forests"]:
            seed = doc["seed"]
            spec = random_forest_spec(seed, with_masks=doc["masks"])
            fd = oracle_forest(spec)
            ref = z[f"naive_{seed}"]
            assert rel_err(OA.naive_attention(spec.queries, fd), ref) <= 1e-12
            for key, plan in (("exec_u", doc["plan_u"]), ("exec_a", doc["plan_a"])):
                subs = [(st[1], st[2], st[3]) for st in plan["subtasks"]]
                out = OA.execute(fd, spec.queries, subs)
                assert rel_err(out, z[f"{key}_{seed}"]) <= 1e-12
                assert rel_err(out, ref) <= 1e-10
