"""K1 parity: the C++ planner (through the package API and the C ABI) is
bit-exact with the reference scheduler -- against the golden plans
recorded from the reference and against the oracle on fresh random
instances. CPU only (host code of the shared library)."""
from __future__ import annotations

import io

import numpy as np
import pytest

from conftest import golden_json, golden_table_text
from recipes import random_micro_tasks
from oracle import plan as OP
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import scheduler as S
from paper_2505_17694_b200.errors import SearchSpaceOverflow


@pytest.fixture(scope="module")
def tables():
    return {"a100": P.load_profile(io.StringIO(golden_table_text("a100_d128.csv"))),
            "proxy": P.load_profile(io.StringIO(golden_table_text("proxy_b200.csv")))}


def f(s):
    return float(s)


def T(tasks):
    return [P.Task(*t) for t in tasks]


def check(plan, doc):
    assert list(plan.b_k) == doc["b_k"]
    assert [[s.task_index, s.node, s.start, s.stop] for s in plan.subtasks] == [st[:4] for st in doc["subtasks"]]
    assert [s.cost_ms for s in plan.subtasks] == [f(st[4]) for st in doc["subtasks"]]
    assert list(plan.assignment.block_of) == doc["block_of"]
    assert list(plan.assignment.loads) == [f(x) for x in doc["loads"]]
    assert plan.makespan_ms == f(doc["makespan"])
    assert plan.search_truncated == doc["truncated"]
    if doc["cost_l"] is not None:
        assert plan.cost_l_ms == f(doc["cost_l"])


class TestGoldenBitExact:
    def test_estimate(self, tables):
        for name, q, n, val in golden_json("planner.json")["estimate"]:
            assert P.estimate(tables[name], q, n) == f(val), (name, q, n)

    def test_slices(self):
        for n, b, ranges, count in golden_json("planner.json")["slices"]:
            assert [list(x) for x in S.slice_ranges(n, b)] == ranges
            assert S.canonical_division(n, b) == count

    def test_micro(self, tables):
        for doc in golden_json("planner.json")["micro"]:
            tasks = T(doc["tasks"])
            t = tables[doc["table"]]
            cl = P.lower_bound(tasks, t, doc["m"])
            assert cl == f(doc["cost_l"])
            assert P.division_caps(tasks, t, cl) == doc["caps"]
            check(P.divide_and_schedule(tasks, t, doc["m"], search_limit=doc["limit"]), doc["plan"])

    def test_flagship(self, tables):
        pl = golden_json("planner.json")
        flag = [P.Task(1, 8, 16384)] + [P.Task(2 + i, 1, 512) for i in range(8)]
        check(P.divide_and_schedule(flag, tables["a100"], 8), pl["flagship"])
        check(P.plan_uniform_bk(flag, tables["a100"], 8, 1), pl["flagship_identity"])
        for u in pl["uniform"]:
            check(P.plan_uniform_bk(flag, tables["a100"], 8, u["bk"]), u["plan"])

    def test_greedy(self):
        for doc in golden_json("planner.json")["greedy"]:
            a = P.greedy_assign([f(c) for c in doc["costs"]], doc["m"])
            assert list(a.block_of) == doc["block_of"]
            assert list(a.loads) == [f(x) for x in doc["loads"]]

    def test_overflow(self, tables):
        doc = golden_json("planner.json")["overflow"][0]
        check(P.divide_and_schedule(T(doc["tasks"]), tables["a100"], doc["m"], search_limit=doc["limit"]),
              doc["plan"])
        with pytest.raises(SearchSpaceOverflow, match="exceed the limit"):
            P.divide_and_schedule(T(doc["tasks"]), tables["a100"], doc["m"], search_limit=2, on_overflow="raise")

    def test_config_scale(self, tables):
        for doc in golden_json("planner.json")["configs"]:
            check(P.divide_and_schedule(T(doc["tasks"]), tables[doc["table"]], doc["m"], search_limit=doc["limit"]),
                  doc["plan"])


class TestAgainstOracle:
    """Fresh instances the goldens do not contain: product == oracle."""

    @pytest.mark.parametrize("seed", range(60, 100))
    def test_random_instances(self, tables, seed):
        rng = np.random.default_rng(seed)
        name = "a100" if seed % 2 else "proxy"
        grid = OP.parse_profile(golden_table_text("a100_d128.csv" if name == "a100" else "proxy_b200.csv"))
        t = int(rng.integers(1, 7))
        m = int(rng.integers(1, 40))
        tasks = [(j + 1, int(rng.integers(1, 300)), int(rng.integers(1, 70000))) for j in range(t)]
        limit = 3000
        ref = OP.divide_and_schedule(tasks, grid, m, limit=limit)
        got = P.divide_and_schedule(T(tasks), tables[name], m, search_limit=limit)
        assert got.b_k == ref.b_k
        assert [(s.task_index, s.node, s.start, s.stop, s.cost_ms) for s in got.subtasks] == list(ref.subtasks)
        assert got.assignment.block_of == ref.block_of
        assert got.makespan_ms == ref.makespan
        assert got.cost_l_ms == ref.cost_l

    def test_known_reference_values(self, tables):
        # reference tests: test_scheduler.py:111-115, :163-175; test_cost_model.py:43-47
        tasks = [P.Task(1, 2, 16384)] + [P.Task(2 + i, 1, 512) for i in range(4)]
        cl = P.lower_bound(tasks, tables["a100"], 4)
        assert cl == pytest.approx(0.12531152343749996, rel=1e-12)
        assert P.division_caps(tasks, tables["a100"], cl) == [3, 1, 1, 1, 1]
        assert P.estimate(tables["a100"], 1, 2896) == pytest.approx(0.07599506838666258, rel=1e-13)
        assert P.estimate(tables["a100"], 3, 1024) == pytest.approx(0.04333333333333333, rel=1e-13)
        a = P.greedy_assign([5, 4, 3, 3, 2], 2)
        assert sorted(a.loads) == [8.0, 9.0]

    def test_validation_errors(self, tables):
        with pytest.raises(ValueError, match="no tasks"):
            P.divide_and_schedule([], tables["a100"], 4)
        with pytest.raises(ValueError, match="m >= 1"):
            P.greedy_assign([1.0], 0)
        with pytest.raises(ValueError, match="b_k must be >= 1"):
            P.plan_uniform_bk([P.Task(1, 1, 10)], tables["a100"], 2, 0)
        with pytest.raises(ValueError, match="cost_l must be positive"):
            P.division_caps([P.Task(1, 1, 10)], tables["a100"], 0.0)


def test_planner_speed_cfg4(tables):
    """cfg4-scale planning (4744 tasks, m=148) in C++ is interactive."""
    import time
    from paper_2505_17694_b200 import workloads as W
    from oracle import index as OI
    spec = W.make_config("cfg4", tensors=False)
    qs = OI.query_sets(spec.paths, spec.n_nodes)
    tasks = [P.Task(*t) for t in OP.node_tasks(qs, spec.length)]
    t0 = time.perf_counter()
    plan = P.divide_and_schedule(tasks, tables["proxy"], 148)
    dt = time.perf_counter() - t0
    assert plan.makespan_ms > 0 and dt < 5.0
