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


def test_profile_error_contract():
    """load_profile / CostTable / dump_profile against the reference's own
    results on good and malformed CSVs (tests/golden/profile_errors.json):
    same exception class and message, same canonical dump."""
    from recipes import PROFILE_CASES
    gold = golden_json("profile_errors.json")
    for name, text in PROFILE_CASES.items():
        kind, payload = gold[name]
        if kind == "ok":
            buf = io.StringIO()
            P.dump_profile(P.load_profile(io.StringIO(text)), buf)
            assert buf.getvalue() == payload, name
        else:
            with pytest.raises(Exception) as ei:
                P.load_profile(io.StringIO(text))
            assert (type(ei.value).__name__, str(ei.value)) == (kind, payload), name


def test_cost_table_invariants():
    from paper_2505_17694_b200.errors import DuplicateKnot, IncompleteGrid, NonPositiveCost
    with pytest.raises(IncompleteGrid, match=r"grid \(2,\) does not match knots \(1, 2\)"):
        P.CostTable((1, 2), (512,), np.ones(2))
    with pytest.raises(DuplicateKnot, match=r"n knots must be strictly ascending positives: \(512, 512\)"):
        P.CostTable((1,), (512, 512), np.ones((2, 1)))
    with pytest.raises(NonPositiveCost, match="every grid cost must be > 0"):
        P.CostTable((1,), (512,), np.zeros((1, 1)))
    t = P.profile_synthetic(0.01, 1e-5, 2e-6)
    assert t.cell(5, 2048) == pytest.approx(0.01 + 1e-5 * 2048 + 2e-6 * 2048 * 5, rel=1e-15)


def test_merge_schedules_golden():
    """merge_schedule / sequential_schedule equal the reference's
    (tests/golden/schedules.json; executor.py:86-117)."""
    gold = golden_json("schedules.json")
    for L, counts, rounds in gold["balanced"]:
        assert [[list(p) for p in rnd] for rnd in P.merge_schedule(L, counts)] == rounds
    for total, rounds in gold["sequential"]:
        assert [[list(p) for p in rnd] for rnd in P.sequential_schedule(total)] == rounds
    assert P.merge_schedule(2, [3, 2]) == [[(0, 1), (2, 3)], [(0, 2)], [(0, 4)]]  # test_executor.py:66-76
    with pytest.raises(ValueError, match="path_len must be >= 1"):
        P.merge_schedule(0, [])
    with pytest.raises(ValueError, match="expected 2 per-node slice counts, got 1"):
        P.merge_schedule(2, [1])


def test_run_report_golden():
    """run_report() equals the reference CLI's RunReport for the same
    workload points (tests/golden/reports.json, cli.py:130-184), and passes
    the schema check."""
    from paper_2505_17694_b200 import workloads as W
    from paper_2505_17694_b200.report import check_report, run_report
    table = P.load_profile(io.StringIO(golden_table_text("a100_d128.csv")))
    for item in golden_json("reports.json"):
        ref = item["report"]
        w = ref["workload"]
        fn = {"two_level": W.two_level, "full_tree": W.full_tree}[w["family"]]
        spec = fn(**w["params"], **w["dims"], seed=w["seed"], tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, spec.h_kv, spec.d)
        plan = P.divide_and_schedule(P.tasks_from_forest(f), table, item["blocks"])
        got = run_report(f, plan, table, item["blocks"], w, element_size=8)
        assert got == ref
        check_report(got)
    bad = dict(got, extra=1)
    with pytest.raises(ValueError, match="unknown keys"):
        check_report(bad)
