"""Task division and block scheduling (K1), reference-compatible API.

Types and signatures follow prefixdec/scheduler.py:26-242; the
arithmetic (cost estimate, Eq. 4 bisection, Eq. 5 caps, LPT, grid search
with the {identity, all-at-cap} overflow fallback) runs in the C++
planner of the shared library (csrc/host_plan.cpp), bit-exact with the
reference, typically 100-1000x faster than the Python original.

`device_tasks()` is the B200 addition: it splits every node task into
row chunks (<= 128 query-head rows, one tcgen05 M tile) so the planner
divides and balances exactly the units the GPU runs as CTAs.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cost_model import CostTable
from .errors import InstanceTooLarge

DEFAULT_SEARCH_LIMIT = 10**6
DEFAULT_REPLAN_EVERY = 4  # decode steps between re-plans (scheduler.py:23)


@dataclass(frozen=True)
class Task:
    node: int
    n_q: int
    n: int

    def __post_init__(self):
        if self.n < 1 or self.n_q < 1:
            raise ValueError(f"task ({self.n_q}, {self.n}) must have n, n_q >= 1")


@dataclass(frozen=True)
class Subtask:
    task_index: int
    node: int
    start: int
    stop: int
    cost_ms: float


@dataclass(frozen=True)
class Assignment:
    block_of: tuple
    loads: tuple

    @property
    def makespan_ms(self) -> float:
        return max(self.loads) if self.loads else 0.0


@dataclass(frozen=True)
class DivisionPlan:
    tasks: tuple
    b_q: tuple
    b_k: tuple
    subtasks: tuple
    assignment: Assignment
    blocks: int
    makespan_ms: float
    cost_l_ms: float | None = None
    search_truncated: bool = False

    def to_dict(self) -> dict:
        return {
            "tasks": [{"node": t.node, "b_q": bq, "b_k": bk}
                      for t, bq, bk in zip(self.tasks, self.b_q, self.b_k)],
            "assignment": {str(i): b for i, b in enumerate(self.assignment.block_of)},
            "blocks": self.blocks,
            "makespan_ms": self.makespan_ms,
            "cost_l_ms": self.cost_l_ms,
        }


def _arr(xs, dt):
    return np.ascontiguousarray(np.asarray(xs, dtype=dt))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _task_arrays(tasks):
    tasks = list(tasks)
    node = _arr([t.node for t in tasks], np.int64)
    nq = _arr([t.n_q for t in tasks], np.int64)
    n = _arr([t.n for t in tasks], np.int64)
    return tasks, node, nq, n


def slice_ranges(n: int, b: int):
    """Contiguous ceil-size slices, b clamped to 1..n (scheduler.py:81-86)."""
    L = _lib.lib()
    cnt = C.c_int64()
    _lib.check(L.codec_slice_ranges(int(n), int(b), None, 0, C.byref(cnt)))
    buf = np.zeros(2 * cnt.value, dtype=np.int64)
    _lib.check(L.codec_slice_ranges(int(n), int(b), _ptr(buf, C.c_int64), cnt.value, C.byref(cnt)))
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt.value)]


def canonical_division(n: int, b: int) -> int:
    """Slice count actually produced for a request of b (scheduler.py:89-92)."""
    L = _lib.lib()
    cnt = C.c_int64()
    _lib.check(L.codec_slice_ranges(int(n), int(b), None, 0, C.byref(cnt)))
    return cnt.value


def tasks_from_forest(forest, head_multiplicity: int = 1) -> list:
    """One task per node with a non-empty query set (scheduler.py:95-103)."""
    return [Task(node.id, len(node.query_set) * head_multiplicity, node.len)
            for node in forest.nodes[1:] if node.query_set]


def device_tasks(forest, group_size: int, rows_per_tile: int = 256) -> list:
    """Node tasks split into consecutive query-set chunks of at most
    rows_per_tile // g requests (g = q heads per kv head), n_q counted in
    query-head rows (head_multiplicity = g). Each chunk is what one
    tcgen05 CTA (or GEMV CTA group) processes, so the planner balances the
    real device units. Execute() maps chunk i of node n back to its
    requests by the order the node's tasks appear."""
    g = int(group_size)
    per = max(1, rows_per_tile // g)
    out = []
    for node in forest.nodes[1:]:
        qs = node.query_set
        for c in range(0, len(qs), per):
            out.append(Task(node.id, len(qs[c:c + per]) * g, node.len))
    return out


TC_MIN_ROWS = 16  # query-head rows from which a subtask takes the tensor-core kernel (device_table.h)
# with the multi-request suffix kernel: slices up to this many rows take it
# (device_table.h kMultiMaxRows; the library and this module read the same
# CODEC_MULTI_MAX_ROWS override)
MULTI_MAX_ROWS = int(os.environ.get("CODEC_MULTI_MAX_ROWS", "16"))
# transposed tensor-core kernel (kern_tct.cu): nodes with at most this many
# query-head rows in all (device_table.h kTctMaxRows; the library reads the
# same CODEC_TCT_MAX_ROWS override), cut into slices of TCT_SLICE tokens
TCT_MAX_ROWS = int(os.environ.get("CODEC_TCT_MAX_ROWS", "64"))
TCT_WIDE_ROWS = 128  # with CODEC_FLAG_TCT_WIDE (device_table.h kTctRows)
TCT_SLICE = int(os.environ.get("CODEC_TCT_SLICE", "4096"))
TC_CTAS_PER_BLOCK = 2  # a tensor-core schedule block is a cta_group::2 CTA pair (device_table.h)
SUFFIX_SLICE = 4096    # longest KV slice one suffix-kernel CTA streams (plan_device)
SUFFIX_SLICE_MIN = 320  # shortest slice plan_device cuts a suffix / lightly shared node into (g = 4, d = 128)
# Partial-output pricing: a slice writes one partial (o[d], m, l) per
# query-head row and the merge reads it back, 2 * (4 d + 8) bytes per row;
# plan_device keeps that below this fraction of the slice's KV bytes
PARTIAL_FRACTION = float(os.environ.get("CODEC_PARTIAL_FRACTION", "0.026"))


def partial_bytes(rows: int, d: int = 128) -> int:
    """HBM bytes one extra slice costs in partial outputs: written by the
    split kernel, read by the merge (fp32 o[d] plus (m, l) per row)."""
    return int(rows) * 2 * (4 * int(d) + 8)


def min_slice_tokens(g: int, d: int = 128, elem: int = 2) -> int:
    """Shortest slice whose partial bytes stay within PARTIAL_FRACTION of
    its KV bytes (2 * d * elem per token per kv head), on 64-token steps:
    320 for the Llama-3-8B shape (g = 4), 640 for g = 8."""
    t = partial_bytes(g, d) / (PARTIAL_FRACTION * 2 * d * elem)
    return max(64, -(-int(math.ceil(t)) // 64) * 64)
SUFFIX_WAVES = float(os.environ.get("CODEC_SUFFIX_WAVES", "2"))  # suffix-grid CTA waves (of 6 CTAs per SM) plan_device aims for


def concat_plans(plans) -> DivisionPlan:
    """One DivisionPlan from several plans over disjoint task lists (task
    indices and block ids are offset; makespan = max)."""
    tasks, subs, owner, loads, bk = [], [], [], [], []
    t_off = b_off = 0
    for p in plans:
        tasks.extend(p.tasks)
        bk.extend(p.b_k)
        subs.extend(Subtask(st.task_index + t_off, st.node, st.start, st.stop, st.cost_ms) for st in p.subtasks)
        owner.extend(b + b_off for b in p.assignment.block_of)
        loads.extend(p.assignment.loads)
        t_off += len(p.tasks)
        b_off += p.blocks
    return DivisionPlan(tasks=tuple(tasks), b_q=(1,) * len(tasks), b_k=tuple(bk), subtasks=tuple(subs),
                        assignment=Assignment(tuple(owner), tuple(loads)), blocks=b_off,
                        makespan_ms=max(p.makespan_ms for p in plans),
                        cost_l_ms=plans[0].cost_l_ms, search_truncated=any(p.search_truncated for p in plans))


def node_kernel(rows: int, n_requests: int, multi: bool = True, tct: bool = True, node_rows: int | None = None,
                tct_wide: bool = False) -> str:
    """Which kernel runs a slice with `rows` query-head rows of
    `n_requests` requests of a node with `node_rows` rows in all (default:
    rows) -- host_table.cpp's routing for bf16, d = 128, g <= 8: "tct"
    (transposed tcgen05 kernel: 2+ requests of a node of <= TCT_MAX_ROWS
    rows), "tc" (tcgen05 shared-node kernel),
    "multi" (multi-request mma.sync kernel) or "suffix" (single-request
    mma.sync kernel)."""
    lo = MULTI_MAX_ROWS if multi else TC_MIN_ROWS - 1
    tmax = TCT_WIDE_ROWS if tct_wide else TCT_MAX_ROWS
    if tct and n_requests >= 2 and (rows if node_rows is None else node_rows) <= tmax:
        return "tct"
    if rows > lo:
        return "tc"
    if multi and n_requests >= 2:
        return "multi"
    return "suffix"


def plan_device(forest, group_size: int, table: CostTable, h_local: int, sm_count: int = 148,
                tc_sm_budget: int = 0, search_limit: int = DEFAULT_SEARCH_LIMIT, page_size: int = 0,
                multi: bool = True, tct: bool = True, tct_wide: bool = False) -> DivisionPlan:
    """The B200 plan of one decode step. Shared nodes (more than
    MULTI_MAX_ROWS query-head rows per chunk; TC_MIN_ROWS with multi=False)
    stay whole here: on the tensor cores every KV tile costs the same (an
    M=256 MMA pair whatever the rows), so the device balancer in the task
    table (host_table.cpp) divides them itself -- stream-K over the CTA
    pairs, per kv head, into equal tile ranges with the row chunks of a
    slice in lockstep. Lightly shared and unshared nodes go to the mma.sync
    kernels (multi-request / single-request), whose CTAs are
    hardware-scheduled and stream at HBM speed regardless of order; long
    ones are cut into slices of <= SUFFIX_SLICE tokens. Returns one plan
    over both, in the reference's DivisionPlan form (any reference plan is
    accepted by execute() as well; its slices then bound the device
    pieces). With a paged pool (page_size > 0, paging.py) those nodes stay
    whole: a slice must start on a 32-token chunk boundary of its node."""
    tasks = device_tasks(forest, group_size)
    g = int(group_size)
    kind = [node_kernel(t.n_q, t.n_q // g, multi, tct, len(forest.node(t.node).query_set) * g, tct_wide)
            for t in tasks]
    tc = [t for t, k in zip(tasks, kind) if k == "tc"]
    tcts = [t for t, k in zip(tasks, kind) if k == "tct"]
    gv = [t for t, k in zip(tasks, kind) if k not in ("tc", "tct")]
    pairs = max(1, (tc_sm_budget or sm_count) // TC_CTAS_PER_BLOCK)
    plans = []
    if tc:
        plans.append(plan_uniform_bk(tc, table, pairs, 1))
    # transposed tensor-core kernel: one CTA per slice and kv head, slices
    # of <= TCT_SLICE tokens (a paged pool keeps nodes whole, like below)
    by_bk = {}
    for t in tcts:
        by_bk.setdefault(1 if page_size else max(1, -(-t.n // TCT_SLICE)), []).append(t)
    for bk in sorted(by_bk):
        plans.append(plan_uniform_bk(by_bk[bk], table, len(by_bk[bk]) * bk, bk))
    # mma.sync-kernel tasks: one CTA streams a slice at only a few tens of
    # GB/s (bytes in flight per CTA are bounded by its SMEM ring), so the
    # machine needs many CTAs: long slices are cut so the suffix grids hold
    # >= SUFFIX_WAVES waves of CTAs (6 per SM), never below
    # min_slice_tokens (each slice adds a partial to write and merge:
    # priced in HBM bytes, PARTIAL_FRACTION) nor above
    # SUFFIX_SLICE (a lightly shared 128K-token root in cfg4)
    work = sum(t.n for t in gv) * h_local
    target = max(1, int(sm_count * 6 * SUFFIX_WAVES))
    slice_min = min_slice_tokens(g, forest.d)
    slice_len = min(SUFFIX_SLICE, max(slice_min, -(-work // target)))
    slice_len = -(-slice_len // 64) * 64
    by_bk = {}
    for t in gv:
        by_bk.setdefault(1 if page_size else max(1, -(-t.n // slice_len)), []).append(t)
    for bk in sorted(by_bk):
        plans.append(plan_uniform_bk(by_bk[bk], table, len(by_bk[bk]) * bk, bk))
    return concat_plans(plans)


def lower_bound(tasks, table: CostTable, m: int, tol: float = 1e-4) -> float:
    """Eq. 4 bisection (scheduler.py:106-131)."""
    tasks, _, nq, n = _task_arrays(tasks)
    if not tasks:
        raise ValueError("no tasks to schedule")
    out = C.c_double()
    _lib.check(_lib.lib().codec_lower_bound(table.c_ref, len(tasks), _ptr(nq, C.c_int64), _ptr(n, C.c_int64),
                                            int(m), float(tol), C.byref(out)))
    return out.value


def division_caps(tasks, table: CostTable, cost_l: float) -> list:
    """Eq. 5 (scheduler.py:134-139)."""
    if cost_l <= 0:
        raise ValueError(f"cost_l must be positive, got {cost_l}")
    tasks, _, nq, n = _task_arrays(tasks)
    caps = np.zeros(len(tasks), dtype=np.int64)
    _lib.check(_lib.lib().codec_division_caps(table.c_ref, len(tasks), _ptr(nq, C.c_int64), _ptr(n, C.c_int64),
                                              float(cost_l), _ptr(caps, C.c_int64)))
    return [int(c) for c in caps]


def greedy_assign(subtask_costs, m: int) -> Assignment:
    """LPT (scheduler.py:142-155)."""
    if m < 1:
        raise ValueError(f"need m >= 1 blocks, got {m}")
    costs = _arr([float(c) for c in subtask_costs], np.float64)
    owner = np.zeros(len(costs), dtype=np.int32)
    loads = np.zeros(m, dtype=np.float64)
    _lib.check(_lib.lib().codec_greedy_assign(len(costs), _ptr(costs, C.c_double), int(m),
                                              _ptr(owner, C.c_int32), _ptr(loads, C.c_double)))
    return Assignment(tuple(int(b) for b in owner), tuple(float(x) for x in loads))


def _read_plan(handle, tasks) -> DivisionPlan:
    L = _lib.lib()
    try:
        info = _lib.PlanInfo()
        _lib.check(L.codec_plan_info_get(handle, C.byref(info)))
        S = info.n_subtasks
        bk = np.zeros(info.n_tasks, np.int64)
        st_task = np.zeros(S, np.int32)
        st_node = np.zeros(S, np.int64)
        st_a = np.zeros(S, np.int64)
        st_b = np.zeros(S, np.int64)
        st_c = np.zeros(S, np.float64)
        owner = np.zeros(S, np.int32)
        loads = np.zeros(info.blocks, np.float64)
        _lib.check(L.codec_plan_read(handle, _ptr(bk, C.c_int64), _ptr(st_task, C.c_int32),
                                     _ptr(st_node, C.c_int64), _ptr(st_a, C.c_int64), _ptr(st_b, C.c_int64),
                                     _ptr(st_c, C.c_double), _ptr(owner, C.c_int32), _ptr(loads, C.c_double)))
    finally:
        L.codec_plan_free(handle)
    subs = tuple(Subtask(int(a), int(b), int(c), int(d), float(e))
                 for a, b, c, d, e in zip(st_task, st_node, st_a, st_b, st_c))
    cost_l = None if math.isnan(info.cost_l_ms) else float(info.cost_l_ms)
    return DivisionPlan(tasks=tuple(tasks), b_q=(1,) * len(tasks), b_k=tuple(int(x) for x in bk),
                        subtasks=subs,
                        assignment=Assignment(tuple(int(b) for b in owner), tuple(float(x) for x in loads)),
                        blocks=info.blocks, makespan_ms=float(info.makespan_ms), cost_l_ms=cost_l,
                        search_truncated=bool(info.truncated))


def divide_and_schedule(tasks, table: CostTable, m: int, search_limit: int = DEFAULT_SEARCH_LIMIT,
                        on_overflow: str = "fallback") -> DivisionPlan:
    """Grid search over capped divisions scored by LPT; ties toward fewer
    subtasks then lexicographic b_k; {identity, all-at-cap} past the
    limit (scheduler.py:187-222)."""
    tasks, node, nq, n = _task_arrays(tasks)
    if not tasks:
        raise ValueError("no tasks to schedule")
    if on_overflow not in ("fallback", "raise"):
        raise ValueError(f"on_overflow must be fallback or raise, got {on_overflow!r}")
    h = C.c_void_p()
    _lib.check(_lib.lib().codec_divide_and_schedule(
        table.c_ref, len(tasks), _ptr(node, C.c_int64), _ptr(nq, C.c_int64), _ptr(n, C.c_int64), int(m),
        int(search_limit), 1 if on_overflow == "raise" else 0, C.byref(h)))
    return _read_plan(h, tasks)


def plan_uniform_bk(tasks, table: CostTable, m: int, bk: int, cost_l: float | None = None) -> DivisionPlan:
    """Fixed division count for every task (scheduler.py:225-233)."""
    tasks, node, nq, n = _task_arrays(tasks)
    if bk < 1:
        raise ValueError(f"b_k must be >= 1, got {bk}")
    h = C.c_void_p()
    _lib.check(_lib.lib().codec_plan_uniform(
        table.c_ref, len(tasks), _ptr(node, C.c_int64), _ptr(nq, C.c_int64), _ptr(n, C.c_int64), int(m),
        int(bk), float("nan") if cost_l is None else float(cost_l), C.byref(h)))
    return _read_plan(h, tasks)


def makespan(plan: DivisionPlan, table: CostTable) -> float:
    """Recompute the maximum per-block load (scheduler.py:236-242)."""
    from .cost_model import estimate
    loads = [0.0] * plan.blocks
    for st, b in zip(plan.subtasks, plan.assignment.block_of):
        task = plan.tasks[st.task_index]
        loads[b] += estimate(table, task.n_q, st.stop - st.start)
    return max(loads) if loads else 0.0


def brute_force_guard(tasks, m, caps):
    """The reference's exact oracle (scheduler.py:245-324) is test-only
    and lives in oracle/; this keeps its guard semantics for callers."""
    if len(tasks) > 4 or m > 4 or any(c > 8 for c in caps):
        raise InstanceTooLarge(
            f"brute force needs t <= 4, m <= 4, caps <= 8; got t={len(tasks)}, m={m}, caps={list(caps)}")
