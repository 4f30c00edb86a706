"""Oracle: cost model, task division and LPT block schedule (the K1
planner), restated in float64 Python with the reference's operation
order so results can be compared bit-for-bit.

Reference: prefixdec/cost_model.py and prefixdec/scheduler.py.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np

SEARCH_LIMIT = 10**6  # scheduler.py:22


@dataclass(frozen=True)
class Grid:
    """Cost grid: cost[n_index][nq_index] in ms (cost_model.py:32-53)."""

    nq: tuple
    n: tuple
    cost: np.ndarray


def parse_profile(text: str) -> Grid:
    """CSV '# meta' lines, header n_q,n,cost_ms, one row per cell
    (cost_model.py:102-150). Validation is the product's job; the oracle
    only needs the grid."""
    cells = {}
    for line in text.splitlines():
        if not line.strip() or line.startswith("#") or line.startswith("n_q"):
            continue
        a, b, c = line.split(",")
        cells[(int(a), int(b))] = float(c)
    nq = tuple(sorted({k[0] for k in cells}))
    n = tuple(sorted({k[1] for k in cells}))
    cost = np.array([[cells[(q, x)] for q in nq] for x in n], dtype=np.float64)
    return Grid(nq, n, cost)


def _segment(knots, x):
    """Clamped bracket of x in ascending knots (cost_model.py:56-65)."""
    if x <= knots[0]:
        return 0, 0
    last = len(knots) - 1
    if x >= knots[last]:
        return last, last
    hi = 1
    while knots[hi] < x:
        hi += 1
    return hi - 1, hi


def estimate(grid: Grid, n_q, n) -> float:
    """Bilinear: linear in n_q, linear in log2 n, clamped at the edge knots
    (cost_model.py:68-84). Same association order as the reference."""
    a, b = _segment(grid.nq, n_q)
    tq = 0.0 if a == b else (n_q - grid.nq[a]) / (grid.nq[b] - grid.nq[a])
    c, d = _segment(grid.n, n)
    if c == d:
        tn = 0.0
    else:
        la = math.log2(grid.n[c])
        lb = math.log2(grid.n[d])
        tn = (math.log2(n) - la) / (lb - la)
    g = grid.cost
    lo_row = g[c, a] + tq * (g[c, b] - g[c, a])
    hi_row = g[d, a] + tq * (g[d, b] - g[d, a])
    return float(lo_row + tn * (hi_row - lo_row))


def slices(n: int, b: int):
    """Contiguous ceil-size slices; b clamped into 1..n
    (scheduler.py:81-86)."""
    b = min(max(b, 1), n)
    step = (n + b - 1) // b
    return [(s, min(s + step, n)) for s in range(0, n, step)]


def n_slices(n: int, b: int) -> int:
    """Slice count actually produced (scheduler.py:89-92)."""
    b = min(max(b, 1), n)
    step = (n + b - 1) // b
    return (n + step - 1) // step


def node_tasks(qsets, length, head_multiplicity=1):
    """(node, n_q, n) for every node carrying queries
    (scheduler.py:95-103)."""
    return [
        (nid, len(qsets[nid]) * head_multiplicity, length[nid])
        for nid in range(1, len(length))
        if qsets[nid]
    ]


def py_sum(values) -> float:
    """The builtin sum() of CPython >= 3.12 over floats, spelled out: the
    int start 0 is absorbed by the first item, the rest are added with
    Neumaier compensation, and the compensation is folded in at the end
    if it is finite and non-zero (Python/bltinmodule.c builtin_sum_impl).
    The reference's `sum(...)` calls (scheduler.py:114, :123) round this
    way, so a bit-exact restatement must too."""
    it = iter(values)
    try:
        total = float(next(it))
    except StopIteration:
        return 0
    comp = 0.0
    for x in it:
        t = total + x
        if abs(total) >= abs(x):
            comp += (total - t) + x
        else:
            comp += (x - t) + total
        total = t
    if comp and math.isfinite(comp):
        total += comp
    return total


def lower_bound(tasks, grid, m, tol=1e-4) -> float:
    """Eq. 4 bisection (scheduler.py:106-131)."""
    full = [estimate(grid, nq, n) for _, nq, n in tasks]
    hi = py_sum(full)
    lo = max(estimate(grid, nq, 1) for _, nq, _n in tasks)

    def ok(c):
        vol = 0.0
        for (_, nq, n), f in zip(tasks, full):
            vol += py_sum(estimate(grid, nq, e - s) for s, e in slices(n, math.ceil(f / c)))
        return vol / m <= c

    if ok(lo):
        return lo
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if ok(mid):
            hi = mid
        else:
            lo = mid
    return hi


def caps(tasks, grid, cost_l):
    """Eq. 5 per-task division ceiling (scheduler.py:134-139)."""
    return [math.ceil(estimate(grid, nq, n) / cost_l) for _, nq, n in tasks]


def lpt(costs, m):
    """LPT: descending cost (ties: lower index), each onto the least
    loaded block (ties: lower block) (scheduler.py:142-155)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * m
    owner = [0] * len(costs)
    for i in order:
        best = 0
        for j in range(1, m):
            if load[j] < load[best]:
                best = j
        owner[i] = best
        load[best] += costs[i]
    return owner, load


@dataclass(frozen=True)
class Plan:
    b_k: tuple
    subtasks: tuple  # (task_index, node, start, stop, cost)
    block_of: tuple
    loads: tuple
    makespan: float
    cost_l: float | None
    truncated: bool


def plan_for(tasks, b_k, grid, m, cost_l=None, truncated=False) -> Plan:
    """Expand a division into subtasks and LPT-pack them
    (scheduler.py:158-180)."""
    bk = tuple(n_slices(n, b) for (_, _, n), b in zip(tasks, b_k))
    subs = []
    for j, ((node, nq, n), b) in enumerate(zip(tasks, bk)):
        for s, e in slices(n, b):
            subs.append((j, node, s, e, estimate(grid, nq, e - s)))
    owner, load = lpt([st[4] for st in subs], m)
    return Plan(bk, tuple(subs), tuple(owner), tuple(load),
                max(load) if load else 0.0, cost_l, truncated)


def divide_and_schedule(tasks, grid, m, limit=SEARCH_LIMIT) -> Plan:
    """Grid search over capped divisions; key (makespan, #subtasks, b_k);
    {identity, all-at-cap} fallback past `limit` (scheduler.py:187-222)."""
    cost_l = lower_bound(tasks, grid, m)
    cp = caps(tasks, grid, cost_l)
    options = [
        sorted({n_slices(n, b) for b in range(1, max(1, min(c, n)) + 1)})
        for (_, _, n), c in zip(tasks, cp)
    ]
    total = 1
    for o in options:
        total *= len(o)
    if total > limit:
        combos = [(1,) * len(tasks), tuple(o[-1] for o in options)]
        truncated = True
    else:
        combos = itertools.product(*options)
        truncated = False
    best, best_key = None, None
    for bk in combos:
        p = plan_for(tasks, bk, grid, m, cost_l, truncated)
        key = (p.makespan, len(p.subtasks), p.b_k)
        if best_key is None or key < best_key:
            best, best_key = p, key
    return best


def uniform(tasks, grid, m, bk, cost_l=None) -> Plan:
    """Same division count for every task (scheduler.py:225-233)."""
    return plan_for(tasks, (bk,) * len(tasks), grid, m, cost_l)
