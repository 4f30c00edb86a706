"""RunReport lines: the reference CLI's per-point
report (cli.py:130-184; schema schemas/report.schema.json) from a forest
and its plan, so B200 runs report in the schema the reference's tooling
reads. bench.py embeds one for its workload.

Fields: the workload description, the exact KV-read traffic
(traffic_report, metrics.py:36-70), the plan summary, the per-request
baseline makespan (each request's whole path on one block, LPT over the
blocks: cli.py:161-162), the simulated speedup over it, the ablation flags
and optionally the max-norm relative error against the oracle.
"""
from __future__ import annotations

from .cost_model import estimate
from .metrics import traffic_report
from .scheduler import DEFAULT_REPLAN_EVERY, greedy_assign

ABLATIONS = ("share_tree", "partition", "parallel_reduce")
FAMILIES = ("two_level", "full_tree", "degenerate", "shared_ratio")


def run_report(forest, plan, table, blocks: int, workload: dict, *, max_rel_err=None,
               replan_every: int = DEFAULT_REPLAN_EVERY, ablation=None, element_size=None) -> dict:
    """The RunReport dict of one workload point (cli.py:161-184)."""
    base = greedy_assign([estimate(table, 1, forest.request_len(r)) for r in range(forest.bs)], blocks).makespan_ms
    summary = {"tasks": len(plan.tasks), "subtasks": len(plan.subtasks), "makespan_ms": plan.makespan_ms,
               "cost_l_ms": plan.cost_l_ms, "replan_every": int(replan_every)}
    if plan.search_truncated:
        summary["search_truncated"] = True
    flags = {name: True for name in ABLATIONS}
    flags.update(ablation or {})
    rep = {"workload": workload, "traffic": traffic_report(forest, element_size).to_dict(), "plan_summary": summary,
           "baseline_makespan_ms": base, "sim_speedup": base / plan.makespan_ms, "ablation_flags": flags}
    if max_rel_err is not None:
        rep["max_rel_err_vs_oracle"] = float(max_rel_err)
    return rep


def _num(x):
    return isinstance(x, (int, float)) and not isinstance(x, bool)


def check_report(rep: dict) -> None:
    """Structural check against the RunReport schema (required keys, no
    extra keys, value types and bounds); ValueError on the first problem."""
    def need(obj, where, req, opt=()):
        if not isinstance(obj, dict):
            raise ValueError(f"{where} must be an object")
        miss = [k for k in req if k not in obj]
        if miss:
            raise ValueError(f"{where} misses {miss}")
        extra = sorted(set(obj) - set(req) - set(opt))
        if extra:
            raise ValueError(f"{where} has unknown keys {extra}")

    need(rep, "report", ("workload", "traffic", "plan_summary", "baseline_makespan_ms", "sim_speedup",
                         "ablation_flags"), ("max_rel_err_vs_oracle",))
    w = rep["workload"]
    need(w, "workload", ("family", "params", "seed", "dims"))
    if w["family"] not in FAMILIES:
        raise ValueError(f"workload.family {w['family']!r} not in {FAMILIES}")
    if not all(_num(v) for v in w["params"].values()):
        raise ValueError("workload.params must be numbers")
    if not (isinstance(w["seed"], int) and w["seed"] >= 0):
        raise ValueError("workload.seed must be a non-negative integer")
    need(w["dims"], "workload.dims", ("h_q", "h_kv", "d"))
    if not all(isinstance(v, int) and v >= 1 for v in w["dims"].values()):
        raise ValueError("workload.dims must be positive integers")
    t = rep["traffic"]
    need(t, "traffic", ("kv_rows_codec", "kv_rows_baseline", "bytes_codec", "bytes_baseline", "reduction_ratio",
                        "nq_bar"))
    for k in ("kv_rows_codec", "kv_rows_baseline", "bytes_codec", "bytes_baseline"):
        if not (isinstance(t[k], int) and t[k] >= 0):
            raise ValueError(f"traffic.{k} must be a non-negative integer")
    for k in ("reduction_ratio", "nq_bar"):
        if not (_num(t[k]) and t[k] >= 1):
            raise ValueError(f"traffic.{k} must be a number >= 1")
    p = rep["plan_summary"]
    need(p, "plan_summary", ("tasks", "subtasks", "makespan_ms", "cost_l_ms"), ("replan_every", "search_truncated"))
    if not (_num(p["makespan_ms"]) and p["makespan_ms"] >= 0) or not (p["cost_l_ms"] is None or _num(p["cost_l_ms"])):
        raise ValueError("plan_summary costs must be numbers")
    if "replan_every" in p and not (isinstance(p["replan_every"], int) and p["replan_every"] >= 1):
        raise ValueError("plan_summary.replan_every must be an integer >= 1")
    for k in ("baseline_makespan_ms", "sim_speedup"):
        if not (_num(rep[k]) and rep[k] >= 0):
            raise ValueError(f"{k} must be a non-negative number")
    need(rep["ablation_flags"], "ablation_flags", ABLATIONS)
    if not all(isinstance(v, bool) for v in rep["ablation_flags"].values()):
        raise ValueError("ablation_flags must be booleans")
    if "max_rel_err_vs_oracle" in rep and not (_num(rep["max_rel_err_vs_oracle"]) and rep["max_rel_err_vs_oracle"] >= 0):
        raise ValueError("max_rel_err_vs_oracle must be a non-negative number")
