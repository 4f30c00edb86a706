"""B200-native prefix-shared decode attention (CoDec, arXiv 2505.17694).

Drop-in for the hot path of the reference package `prefixdec`: the same
entry points (build_forest, QueryBatch, tasks_from_forest,
divide_and_schedule, execute, pac, por, ...) backed by a C-ABI shared
library (_codec_b200.so) with hand-written sm_100a kernels:
tcgen05/TMEM/TMA shared-node attention, a bulk-async warp-shuffle GEMV
for unshared suffixes and a log-sum-exp merge; the planner (cost model,
task division, LPT schedule) runs in C++ and is bit-exact with the
reference. There is no CPU fallback.
"""
from .attention import PartialResult, empty_partial, finalize, pac, por
from .cost_model import (CostTable, default_profile_path, dump_profile, estimate, load_default_profile,
                         load_profile, profile_synthetic)
from .errors import *  # noqa: F401,F403
from .executor import BlockPool, DecodeStep, autotune_step, execute
from .reduce import PartialTree, merge_schedule, reduce_tree, sequential_schedule
from .serialize import dump_forest, load_forest
from .forest import (Forest, KvNode, QueryBatch, Violation, build_forest, forest_from_pool, node_query_set,
                     prefix_path, validate)
from .metrics import TrafficReport, count_kv_reads, device_work, traffic_report, weighted_avg_sharing
from .scheduler import (Assignment, DivisionPlan, Subtask, Task, canonical_division, device_tasks,
                        concat_plans, divide_and_schedule, division_caps, greedy_assign, lower_bound, makespan, plan_device,
                        plan_uniform_bk, slice_ranges, tasks_from_forest)

__version__ = "0.1.0"
