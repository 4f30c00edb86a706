"""Golden violations of the reference's validate() (forest.py:266-363) on
the corrupted forests of tests/recipes.py (VALIDATE_CASES), recorded by
running the real reference. Run: python tests/golden/make_validate_golden.py"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, os.environ.get("PREFIXDEC_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

import prefixdec as R  # noqa: E402

from recipes import VALIDATE_CASES, mutate, validate_forest_specs  # noqa: E402

out = {}
for case in VALIDATE_CASES:
    specs, paths = validate_forest_specs()
    f = mutate(R.build_forest(specs, paths), case)
    out[case] = [[v.code, v.message, v.node, v.request] for v in R.validate(f)]
(HERE / "validate.json").write_text(json.dumps(out, indent=1) + "\n")
print({k: len(v) for k, v in out.items()})

# load_profile error contract
import io  # noqa: E402

from recipes import PROFILE_CASES  # noqa: E402

prof = {}
for name, text in PROFILE_CASES.items():
    try:
        t = R.load_profile(io.StringIO(text))
        buf = io.StringIO()
        R.dump_profile(t, buf)
        prof[name] = ["ok", buf.getvalue()]
    except Exception as e:  # noqa: BLE001
        prof[name] = [type(e).__name__, str(e)]
(HERE / "profile_errors.json").write_text(json.dumps(prof, indent=1) + "\n")
print(prof)

# merge_schedule / sequential_schedule (executor.py:86-117)
import numpy as np  # noqa: E402
from prefixdec.executor import merge_schedule, sequential_schedule  # noqa: E402

rng = np.random.default_rng(5)
sched = {"balanced": [], "sequential": []}
for _ in range(40):
    L = int(rng.integers(1, 6))
    counts = [int(x) for x in rng.integers(0, 7, size=L)]
    sched["balanced"].append([L, counts, [[list(p) for p in rnd] for rnd in merge_schedule(L, counts)]])
for total in range(0, 9):
    sched["sequential"].append([total, [[list(p) for p in rnd] for rnd in sequential_schedule(total)]])
(HERE / "schedules.json").write_text(json.dumps(sched) + "\n")

# RunReport lines (cli.py:130-184, schemas/report.schema.json) of small
# workloads, plan on the bundled A100 profile (no execution: timing-free)
from prefixdec.cli import run_point  # noqa: E402
from prefixdec.cost_model import load_default_profile  # noqa: E402
from prefixdec.workloads import Dims, WorkloadSpec  # noqa: E402

reports = []
for fam, params, blocks in (("two_level", {"shared_len": 1024, "leaf_len": 64, "batch": 16}, 8),
                            ("two_level", {"shared_len": 4096, "leaf_len": 300, "batch": 40}, 18),
                            ("full_tree", {"arity": 3, "depth": 3, "node_len": 200}, 6)):
    spec = WorkloadSpec(fam, params, 0, Dims(8, 4, 16))
    rep, _, _ = run_point(spec, load_default_profile(), blocks=blocks, workers=1, fp32=False, oracle=False,
                          ablation={"share_tree": True, "partition": True, "parallel_reduce": True},
                          force_bk=None, replan_every=4)
    reports.append({"blocks": blocks, "report": rep})
(HERE / "reports.json").write_text(json.dumps(reports, indent=1) + "\n")
