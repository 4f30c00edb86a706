"""A/B of library variants on a config: the bench's autotune pass (best
step time over tensor-core SM budgets, short windows) plus the suffix
kernel alone, for the library named by CODEC_B200_LIB.

    CODEC_B200_LIB=paper_2505_17694_b200/_codec_b200_<tag>.so python tools/ab.py cfg2 [cfg3 ...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def suffix_alone(ns, n=20):
    st = ns.step.with_budget(ns.sms, flags=16 | 64)  # SKIP_TC | SKIP_MERGE
    for _ in range(3):
        st(ns.q_dev, ns.kp, ns.vp, out=ns.out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        st(ns.q_dev, ns.kp, ns.vp, out=ns.out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


# (CODEC_MULTI_MAX_ROWS is read by both the library and scheduler.py)
if os.environ.get("SUFFIX_WAVES"):
    from paper_2505_17694_b200 import scheduler
    scheduler.SUFFIX_WAVES = float(os.environ["SUFFIX_WAVES"])
if os.environ.get("PARTIAL_FRACTION"):
    from paper_2505_17694_b200 import scheduler
    scheduler.PARTIAL_FRACTION = float(os.environ["PARTIAL_FRACTION"])
if os.environ.get("SUFFIX_SLICE"):
    from paper_2505_17694_b200 import scheduler
    scheduler.SUFFIX_SLICE = int(os.environ["SUFFIX_SLICE"])
for cfg in sys.argv[1:] or ["cfg2"]:
    ns = bench.prepare(cfg, torch.device("cuda", 0), flags=int(os.environ.get("FLAGS", "0")))
    best = min(ns.tune_ms.values())
    print(json.dumps({"lib": os.path.basename(os.environ.get("CODEC_B200_LIB", "default")), "config": cfg,
                      "suffix_slice": os.environ.get("SUFFIX_SLICE"), "flags": os.environ.get("FLAGS"),
                      "best_ms": best, "budget": ns.budget, "suffix_alone_ms": round(suffix_alone(ns), 4),
                      "tune_ms": ns.tune_ms}), flush=True)
    del ns
    torch.cuda.empty_cache()
