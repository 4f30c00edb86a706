"""B200 per-CTA cost profile (K6) in the reference's CSV format
(cost_model.py:102-160): cost_ms of one CTA processing n_q query-head
rows of one kv head over n tokens.

    python -m paper_2505_17694_b200.profile_b200 model    # analytic table
    python -m paper_2505_17694_b200.profile_b200 measure  # time kernels (GPU)

`model` derives the table from the B200 roofline: GEMV CTAs (< 16 rows)
stream K+V (512 B/token at d=128 bf16) at a per-SM share of measured HBM
bandwidth; tensor-core CTAs cost a fixed time per 128-token tile per
128-row M tile. `measure` replaces it with CUDA-event timings of the real
kernels on single-node forests (one CTA per SM, all SMs busy) and writes
profiles/b200_d128.csv.
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

from .cost_model import CostTable, dump_profile

NQ_KNOTS = (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024)
N_KNOTS = (64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072)
OUT = Path(__file__).resolve().parent / "profiles" / "b200_d128.csv"


def model_cost(n_q: int, n: int, hbm_gbs: float = 6515.7, sms: int = 148, tile_us: float = 0.60) -> float:
    if n_q < 16:
        per_sm = hbm_gbs * 1e9 / sms
        return 0.003 + n * 512 / per_sm * 1e3
    tiles = math.ceil(n / 128) * math.ceil(n_q / 128)
    return 0.004 + tiles * tile_us * 1e-3


def model_table() -> CostTable:
    grid = np.array([[model_cost(q, n) for q in NQ_KNOTS] for n in N_KNOTS])
    return CostTable(NQ_KNOTS, N_KNOTS, grid, meta={"d": "128", "hardware": "b200", "source": "roofline-model"})


def measure_table(reps: int = 5) -> CostTable:
    import torch

    from . import DecodeStep, Task, forest_from_pool, plan_uniform_bk
    from .cost_model import load_profile

    dev = torch.device("cuda")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid = np.zeros((len(N_KNOTS), len(NQ_KNOTS)))
    h_kv, d = sms, 128   # one CTA per SM: `sms` kv heads, g = 1 row per request... (rows = n_q)
    for i, n in enumerate(N_KNOTS):
        for j, nq in enumerate(NQ_KNOTS):
            g = 1
            reqs = nq
            f = forest_from_pool([0], [n], [(1,)] * reqs, h_kv, d)
            k = torch.randn(h_kv, n, d, device=dev, dtype=torch.bfloat16) * (1 / math.sqrt(d))
            v = torch.randn_like(k)
            q = torch.randn(reqs, h_kv * g, d, device=dev, dtype=torch.bfloat16) * (1 / math.sqrt(d))
            tab = load_profile(OUT) if OUT.exists() else model_table()
            plan = plan_uniform_bk([Task(1, reqs, n)], tab, 1, 1)
            step = DecodeStep(f, plan, h_kv * g, "bfloat16")
            for _ in range(2):
                step(q, k, v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                step(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            grid[i, j] = e0.elapsed_time(e1) / reps
            print(json.dumps({"n": n, "n_q": nq, "ms": grid[i, j]}), flush=True)
    return CostTable(NQ_KNOTS, N_KNOTS, grid, meta={"d": "128", "hardware": "b200", "source": "measured"})


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "model"
    table = model_table() if mode == "model" else measure_table()
    OUT.parent.mkdir(parents=True, exist_ok=True)
    dump_profile(table, OUT)
    print(OUT)
