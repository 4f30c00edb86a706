"""B200 per-CTA cost profile (K6) in the reference's CSV format
(cost_model.py:102-160): cost_ms of one CTA processing n_q query-head
rows of one kv head over n tokens.

    python -m paper_2505_17694_b200.profile_b200 model    # analytic table
    python -m paper_2505_17694_b200.profile_b200 measure  # time kernels (GPU)

`model` derives the table from the B200 roofline: GEMV CTAs (< 16 rows)
stream K+V (512 B/token at d=128 bf16) at a per-SM share of measured HBM
bandwidth; tensor-core CTAs cost a fixed time per 128-token tile per
128-row M tile. `measure` replaces it with CUDA-event timings of the real
kernels (see measure_table: one work unit on one CTA slot with every slot
busy, graph-replayed, launch overhead excluded) and writes
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


def measure_table(reps: int = 40, h_q: int = 32, h_kv: int = 8, d: int = 128) -> CostTable:
    """cost_ms(n_q, n) = device time of ONE work unit -- one kv head of a
    subtask of n_q requests x n tokens -- on one CTA slot of the kernel the
    device router picks for it (a CTA pair of the tensor-core kernel for
    more than MULTI_MAX_ROWS query-head rows, a CTA of the multi-request or
    the suffix kernel below), with every slot of the GPU busy: U identical
    single-node trees, the step's other kernels skipped, the launch replayed
    from a CUDA graph (no launch overhead), kernel time / waves of units."""
    import torch

    from . import DecodeStep, device_tasks, forest_from_pool, plan_uniform_bk
    from .executor import FLAG_NO_MULTI  # noqa: F401  (documented knob)
    from .scheduler import MULTI_MAX_ROWS, TC_CTAS_PER_BLOCK, node_kernel

    dev = torch.device("cuda")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    g = h_q // h_kv
    grid = np.zeros((len(N_KNOTS), len(NQ_KNOTS)))
    table = model_table()
    slots_of = {"tc": sms // TC_CTAS_PER_BLOCK, "multi": sms * 3, "suffix": sms * 6}
    skip = {"tc": 8 | 32 | 64, "multi": 8 | 16 | 64, "suffix": 8 | 16 | 64}
    for i, n in enumerate(N_KNOTS):
        for j, nq in enumerate(NQ_KNOTS):
            kind = node_kernel(nq * g, nq, True)
            lanes = -(-nq * g // 256) if kind == "tc" else 1
            slots = slots_of[kind]
            per_tree = h_kv * lanes
            U = max(1, -(-2 * slots // per_tree))           # ~2 full waves of units
            U = max(1, min(U, (1 << 25) // (n * h_kv)))     # bounded pool (<= 2^25 token-heads)
            f = forest_from_pool([0] * U, [n] * U, [(t + 1,) for t in range(U) for _ in range(nq)], h_kv, d)
            T = f.total_tokens
            k = (torch.randn(h_kv, T, d, device=dev) / math.sqrt(d)).to(torch.bfloat16)
            v = (torch.randn(h_kv, T, d, device=dev) / math.sqrt(d)).to(torch.bfloat16)
            q = (torch.randn(f.bs, h_q, d, device=dev) / math.sqrt(d)).to(torch.bfloat16)
            plan = plan_uniform_bk(device_tasks(f, g), table, slots, 1)
            step = DecodeStep(f, plan, h_q, "bfloat16", flags=skip[kind], tc_sm_budget=sms, concurrent=False)
            out = torch.empty((f.bs, h_q, d), dtype=torch.float32, device=dev)
            replay = step.capture(q, k, v, out)
            for _ in range(3):
                replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            units = U * per_tree
            waves = units / slots if kind == "tc" else math.ceil(units / slots)  # TC: stream-K spreads tiles evenly
            # a kv head of the subtask = `lanes` units (256-row chunks) on the tensor cores
            grid[i, j] = ms / waves * lanes
            print(json.dumps({"n": n, "n_q": nq, "kernel": kind, "trees": U, "units": units, "slots": slots,
                              "step_ms": ms, "unit_ms": grid[i, j]}), flush=True)
            del step, k, v, q, out
            torch.cuda.empty_cache()
    return CostTable(NQ_KNOTS, N_KNOTS, grid,
                     meta={"d": "128", "hardware": "b200", "source": "measured",
                           "unit": f"one kv head of a subtask (all its 256-row tensor-core lanes) on one CTA slot, "
                                   f"h_q {h_q} / h_kv {h_kv}, every slot busy, graph replay"})


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "model"
    table = model_table() if mode == "model" else measure_table()
    OUT.parent.mkdir(parents=True, exist_ok=True)
    dump_profile(table, OUT)
    print(OUT)
