"""Experiment: how much does the tensor-core kernel's L2 traffic slow the
concurrent suffix stream? cfg2 step over SM budgets with the TC kernel's
K/V loads on (normal) and off (CODEC_FLAG_DBG_NO_LOADS: timing only, wrong
output) -- needs the -DCODEC_TC_DEBUG build (CODEC_B200_LIB=..._dbg.so)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
for flags in (0, 32768):
    ns = bench.prepare(cfg, torch.device("cuda", 0), flags=flags, budgets=[148, 120, 112, 104, 96, 88, 80])
    print(cfg, "flags", flags, "best", min(ns.tune_ms.values()), ns.budget, ns.tune_ms, flush=True)
    del ns
    torch.cuda.empty_cache()
