"""Debug: clocks the TC epilogue takes per unit (build with
CODEC_NVCC_EXTRA=-DCODEC_TC_EPI_TIMING, select with CODEC_B200_LIB), in the
full step and with the tensor-core kernel alone (no suffix stream).

    python tools/epi_timing.py [config] [budget]
"""
import ctypes as C, math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import _lib, workloads as W
from paper_2505_17694_b200.executor import DecodeStep
config = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 96
dev = torch.device("cuda")
spec = W.make_config(config, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((f.bs, spec.h_q, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
plan = P.plan_device(f, spec.h_q // 8, P.load_default_profile(), 8, 148, budget)
for name, extra in (("full step", 0), ("TC alone", 8 | 32 | 64)):
    step = DecodeStep(f, plan, spec.h_q, "bfloat16", flags=1024 | extra, tc_sm_budget=budget, concurrent=True)
    step(q, kp, vp)
    torch.cuda.synchronize()
    n = 4 * (4096 + 65536)
    buf = (C.c_longlong * n)()
    _lib.check(_lib.lib().codec_debug_ctalog(buf, n))
    a = np.array(buf, dtype=np.int64).reshape(-1, 4)[2048:4096]
    a = a[a[:, 1] > 0]
    units = np.diff(step.blob_host[step.info.off_tc_block_ptr: step.info.off_tc_block_ptr + step.info.n_tc_blocks + 1])
    u = np.repeat(units, 2)[:len(a)]
    print(f"{config} budget {budget} {name}: per epilogue: unit end -> O read {np.median(a[:, 1] / u):.0f} clk, "
          f"O read -> stores done {np.median(a[:, 2] / u):.0f} clk (medians over {len(a)} CTAs)", flush=True)
    if os.environ.get("EPI_SPLIT"):  # library built with -DCODEC_TC_EPI_TIMING -DCODEC_TC_EPI_SPLIT
        print(f"    of which staging writes {np.median(a[:, 0] / u):.0f} clk, global stores {np.median(a[:, 3] / u):.0f} clk",
              flush=True)
