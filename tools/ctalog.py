"""Debug: per-CTA timeline (SM, start, end) of one cfg2 decode step with the
TC and GEMV kernels on concurrent streams -- shows whether GEMV CTAs
co-reside with the persistent TC CTAs.

    python tools/ctalog.py [budget] [flags]
"""
import ctypes as C
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17694_b200 as P  # noqa: E402
from paper_2505_17694_b200 import _lib, workloads as W  # noqa: E402
from paper_2505_17694_b200.executor import DecodeStep  # noqa: E402

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 148
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
config = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
dev = torch.device("cuda")
spec = W.make_config(config, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((f.bs, spec.h_q, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
plan = P.plan_device(f, spec.h_q // 8, P.load_default_profile(), 8, 148, budget)
step = DecodeStep(f, plan, spec.h_q, "bfloat16", flags=1024 | extra, tc_sm_budget=budget, concurrent=True)
for _ in range(3):
    step(q, kp, vp)
torch.cuda.synchronize()
n = 4 * (4096 + 65536)
buf = (C.c_longlong * n)()
_lib.check(_lib.lib().codec_debug_ctalog(buf, n))
a = np.array(buf, dtype=np.int64).reshape(-1, 4)
tc = a[:4096][a[:4096, 2] > 0]
gv = a[4096:][a[4096:, 2] > 0]
t0 = min(tc[:, 1].min() if len(tc) else 1 << 62, gv[:, 1].min() if len(gv) else 1 << 62)
us = lambda x: (x - t0) / 1e3
print(f"TC CTAs {len(tc)}: start {us(tc[:,1]).min():.1f}-{us(tc[:,1]).max():.1f} us, "
      f"end {us(tc[:,2]).min():.1f}-{us(tc[:,2]).max():.1f} us, SMs {len(set(tc[:,0]))}")
if len(gv):
    print(f"GEMV CTAs {len(gv)}: start {us(gv[:,1]).min():.1f}-{us(gv[:,1]).max():.1f} us, "
          f"end max {us(gv[:,2]).max():.1f} us, SMs {len(set(gv[:,0]))}, "
          f"dur median {np.median(gv[:,2]-gv[:,1])/1e3:.2f} us")
    tc_end = tc[:, 2].max() if len(tc) else t0
    during = gv[gv[:, 1] < tc_end]
    print(f"GEMV CTAs started while TC ran: {len(during)} on {len(set(during[:,0]))} SMs; "
          f"SMs shared with a TC CTA: {len(set(during[:,0]) & set(tc[:,0]))}")
    # GEMV concurrency over time
    for t in np.linspace(0, us(max(gv[:, 2].max(), tc[:, 2].max() if len(tc) else 0)), int(os.environ.get("CTALOG_POINTS", "12"))):
        tt = t0 + t * 1e3
        live = ((gv[:, 1] <= tt) & (gv[:, 2] > tt)).sum()
        tlive = ((tc[:, 1] <= tt) & (tc[:, 2] > tt)).sum() if len(tc) else 0
        print(f"  t={t:7.1f} us  TC live {tlive:4d}  GEMV live {live:4d}")

# fused kernel: per CTA {TC work drained, suffix warp 0 done, suffix warp 1 done, start}
fz = a[2048:4096]
fz = fz[fz[:, 3] > 0]
if len(fz):
    print(f"fused: TC done {us(fz[:,0]).min():.1f}-{np.median(us(fz[:,0])):.1f}-{us(fz[:,0]).max():.1f} us (min-med-max); "
          f"suffix w0 done {us(fz[:,1]).min():.1f}-{np.median(us(fz[:,1])):.1f}-{us(fz[:,1]).max():.1f}; "
          f"w1 {us(fz[:,2]).min():.1f}-{np.median(us(fz[:,2])):.1f}-{us(fz[:,2]).max():.1f}")

# TC units per pair (table)
info = step.info
blob = step.blob_host
bp = blob[info.off_tc_block_ptr: info.off_tc_block_ptr + info.n_tc_blocks + 1]
units = np.diff(bp)
recs = blob[info.off_tc: info.off_tc + 8 * info.n_tc_groups].reshape(-1, 8)
tiles = [int(sum((recs[j, 4] + 127) // 128 for j in range(bp[b], bp[b + 1]))) for b in range(info.n_tc_blocks)]
print("TC pairs", info.n_tc_blocks, "units/pair", np.bincount(units).tolist(), "tiles/pair min/med/max",
      min(tiles), int(np.median(tiles)), max(tiles))

# per-pair duration against its tiles / units (TC entries are indexed by blockIdx.x)
tcl = a[:4096]
dur = {}
for x in range(2 * info.n_tc_blocks):
    if tcl[x, 2] > 0:
        dur.setdefault(x >> 1, []).append((tcl[x, 2] - tcl[x, 1]) / 1e3)
rows = []
for b in range(info.n_tc_blocks):
    if b in dur:
        rows.append((max(dur[b]), tiles[b], int(units[b]), int(tcl[2 * b, 0]), b))
if os.environ.get("CTALOG_ALL"):
    for r in sorted(rows, key=lambda x: x[4]):
        print("  pair %d: %.1f us, %d tiles, %d units" % (r[4], r[0], r[1], r[2]))
rows = [r[:4] for r in rows]
rows.sort()
print("pair duration us / tiles / units / smid (fastest 8, slowest 8):")
for r in rows[:8] + rows[-8:]:
    print("  %.1f %d %d %d" % r)
for u in sorted(set(r[2] for r in rows)):
    d = [r[0] / r[1] for r in rows if r[2] == u]
    print(f"units {u}: n={len(d)} us/tile mean {np.mean(d):.3f} min {np.min(d):.3f} max {np.max(d):.3f}")
