"""Debug: the MMA issuers' event sequence on pair 0 of cfg2 (CODEC_FLAG_TRACE;
needs a build with CODEC_NVCC_EXTRA=-DCODEC_TC_TRACE, e.g. CODEC_BUILD_TAG=trace,
selected with CODEC_B200_LIB).

    python tools/trace_seq.py [flags] [first_event] [n_events]

Codes: 1 S(ts) wants s_free(ts-2), 2 q_full ok, 3 k_full ok, 4 S issued,
5 PV(tp) wants p_full, 6 p_full ok, 7 v_full ok, 9 PV issued.
"""
import ctypes as C, math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W, _lib
from paper_2505_17694_b200.executor import DecodeStep

extra = int(sys.argv[1]) if len(sys.argv) > 1 else 0
first = int(sys.argv[2]) if len(sys.argv) > 2 else 40
count = int(sys.argv[3]) if len(sys.argv) > 3 else 60
dev = torch.device('cuda')
spec = W.two_level(32768, 512, 256, h_q=32, h_kv=8, d=128, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((256, 32, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
plan = P.plan_device(f, 4, P.load_default_profile(), 8)
step = DecodeStep(f, plan, 32, 'bfloat16', flags=128 | 8 | 32 | 64 | extra, concurrent=False)
for _ in range(3):
    step(q, kp, vp)
torch.cuda.synchronize()
n = 17 * 2 * 64 + 4096
buf = (C.c_longlong * n)()
_lib.check(_lib.lib().codec_debug_trace(buf, n))
a = np.array(buf, dtype=np.int64)[17 * 2 * 64:].reshape(-1, 2)
a = a[a[:, 0] > 0]
a = a[np.argsort(a[:, 0], kind='stable')]  # S and PV issuers log separately
names = {1: 'S want s_free', 2: 'S q ok', 3: 'S k_full ok', 4: 'S issued', 5: 'PV want p_full',
         6: 'PV p_full ok', 7: 'PV v_full ok', 9: 'PV issued'}
t0 = a[0, 0]
prev = a[max(first - 1, 0), 0]
for clk, tag in a[first:first + count]:
    code, tt = tag >> 16, tag & 0xffff
    print(f'{clk - t0:8d} +{clk - prev:6d}  {names.get(int(code), code):16s} {tt}')
    prev = clk
# steady-state per-event mean durations (time from previous event)
d = np.diff(a[:, 0])
codes = a[1:, 1] >> 16
print('mean time spent before each event (events 20..):')
for c in sorted(names):
    m = codes[20:] == c
    if m.any():
        print(f'  {names[c]:16s} {d[20:][m].mean():7.1f}')

# whole-kernel view: big gaps (> 800 clk) and the steady-state S->S period
print('events', len(a), 'span', a[-1, 0] - a[0, 0], 'clk')
gaps = np.nonzero(np.diff(a[:, 0]) > 800)[0]
for i in gaps:
    c, tt = a[i + 1, 1] >> 16, a[i + 1, 1] & 0xffff
    print(f'  gap {a[i + 1, 0] - a[i, 0]:6d} before {names.get(int(c), c)} {tt} (at {a[i + 1, 0] - t0})')
si = a[(a[:, 1] >> 16) == 4, 0]
print('S issued period: median', int(np.median(np.diff(si))), 'mean', int(np.diff(si).mean()), 'n', len(si))

# per-tile chain on CTA rank 0 (softmax stamps: 14 wait S, 2 saw S, 4 freed S,
# 5 row max settled, 12 P buffer free, 3 P released), times relative to S issued
st = np.array(buf, dtype=np.int64)[:17 * 2 * 64].reshape(17, 2, 64)
ev = {}
for clk, tag in a:
    ev[(int(tag >> 16), int(tag & 0xffff))] = clk
print('tile: S_issued->sawS  ->freedS  ->m_set  ->Pbuf_ok  ->relP  ->PV_sees_P  ->PV_issued | S_issued(t)-S_issued(t-1) | relP w0r1 w3r0 w3r1 w1r0 w1r1 w2r0 w2r1')
for t in range(20, 40):
    s_iss = ev.get((4, t))
    if s_iss is None:
        continue
    r = lambda e: st[e, 0, t] - s_iss if st[e, 0, t] > 0 else -1
    pv_p = ev.get((6, t), s_iss) - s_iss
    pv_i = ev.get((9, t), s_iss) - s_iss
    rr = lambda e, k: st[e, k, t] - s_iss if st[e, k, t] > 0 else -1
    print(f'{t:3d}: {r(2):6d} {r(4):8d} {r(5):8d} {r(12):9d} {r(3):7d} {pv_p:10d} {pv_i:11d} | {s_iss - ev.get((4, t - 1), s_iss):6d} |'
          f' {rr(3, 1):6d} {rr(7, 0):6d} {rr(7, 1):6d} {rr(10, 0):6d} {rr(10, 1):6d} {rr(11, 0):6d} {rr(11, 1):6d}')
