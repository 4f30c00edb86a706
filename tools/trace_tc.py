"""Debug: print the tensor-core kernel timeline of CTA (0,0) on cfg2."""
import ctypes as C, math, sys
import numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W, _lib
from paper_2505_17694_b200.executor import DecodeStep
dev = torch.device('cuda')
spec = W.two_level(32768, 512, 256, h_q=32, h_kv=8, d=128, tensors=False)
f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
T = f.total_tokens
kp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
vp = (torch.randn((8, T, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
q = (torch.randn((256, 32, 128), device=dev) / math.sqrt(128)).to(torch.bfloat16)
plan = P.plan_device(f, 4, P.load_default_profile(), 8)
step = DecodeStep(f, plan, 32, 'bfloat16', flags=128 | 8 | 32 | 64 | int(sys.argv[1] if len(sys.argv) > 1 else 0), concurrent=False)
for _ in range(3): step(q, kp, vp)
torch.cuda.synchronize()
buf = (C.c_longlong * 2176)()
_lib.check(_lib.lib().codec_debug_trace(buf, 2176))
a = np.array(buf, dtype=np.int64).reshape(17, 2, 64)
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, -1)
# a[event, cta rank, tile]: 0 MMA saw P(t), 1 MMA issued PV(t), 2 softmax saw S(t),
# 3 softmax released P(t), 4 softmax freed S(t), 5 row max settled, 6 MMA issued S(t+2)
n = 40
print('period (sm_saw_S rank0):', np.diff(a[2, 0, :n]))
print('softmax X (saw S -> rel P) r0:', a[3, 0, :n] - a[2, 0, :n])
print('  saw S -> S freed:', a[4, 0, :n] - a[2, 0, :n])
print('  S freed -> m settled:', a[5, 0, :n] - a[4, 0, :n])
print('  m settled -> rel P:', a[3, 0, :n] - a[5, 0, :n])
print('rel P (max of ranks) -> MMA saw P:', a[0, 0, :n] - np.maximum(a[3, 0, :n], a[3, 1, :n]))
print('MMA PV issue:', a[1, 0, :n] - a[0, 0, :n])
print('S freed -> MMA issued S(t+2):', a[6, 0, :n] - np.maximum(a[4, 0, :n], a[4, 1, :n]))
print('MMA issued S(t) -> softmax saw S(t):', a[2, 0, 2:n] - a[6, 0, :n - 2])
print('TC busy estimate per tile (1024/period):', np.round(1024 / np.maximum(np.diff(a[2, 0, :n]), 1), 2))
rel = np.stack([a[3, r, :n] for r in (0, 1)] + [a[7, r, :n] for r in (0, 1)])
print('last warp rel P -> MMA saw P:', a[0, 0, :n] - rel.max(0))
# ev 8/9 indexed by the S tile ts: first seen s_free(ts-2) / k_full(ts) ready
print('S(ts): s_free(ts-2) seen - k_full(ts) seen (neg: K later):', a[8, 0, 2:n] - a[9, 0, 2:n])
print('S(ts): issue - max(seen):', a[6, 0, :n - 2] - np.maximum(a[8, 0, 2:n], a[9, 0, 2:n]))
print('S(ts): s_free(ts-2) released (last softmax) -> seen by MMA:', a[8, 0, 2:n] - np.maximum(a[4, 0, :n - 2], a[4, 1, :n - 2]))
print('PV(t): p_full seen (MMA waited) - last rel:', a[10, 0, :n] - rel.max(0))
print('PV(t): issue start - p_full seen:', a[0, 0, :n] - a[10, 0, :n])
print('S(ts): s_free seen - last s_free release:', a[8, 0, 2:n] - np.maximum(a[4, 0, :n - 2], a[4, 1, :n - 2]))
print('S(ts) issue duration:', a[6, 0, :n - 2] - a[13, 0, 2:n])
print('PV issue(t-2) -> softmax P-buffer wait done (t):', a[12, 0, 2:n] - a[1, 0, :n - 2])
print('softmax m settled -> P-buffer wait done:', a[12, 0, :n] - a[5, 0, :n])

np.set_printoptions(linewidth=250)
print('ready(t) -> saw S(t):', (a[2, 0, :n] - a[14, 0, :n]).tolist())
print('rel P(t-2) [same group] -> ready(t):', (a[14, 0, 2:n] - a[3, 0, :n - 2]).tolist())
ep = np.nonzero(a[15, 0] > 0)[0]
for t in ep:
    print(f'unit ends at tile {t}: epi start {a[16,0,t]-a[3,0,t]} after rel P(last); epi took {a[15,0,t]-a[16,0,t]}; '
          f'staging+copy {a[9,0,t]-a[15,0,t]}; next ready {a[14,0,t+2]-a[9,0,t] if t+2<64 else None}; '
          f'next PV issue (MMA saw P) {a[0,0,t+1]-a[15,0,t] if t+1<64 else None}')
