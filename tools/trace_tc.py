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
plan = P.divide_and_schedule(P.device_tasks(f, 4), P.load_default_profile(), 37)
step = DecodeStep(f, plan, 32, 'bfloat16', flags=128 | 8 | 32 | 64, concurrent=False)
for _ in range(3): step(q, kp, vp)
torch.cuda.synchronize()
buf = (C.c_longlong * 640)()
_lib.check(_lib.lib().codec_debug_trace(buf, 640))
a = np.array(buf, dtype=np.int64).reshape(5, 2, 64)
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, -1)
names = ['mma_saw_P', 'mma_issued', 'sm_saw_S', 'sm_rel_P', 'sm_xch_done']
for t in range(0, 24):
    print(t, ' | '.join(f"{names[e]}[{i}]={a[e,i,t]:7d}" for e in (2, 4, 3, 0, 1) for i in (0, 1)))
d = np.diff(a[2, 0, :40])
print('period (sm_saw_S wg0):', d)
print('softmax X wg0:', (a[3, 0, :40] - a[2, 0, :40]))
print('S latency (P rel -> next S seen) wg0:', (a[2, 0, 1:40] - a[3, 0, :39]))
