import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, io
import paper_2505_17694_b200 as P
from paper_2505_17694_b200.executor import DecodeStep
import test_gpu_parity as T
from conftest import golden_table_text
table = P.load_profile(io.StringIO(golden_table_text("a100_d128.csv")))
spec = T.d128_forest(12, with_masks=True)
f, q = T.build(spec, "bfloat16")
plan = P.plan_device(f, 4, table, 8, 148)
kp, vp = f.device_pool("bfloat16"); qd = q.queries.cuda()
for name, fl in (("fused", 0), ("merge_kernel", 4096), ("simt", 2048)):
    st = DecodeStep(f, plan, 32, "bfloat16", flags=fl, concurrent=False)
    o = T.np_(st(qd, kp, vp))
    bad = np.argwhere(~np.isfinite(o))
    print(name, "n_merge", st.info.n_merge, "fused", st.info.n_merge_fused, "slots", st.info.n_slots, "nonfinite", len(bad), sorted(set(map(tuple, bad[:, :2].tolist())))[:10])
print("paths", spec.paths)
