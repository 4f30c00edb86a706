"""A/B of library builds in SUSTAINED conditions (the bench's regime: the
power cap engaged): each variant in its own subprocess runs the config's
prepared step (fixed SM budget) from a CUDA graph for `seconds`, median of
20-step windows, nvidia-smi clock / power sampled; rounds alternate.

    python tools/ab_sustained.py config budget seconds rounds tag1 tag2 ...  (tag '-' = default library)
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, statistics, time, torch
sys.path.insert(0, %r)
import bench
ns = bench.prepare(%r, torch.device("cuda", 0), budgets=[%d])
g = ns.step.capture(ns.q_dev, ns.kp, ns.vp, ns.out)
for _ in range(10): g()
torch.cuda.synchronize()
clk = bench.ClockSampler(0)
wins, t0 = [], time.perf_counter()
while time.perf_counter() - t0 < %f:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): g()
    e1.record(); torch.cuda.synchronize()
    wins.append(e0.elapsed_time(e1) / 20 * 1e3)
c = clk.stop()
print(json.dumps({"us": statistics.median(wins), "sm": c["sm_mhz"], "w": c["power_w_median"]}))
'''
config, budget, secs, rounds, tags = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), sys.argv[5:]
res = {t: [] for t in tags}
for r in range(rounds):
    for tag in tags:
        env = dict(os.environ)
        if tag != '-':
            env["CODEC_B200_LIB"] = os.path.join(ROOT, "paper_2505_17694_b200", f"_codec_b200_{tag}.so")
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, config, budget, secs)], env=env,
                             capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        res[tag].append(json.loads(line[-1]) if line else {"err": out.stderr[-300:]})
        print(tag, res[tag][-1], flush=True)
for tag in tags:
    ok = sorted(x["us"] for x in res[tag] if "us" in x)
    print(f"{tag:10s} median {ok[len(ok) // 2] if ok else None}")
