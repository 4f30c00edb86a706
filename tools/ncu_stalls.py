"""Per-instruction warp-stall summary of an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass > x.csv).

    python tools/ncu_stalls.py x.csv [min_samples] [first_addr_idx] [last_addr_idx]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 10 ** 9
body = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
agg = {s: 0 for s in stalls}
for k, r in enumerate(body):
    n = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    for s in stalls:
        agg[s] += int(r[idx[s]] or 0)
    if n >= thr and lo <= k <= hi:
        top = sorted(((int(r[idx[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
        print(f"{k:5d} {n:6d} {100*n/tot:5.2f}% {r[1].strip()[:60]:60s} " + " ".join(f"{s}:{v}" for v, s in top if v))
print("total samples", tot)
print(sorted(((v, s) for s, v in agg.items()), reverse=True)[:10])
