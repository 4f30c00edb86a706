"""Per-kernel SASS opcode summary of the built library (cuobjdump -sass):
the instructions that prove where the math and the data movement run --
UTCHMMA (tcgen05.mma), UTMALDG / UTMAPF (TMA loads / L2 prefetches),
UBLKCP (bulk copies), LDTM / STTM (TMEM loads / stores), HMMA (mma.sync),
LDSM / MOVM (ldmatrix / movmatrix), MUFU (exp2), SYNCS (mbarriers).

    python tools/sass_summary.py [lib.so] > profiles/sass_opcodes.md
"""
import collections
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2505_17694_b200" / "_codec_b200.so"
WATCH = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMAPF", "UBLKCP", "UBLKPF", "LDTM", "STTM", "HMMA", "LDSM", "MOVM",
         "MUFU", "FFMA2", "SYNCS", "LDG", "STG", "LDS", "STS"]
KERNELS = {"tc_pac_kernel": "K2 tcgen05 shared-node", "mma_pac_kernel": "K3 mma.sync suffix",
           "mma_multi_kernel": "K3m mma.sync multi-request", "tct_kernel": "K2t transposed tcgen05 (lightly shared)",
           "merge128_kernel": "K4 LSE merge (d=128)",
           "gemv_pac_kernel": "K3' CUDA-core GEMV", "gen_decode_kernel": "generic"}

sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
counts, variants, cur = {}, {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        variants[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Z0-9_]+)*)", line)
    if m and cur:
        op, mods = m.group(1), m.group(2)
        counts[cur][op] += 1
        if op in ("UTCHMMA", "UTMALDG", "UTMAPF", "MUFU", "HMMA", "UTCBAR"):
            variants[cur][op + mods] += 1

rows = {}
for fn, c in counts.items():
    for key, label in KERNELS.items():
        if key in fn:
            if key in ("gemv_pac_kernel", "gen_decode_kernel"):
                if "bfloat16" not in fn or ("Li128ELi4" not in fn and key == "gemv_pac_kernel"):
                    continue  # one representative instantiation
            name = label
            rows[name] = {k: v for k, v in sorted(c.items()) if k in WATCH}
            rows[name]["variants"] = dict(sorted(variants[fn].items()))
print(f"# SASS opcode summary of `{LIB.name}` (cuobjdump -sass, sm_100a)\n")
print("Static instruction counts per kernel (not dynamic counts): which units the code uses.\n")
print("| kernel | " + " | ".join(WATCH) + " |")
print("|---" * (len(WATCH) + 1) + "|")
for name, c in rows.items():
    print(f"| {name} | " + " | ".join(str(c.get(w, 0)) for w in WATCH) + " |")
print("\nVariants (opcode with modifiers):\n")
for name, c in rows.items():
    det = c["variants"]
    if det:
        print(f"* {name}: " + ", ".join(f"`{k}` x{v}" for k, v in det.items()))
(ROOT / "profiles" / "sass_opcodes.json").write_text(json.dumps(rows, indent=1) + "\n")
