"""Summarise ncu --set full captures of the decode step's kernels into
profiles/ncu_summary.json (read by bench.py for roofline.traffic) and a
markdown table.

    python tools/ncu_summary.py cfg2 gpurun_out/prof_tc.ncu-rep gpurun_out/prof_mma.ncu-rep ...
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
        "nsecond": 1e-3, "msecond": 1e3, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1,
        "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def kernel_key(name):
    if "tc_pac" in name:
        return "tc"
    if "mma_multi" in name:
        return "multi"
    if "tct_kernel" in name:
        return "tct"
    if "mma_pac" in name or "gemv_pac" in name:
        return "gemv"
    if "merge" in name:
        return "merge"
    return None


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, out = rows[0], rows[1], {}
    for r in rows[2:]:
        name = r[head.index("Kernel Name")]
        key = kernel_key(name)
        if not key:
            continue
        rec = {"kernel": name.split("(")[0]}
        for col, short in WANT.items():
            if col in head:
                i = head.index(col)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                rec[short] = v * UNIT.get(units[i], 1)
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        out[key] = rec
    return out


def main():
    """ncu_summary.py CONFIG TC_SM_BUDGET REP..."""
    cfg, budget, reps = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
    path = ROOT / "profiles" / "ncu_summary.json"
    allj = json.loads(path.read_text()) if path.exists() else {}
    cur = {}
    for rep in reps:
        cur.update(summarise(rep))
    kernels = [k for k in cur if isinstance(cur[k], dict)]
    cur["tc_sm_budget"] = budget
    cur["step_dram_bytes"] = sum(cur[k].get("dram_bytes", 0) for k in kernels)
    cur["capture"] = ("ncu --set full --clock-control none, one decode step of bench.prepare(cfg) at the "
                      "benchmarked tensor-core SM budget; kernels serialised by the profiler")
    allj[cfg] = cur
    path.write_text(json.dumps(allj, indent=1) + "\n")
    lines = [f"# ncu --set full summary ({cfg})", "",
             "| kernel | duration us | DRAM bytes | DRAM % | tensor % (active) | XU % | FMA % | regs | grid |",
             "|---|---|---|---|---|---|---|---|---|"]
    for k, r in cur.items():
        if not isinstance(r, dict):
            continue
        lines.append(f"| {k} ({r.get('kernel')}) | {r.get('duration', 0):.1f} | {r.get('dram_bytes', 0):.4g} | "
                     f"{r.get('dram_pct', 0):.1f} | {r.get('tensor_pct_active', 0):.1f} | {r.get('xu_pct', 0):.1f} | "
                     f"{r.get('fma_pct', 0):.1f} | {r.get('regs', 0):.0f} | {r.get('grid', 0):.0f} |")
    lines += ["", f"tensor-core SM budget {budget}; step DRAM bytes {cur['step_dram_bytes']:.4g} "
              f"(kernels serialised by ncu, cold caches)"]
    (ROOT / "profiles" / f"ncu_summary_{cfg}.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
