"""Decode-attention benchmark (BASELINE.json metric) for the B200 path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--no-cpu-baseline]

Workload (config[1] of BASELINE.json): Llama-3-8B shape, 32 q / 8 kv
heads, d=128, bf16 KV; 256 requests share a 32K-token system prompt, each
with a private 512-token suffix. Synthetic N(0,1)/sqrt(d) data generated
on the device (K/V pool 671 MB > 126 MB L2, so every step streams from
HBM). A "step" = one decode-attention call over all 256 requests.

value = effective unique-KV GB/s over the whole job (all ranks); with N
GPUs the kv heads are split N ways (tensor-parallel head split) and the
per-rank outputs are all-gathered over NCCL inside the timed step.
`e2e` times the same step through the public API with queries copied from
pinned host memory and the output read back every step.

--impl reference times the reference's CPU algorithm (the oracle port
under oracle/, numpy, all host threads) on the same whole workload per
step (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode-attn µs/step & effective KV GB/s (unique bytes) vs HBM roofline, 1-8 GPU"
CONFIGS = {  # BASELINE.json "configs"; structures from workloads.make_config
    "cfg1": dict(h_q=8, h_kv=8, d=128,
                 label="cfg1: tiny 2-level tree, 16 requests sharing a 1K prefix + 64-token suffixes, 8 heads x d128"),
    "cfg2": dict(h_q=32, h_kv=8, d=128,
                 label="cfg2: Llama-3-8B shape (32 q / 8 kv heads, d128, bf16 KV), 256 requests sharing a "
                       "32K system prompt + 512-token suffixes"),
    "cfg3": dict(h_q=32, h_kv=8, d=128,
                 label="cfg3: tree-of-thought / beam tree, depth 4, branching 4, 8K root, irregular node lengths "
                       "(64 requests), Llama-3-8B heads"),
    "cfg4": dict(h_q=32, h_kv=8, d=128, cpu_trees=range(8),
                 label="cfg4: imbalanced forest, 64 trees with 512..128K shared prefixes and 1..512 requests per "
                       "tree + 512-token suffixes (4680 requests), Llama-3-8B heads"),
    "cfg5": dict(h_q=64, h_kv=8, d=128,
                 label="cfg5: Llama-3-70B shape (64 q / 8 kv heads, d128, bf16 KV), 1024 requests sharing a "
                       "64K prefix + 512-token suffixes"),
}


def structure(name, **kw):
    from paper_2505_17694_b200 import workloads as W
    return W.make_config(name, **kw)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region
    (written by nvidia-smi itself via -f, so nothing is lost on stop)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.proc = None
        self.path = Path("/tmp") / f"bench_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50", "-f", str(self.path)],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        if self.path.exists():
            for line in self.path.read_text().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[0]) for r in rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU side
def cpu_reference_sample(cfg, workers=None, seed=0):
    """The whole workload (every kv head, all requests) through the oracle
    port of the reference executor (numpy, host threads): returns (seconds,
    unique KV bytes at bf16 width, description). Inputs are generated
    once per process (fp32, the reference's CPU dtype) and not timed."""
    from oracle import attention as OA
    from oracle import plan as OP
    from oracle import index as OI
    from paper_2505_17694_b200 import workloads as W

    workers = workers or os.cpu_count()
    key = (cfg["label"], seed)
    if key not in _CPU_CACHE:
        over = {"only_trees": cfg["cpu_trees"]} if "cpu_trees" in cfg else {}
        spec = structure(cfg["name"], dtype=np.float32, **over)
        z = np.zeros((0, cfg["h_kv"], cfg["d"]), np.float32)
        fd = OA.ForestData(spec.parent, [z] + spec.keys[1:], [z] + spec.values[1:], spec.paths)
        # the CPU's own best split: shared nodes sliced once per host thread so
        # every thread has work (the reference's thread pool, executor.py:194)
        qs = OI.query_sets(spec.paths, spec.n_nodes)
        subs = []
        for node, nq, n in OP.node_tasks(qs, spec.length):
            for a, b in OP.slices(n, workers if nq > 1 else 1):
                subs.append((node, a, b))
        _CPU_CACHE[key] = (spec, fd, subs)
    spec, fd, subs = _CPU_CACHE[key]
    t0 = time.perf_counter()
    OA.execute(fd, spec.queries, subs, workers=workers)
    dt = time.perf_counter() - t0
    kv_bytes = sum(spec.length[1:]) * cfg["h_kv"] * cfg["d"] * 2 * 2
    what = (f"trees {list(cfg['cpu_trees'])} of the workload ({spec.bs} requests)" if "cpu_trees" in cfg
            else f"the whole workload ({spec.bs} requests)")
    desc = (f"{what}: all {cfg['h_kv']} kv heads ({cfg['h_q']} q heads), {sum(spec.length[1:])} KV tokens; "
            f"fp32 numpy oracle port of prefixdec.execute, {workers} threads, plan of {len(subs)} subtasks")
    return dt, kv_bytes, desc


_CPU_CACHE = {}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    workers = os.cpu_count()
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, workers=workers)
    times = []
    for _ in range(args.steps):
        dt, kv_bytes, desc = cpu_reference_sample(cfg, workers=workers)
        times.append(dt)
    t = statistics.mean(times)
    value = kv_bytes / t / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["label"], "sample": desc},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": workers, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU side
KERNEL_EVENTS = 16384  # CODEC_FLAG_KERNEL_EVENTS (include/codec_b200.h)


def kernel_times():
    """[calls, 3] ms of (TC, suffix, merge) kernels of the calls recorded
    under CODEC_FLAG_KERNEL_EVENTS since the last read."""
    import ctypes as C
    from paper_2505_17694_b200 import _lib
    buf = (C.c_float * (3 * 512))()
    n = C.c_int32()
    _lib.check(_lib.lib().codec_kernel_times(buf, 512, C.byref(n)))
    return np.array(buf[:3 * n.value], dtype=np.float64).reshape(-1, 3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--blocks", type=int, default=0, help="planner m (0: SMs // local kv heads)")
    ap.add_argument("--quick", action="store_true", help="profiling run: no e2e / clocks / cpu baseline")
    ap.add_argument("--serial", action="store_true", help="one stream: TC, GEMV and merge back to back")
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of a CUDA graph replay")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], name=args.config)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2505_17694_b200 as P
    from paper_2505_17694_b200 import workloads as W
    from paper_2505_17694_b200.executor import DecodeStep

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    h_kv, h_q, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
    assert h_kv % world == 0, "kv heads must split evenly across ranks"
    h_local = h_kv // world
    h0 = rank * h_local
    g = h_q // h_kv

    # structure + device-resident synthetic KV pool (heads [h0, h0 + h_local))
    spec = structure(args.config, tensors=False)
    forest = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, h_kv, d)
    bs = spec.bs
    T = forest.total_tokens
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + h0)
    sc = 1.0 / math.sqrt(d)
    kp = (torch.randn((h_local, T, d), generator=gen, device=dev, dtype=torch.float32) * sc).to(torch.bfloat16)
    vp = (torch.randn((h_local, T, d), generator=gen, device=dev, dtype=torch.float32) * sc).to(torch.bfloat16)
    hq_local = h_local * g
    q_host = (torch.randn((bs, hq_local, d), generator=torch.Generator().manual_seed(99 + rank)) * sc
              ).to(torch.bfloat16).pin_memory()
    q_dev = q_host.to(dev)

    # plan: shared-node row chunks divided + LPT-scheduled onto the persistent
    # tensor-core CTAs (reference planner algorithm, B200 profile), unshared
    # suffixes on the concurrent GEMV kernel; the SM split between the two is
    # tuned once per plan (cuDNN-benchmark style), untimed
    table = P.load_default_profile()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out = torch.empty((bs, hq_local, d), dtype=torch.float32, device=dev)

    def make(budget):
        t0 = time.perf_counter()
        if args.blocks:
            pl = P.divide_and_schedule(P.device_tasks(forest, g), table, args.blocks)
        else:
            pl = P.plan_device(forest, g, table, h_local, sms, budget)
        ms_plan = (time.perf_counter() - t0) * 1e3
        st = DecodeStep(forest, pl, h_q, "bfloat16", head_begin=h0, head_end=h0 + h_local, device=dev,
                        flags=args.flags, tc_sm_budget=budget, concurrent=not args.serial)
        return pl, st, ms_plan

    # TC SM budget: the SMs the TC grid leaves free run the suffix kernel
    # from the start (programmatic dependent launch); tuned once per plan
    budgets = [sms] if (args.serial or args.quick) else [sms] + list(range(136, 63, -8))
    tune_ms = {}
    best = None

    def refine():
        # a finer pass (+-4 SMs) around the coarse optimum
        if len(budgets) < 2 or best is None:
            return []
        b0 = best[1]
        return [b for b in (b0 - 4, b0 + 4) if 16 <= b < sms and b not in tune_ms]

    queue = list(budgets)
    while queue:
        b = queue.pop(0)
        pl, st, ms_plan = make(b)
        for _ in range(3):
            st(q_dev, kp, vp, out=out)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            st(q_dev, kp, vp, out=out)
        e1.record()
        torch.cuda.synchronize(dev)
        t_b = e0.elapsed_time(e1) / 5
        if world > 1:
            tt = torch.tensor([t_b], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_b = float(tt.item())
        tune_ms[b] = round(t_b, 4)
        if best is None or t_b < best[0]:
            best = (t_b, b, pl, st, ms_plan)
        if not queue and not getattr(refine, "done", False):
            refine.done = True
            queue = refine()
    _, budget, plan, step, plan_ms = best
    m = args.blocks or max(1, budget // h_local)
    # a twin step that records CUDA events around each of its kernels on the
    # launching stream (CODEC_FLAG_KERNEL_EVENTS), timed in its own window
    # right after the main one: the events sit between the kernels and
    # would stop the suffix kernel's programmatic early launch in `value`
    step_ev = DecodeStep(forest, plan, h_q, "bfloat16", head_begin=h0, head_end=h0 + h_local, device=dev,
                         flags=args.flags | KERNEL_EVENTS, tc_sm_budget=budget, concurrent=not args.serial)
    gathered = torch.empty((world, bs, hq_local, d), dtype=torch.float32, device=dev) if world > 1 else None

    # the timed step replays a CUDA graph of the decode step (its three
    # launches recorded once; no per-step host work)
    replay = step.capture(q_dev, kp, vp, out) if not args.no_graph else None

    def one_step(qd):
        if replay is not None and qd is q_dev:
            replay()
        else:
            step(qd, kp, vp, out=out)
        if world > 1:
            dist.all_gather_into_tensor(gathered, out)
        return out

    work = P.device_work(forest, h_q, element_size=2, head_fraction=h_local / h_kv)
    stream = torch.cuda.current_stream(dev)

    def timed(n, fn, min_seconds=0.0):
        """ms per call over n calls between barrier+sync on both sides, CUDA
        events on the launching stream, max over ranks. With min_seconds,
        the n-call window is repeated until that much wall time passed (so
        the clock sampler sees the load) and the median window is used."""
        windows = []
        t_start = time.perf_counter()
        while True:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / n
            if world > 1:
                t = torch.tensor([ms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            windows.append(ms)
            if time.perf_counter() - t_start >= min_seconds or len(windows) >= 500:
                break
        return statistics.median(windows), len(windows)

    for _ in range(max(args.warmup, 3)):
        one_step(q_dev)
    torch.cuda.synchronize(dev)
    clocks = None if args.quick else ClockSampler(local_rank)
    ms, windows = timed(args.steps, lambda: one_step(q_dev), min_seconds=0 if args.quick else 2.0)
    clock_rec = clocks.stop() if clocks else None

    # per-kernel device time: events around each kernel on its stream, over
    # a timed window of the twin step (up to 512 calls)
    for _ in range(3):
        step_ev(q_dev, kp, vp, out=out)
    torch.cuda.synchronize(dev)
    kernel_times()  # drop the warm-up calls' events
    ms_ev = timed(args.steps, lambda: step_ev(q_dev, kp, vp, out=out))[0]
    info = step.info
    kt = kernel_times()
    phases = {}
    if len(kt):
        for j, (name, present) in enumerate((("tc", info.n_tc_groups), ("gemv", info.n_gemv_groups),
                                             ("merge", info.n_merge))):
            if present:
                phases[name] = float(np.mean(kt[:, j]))

    hbm, tf_burst, tf_sus, peak_kind = peaks()
    total_bytes = work["unique_kv_bytes"] * world
    value = total_bytes / (ms * 1e-3) / 1e9
    # bytes / flops attributed to each kernel
    tc_rows = sum(n.len for n in forest.nodes[1:] if len(n.query_set) * g >= 16)
    kv_tc = tc_rows * h_local * d * 2 * 2
    kernels = {}
    if "tc" in phases:
        fl = sum(n.len * len(n.query_set) for n in forest.nodes[1:] if len(n.query_set) * g >= 16) * hq_local * 4 * d
        # timed inside the long-running step: the sustained cuBLAS figure
        kernels["tc"] = {"bound": "tensor", "achieved": fl / (phases["tc"] * 1e-3) / 1e12, "peak": tf_sus,
                         "peak_figure": "bf16_tflops_sustained", "unit": "TFLOP/s", "ms": phases["tc"],
                         "algorithmic_flops": fl, "kv_bytes": kv_tc}
        kernels["tc"]["frac"] = kernels["tc"]["achieved"] / tf_sus
        kernels["tc"]["frac_of_burst"] = kernels["tc"]["achieved"] / tf_burst
        # the TC grid holds tc_sm_budget SMs; the others stream the suffixes
        kernels["tc"]["sms"] = int(min(budget, sms))
        kernels["tc"]["frac_per_sm"] = kernels["tc"]["frac"] * sms / max(1, min(budget, sms))
    if "gemv" in phases:
        kb = work["unique_kv_bytes"] - kv_tc
        kernels["gemv"] = {"bound": "hbm", "achieved": kb / (phases["gemv"] * 1e-3) / 1e9, "peak": hbm,
                           "unit": "GB/s", "ms": phases["gemv"], "algorithmic_bytes": kb}
        kernels["gemv"]["frac"] = kernels["gemv"]["achieved"] / hbm
    if "merge" in phases:
        kernels["merge"] = {"ms": phases["merge"]}
    # DRAM traffic per launch from the committed ncu --set full capture of
    # this workload (profiles/ncu_summary.json, tools/ncu_summary.py)
    ncu = {}
    ncu_path = ROOT / "profiles" / "ncu_summary.json"
    if ncu_path.exists():
        try:
            ncu = json.loads(ncu_path.read_text()).get(args.config, {})
        except Exception:
            ncu = {}
    for name in kernels:
        if name in ncu and "dram_bytes" in ncu[name]:
            kernels[name]["traffic"] = ncu[name]["dram_bytes"]
    dominant = max((k for k in kernels if "bound" in kernels[k]), key=lambda k: kernels[k]["ms"], default=None)
    roof = None
    if dominant:
        k = kernels[dominant]
        roof = {"bound": k["bound"], "achieved": k["achieved"], "peak": k["peak"], "unit": k["unit"],
                "frac": k["frac"], "traffic": k.get("traffic"), "kernel": dominant, "peak_kind": peak_kind,
                "sms": k.get("sms"), "frac_per_sm": k.get("frac_per_sm")}

    e2e = None
    if not args.quick:
        # Serving-style pipeline through the public API: every step uploads
        # its queries from pinned host memory and reads its output back;
        # step k's copies run on their own streams, overlapping the compute
        # of steps k - 1 / k + 1 (double-buffered device q / out).
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        qbuf = [torch.empty_like(q_dev) for _ in range(2)]
        obuf = [torch.empty_like(out) for _ in range(2)]
        ohost = [torch.empty((bs, hq_local, d), dtype=torch.float32).pin_memory() for _ in range(2)]
        ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("h2d", "comp", "d2h")}
        gath2 = [torch.empty_like(gathered) for _ in range(2)] if world > 1 else None
        st8 = {"k": 0}

        def e2e_step():
            k = st8["k"]
            sl = k & 1
            st8["k"] += 1
            with torch.cuda.stream(s_h2d):
                if k >= 2:
                    s_h2d.wait_event(ev["comp"][sl])
                qbuf[sl].copy_(q_host, non_blocking=True)
                ev["h2d"][sl].record(s_h2d)
            stream.wait_event(ev["h2d"][sl])
            if k >= 2:
                stream.wait_event(ev["d2h"][sl])
            step(qbuf[sl], kp, vp, out=obuf[sl], stream=stream)
            res = obuf[sl]
            if world > 1:
                dist.all_gather_into_tensor(gath2[sl], obuf[sl])
            ev["comp"][sl].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev["comp"][sl])
                ohost[sl].copy_(res, non_blocking=True)
                ev["d2h"][sl].record(s_d2h)

        def e2e_window(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            e0.record(stream)
            s_h2d.wait_event(e0)
            st8["k"] = 0
            for _ in range(n):
                e2e_step()
            stream.wait_stream(s_d2h)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / n
            if world > 1:
                t = torch.tensor([ms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            return ms

        e2e_window(3)
        e2e_ms = statistics.median(e2e_window(args.steps) for _ in range(5))
        e2e = {"value": total_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": q_host.numel() * q_host.element_size(),
               "d2h_bytes_per_step": ohost[0].numel() * ohost[0].element_size(),
               "pipeline": "per step: pinned H2D of q, decode step, D2H of out; copies on their own streams "
                           "overlap the neighbouring steps' compute (double-buffered)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        dt, kvb, desc = cpu_reference_sample(cfg)
        cpu = {"value": kvb / dt / 1e9, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port",
               "sample": desc, "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "timed_windows": windows, "us_per_step": ms * 1e3, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: N(0,1)/sqrt(d) K/V/Q generated on device (seeded), no checkpoint",
            "config": {"workload": cfg["label"], "bs": bs, "h_q": h_q, "h_kv": h_kv, "d": d,
                       "kv_tokens": int(sum(spec.length[1:])), "nodes": int(spec.n_nodes - 1),
                       "parallelism": f"kv-head split x{world}" + (" + NCCL all-gather" if world > 1 else ""),
                       "l2": "inputs larger than L2 (KV pool %.0f MB > 126 MB)" % (2 * kp.numel() * 2 / 1e6),
                       "planner": {"m_tc": m, "subtasks": len(plan.subtasks), "makespan_ms": plan.makespan_ms,
                                   "truncated": plan.search_truncated, "ms": plan_ms},
                       "launch": "CUDA graph replay of the step" if replay is not None else "direct launches",
                       "suffix_kernel": "mma.sync, early launch on the SMs the TC grid leaves (PDL)",
                       "tc_sm_budget": step.tc_sm_budget, "tc_ctas": step.info.n_tc_blocks * h_local,
                       "autotune_ms": tune_ms},
            "roofline": roof,
            "hbm_roofline_step": {"achieved": value / world, "peak": hbm, "unit": "GB/s",
                                  "frac": value / world / hbm, "frac_of_8tbs": value / world / 8000.0},
            "kernels": kernels,
            "kernels_window_ms_per_step": ms_ev,
            "work": work,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": step.launches * args.steps,
            "clocks": clock_rec,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
