"""Decode-attention benchmark (BASELINE.json metric) for the B200 path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--partition heads|trees] [--no-cpu-baseline]

Workload (config[1] of BASELINE.json): Llama-3-8B shape, 32 q / 8 kv
heads, d=128, bf16 KV; 256 requests share a 32K-token system prompt, each
with a private 512-token suffix. Synthetic N(0,1)/sqrt(d) data generated
on the device (K/V pool 671 MB > 126 MB L2, so every step streams from
HBM). A "step" = one decode-attention call over all requests.

value = effective unique-KV GB/s over the whole job (all ranks). With N
GPUs the step is sharded: `--partition heads` splits the
kv heads N ways (tensor-parallel head split; default) and `--partition
trees` LPT-assigns whole trees of the forest to ranks (cfg4's default);
either way the per-rank outputs are gathered inside the timed step (by
head block or by request): by default fused into the merge kernel, which
stores every output row into all ranks' global output buffers over
NVLink and signals them (parallel.PeerGather), or with `--gather nccl`
by an NCCL all-gather after the step. `e2e` times the same step
through the public API with queries copied from pinned host memory and the
output read back every step, in the same >= 2 s windows as `value`.
After timing, untimed, the bench checks sampled requests of its own output
against a float64 recomputation on the device (and, with N > 1, that the
gathered output holds every rank's rows).

--impl reference times the reference's CPU implementation (prefixdec,
installed unmodified into baseline/_ref; the oracle port under oracle/
when it is absent) on a bounded sample of the same workload (rank 0 only).
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
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode-attn µs/step & effective KV GB/s (unique bytes) vs HBM roofline, 1-8 GPU"
CONFIGS = {  # BASELINE.json "configs"; structures from workloads.make_config
    "cfg1": dict(h_q=8, h_kv=8, d=128,
                 label="cfg1: tiny 2-level tree, 16 requests sharing a 1K prefix + 64-token suffixes, 8 heads x d128"),
    "cfg2": dict(h_q=32, h_kv=8, d=128, ref_heads=2,
                 label="cfg2: Llama-3-8B shape (32 q / 8 kv heads, d128, bf16 KV), 256 requests sharing a "
                       "32K system prompt + 512-token suffixes"),
    "cfg3": dict(h_q=32, h_kv=8, d=128, ref_heads=2,
                 label="cfg3: tree-of-thought / beam tree, depth 4, branching 4, 8K root, irregular node lengths "
                       "(64 requests), Llama-3-8B heads"),
    "cfg4": dict(h_q=32, h_kv=8, d=128, cpu_trees=range(8), ref_heads=2,
                 label="cfg4: imbalanced forest, 64 trees with 512..128K shared prefixes and 1..512 requests per "
                       "tree + 512-token suffixes (4680 requests), Llama-3-8B heads"),
    "cfg5": dict(h_q=64, h_kv=8, d=128, ref_heads=1,
                 label="cfg5: Llama-3-70B shape (64 q / 8 kv heads, d128, bf16 KV), 1024 requests sharing a "
                       "64K prefix + 512-token suffixes"),
}
MIN_WINDOW_S = 2.0  # every timed quantity: >= 2 s of back-to-back windows, median window


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
        pw = [v for v in (num(r[2]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_median": statistics.median(pw) if pw else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU side
def _ref_sample_spec(cfg):
    """The bounded CPU sample of a config: kv heads [0, ref_heads) of the
    whole workload (heads are independent, attention.py:91-92), and for
    cfg4 trees 0..7 only (its fp32 tensors exceed host RAM)."""
    over = {"only_trees": cfg["cpu_trees"]} if "cpu_trees" in cfg else {}
    hk = cfg.get("ref_heads", cfg["h_kv"])
    g = cfg["h_q"] // cfg["h_kv"]
    if hk != cfg["h_kv"]:
        over.update(h_q=hk * g, h_kv=hk)
    spec = structure(cfg["name"], dtype=np.float32, **over)
    what = (f"trees {list(cfg['cpu_trees'])} ({spec.bs} requests)" if "cpu_trees" in cfg
            else f"all {spec.bs} requests")
    desc = f"{what}, kv heads 0..{hk - 1} of {cfg['h_kv']} ({hk * g} q heads), {sum(spec.length[1:])} KV tokens"
    return spec, hk, desc


def _ref_bytes(spec, hk, d):
    """unique KV bytes of the sample at bf16 width (the GPU's unit)"""
    qs = set(n for p in spec.paths for n in p)
    return sum(spec.length[n] for n in qs) * hk * d * 2 * 2


class ReferenceRunner:
    """prefixdec.execute() -- the reference's own CPU path, unmodified,
    from baseline/_ref -- on a bounded sample, with the plan parameters of
    the GPU run: the same cost CSV (the bundled B200
    profile) and m = the GPU plan's tensor-core blocks; the numpy kernel
    backend (faster than Cython at every shared shape);
    BlockPool(worker_count = host threads). Falls back to the oracle port
    when baseline/_ref is absent."""

    def __init__(self, cfg, m=48, workers=None):
        self.cfg = cfg
        self.workers = workers or os.cpu_count()
        spec, hk, desc = _ref_sample_spec(cfg)
        self.bytes = _ref_bytes(spec, hk, cfg["d"])
        ref = ROOT / "baseline" / "_ref"
        self.kind = "port"
        try:
            if ref.exists():
                sys.path.insert(0, str(ref))
                os.environ["PREFIXDEC_KERNEL"] = "python"
                import prefixdec  # noqa: F401
                self.kind = "reference"
        except ImportError:
            self.kind = "port"
        t0 = time.perf_counter()
        if self.kind == "reference":
            import prefixdec as R
            q = R.QueryBatch(spec.queries, hk)
            self.forest = R.build_forest(spec.node_specs(), spec.paths, q)
            self.queries = q
            table = R.load_profile(ROOT / "paper_2505_17694_b200" / "profiles" / "b200_d128.csv")
            self.plan = R.divide_and_schedule(R.tasks_from_forest(self.forest), table, m)
            self.pool = R.BlockPool(worker_count=self.workers)
            self.run = lambda: R.execute(self.forest, self.queries, self.plan, self.pool)
            n_sub = len(self.plan.subtasks)
            plan_desc = f"divide_and_schedule(m={m}, B200 profile CSV): {n_sub} subtasks"
        else:
            from oracle import attention as OA
            from oracle import index as OI
            from oracle import plan as OP
            z = np.zeros((0, hk, cfg["d"]), np.float32)
            fd = OA.ForestData(spec.parent, [z] + spec.keys[1:], [z] + spec.values[1:], spec.paths)
            qs = OI.query_sets(spec.paths, spec.n_nodes)
            subs = [(node, a, b) for node, nq, n in OP.node_tasks(qs, spec.length)
                    for a, b in OP.slices(n, self.workers if nq > 1 else 1)]
            self.run = lambda: OA.execute(fd, spec.queries, subs, workers=self.workers)
            plan_desc = f"oracle port, per-thread split plan of {len(subs)} subtasks"
        self.plan_s = time.perf_counter() - t0
        self.desc = (f"{desc}; fp32 inputs (the reference has no bf16); "
                     f"{'prefixdec.execute from baseline/_ref, numpy backend' if self.kind == 'reference' else 'oracle port'}"
                     f", {self.workers} threads, {plan_desc}")

    def step(self):
        t0 = time.perf_counter()
        self.run()
        return time.perf_counter() - t0


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    r = ReferenceRunner(cfg, m=args.ref_m)
    for _ in range(args.warmup):
        r.step()
    times = [r.step() for _ in range(args.steps)]
    t = statistics.mean(times)
    value = r.bytes / t / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["label"], "sample": r.desc},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": r.workers, "kind": r.kind, "sample": r.desc},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU side
def prepare(config="cfg2", dev=None, rank=0, world=1, partition=None, flags=0, serial=False, blocks=0,
            budgets=None, seed=1234, quick=False):
    """Inputs, plan and the autotuned DecodeStep of one rank of the bench
    (the exact step `value` times; tests/test_gpu_fullsize.py runs it too).

    Synthetic bf16 K/V pools and queries drawn on the device (seeded per
    rank); plan = plan_device (shared nodes whole, divided by the device
    balancer; suffixes on the mma.sync kernel); the tensor-core SM budget
    is tuned once per plan (cuDNN-benchmark style, untimed), max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2505_17694_b200 as P
    from paper_2505_17694_b200 import parallel as PL
    from paper_2505_17694_b200.executor import DecodeStep

    cfg = dict(CONFIGS[config], name=config)
    dev = dev or torch.device("cuda", 0)
    h_kv, h_q, d = cfg["h_kv"], cfg["h_q"], cfg["d"]
    g = h_q // h_kv
    partition = partition or ("trees" if config == "cfg4" and world > 1 else "heads")
    spec = structure(config, tensors=False)
    full = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, h_kv, d)
    table = P.load_default_profile()
    shard = shards = None
    if partition == "trees" and world > 1:
        part = PL.tree_partition(full, table, world, head_multiplicity=g)
        shards = [PL.shard_trees(full, part, r) for r in range(world)]
        shard = shards[rank]
        forest = shard.forest(h_kv, d)
        h0, h_local = 0, h_kv
    elif partition in ("heads", "trees"):
        h0, h1 = PL.head_shard(h_kv, world, rank)
        forest, h_local = full, h1 - h0
    else:
        raise ValueError(f"partition must be heads or trees, got {partition!r}")
    hq_local = h_local * g
    bs = forest.bs
    T = forest.total_tokens
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed + rank)
    sc = 1.0 / math.sqrt(d)
    kp = (torch.randn((h_local, T, d), generator=gen, device=dev, dtype=torch.float32) * sc).to(torch.bfloat16)
    vp = (torch.randn((h_local, T, d), generator=gen, device=dev, dtype=torch.float32) * sc).to(torch.bfloat16)
    q_host = (torch.randn((bs, hq_local, d), generator=torch.Generator().manual_seed(99 + rank)) * sc
              ).to(torch.bfloat16).pin_memory()
    q_dev = q_host.to(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out = torch.empty((bs, hq_local, d), dtype=torch.float32, device=dev)

    def make(cand):
        budget, fl = cand
        t0 = time.perf_counter()
        if blocks:
            pl = P.divide_and_schedule(P.device_tasks(forest, g), table, blocks)
        else:
            pl = P.plan_device(forest, g, table, h_local, sms, budget, multi=not (fl & 524288),  # FLAG_NO_MULTI
                               tct=not (fl & 4194304))  # FLAG_NO_TCT
        ms_plan = (time.perf_counter() - t0) * 1e3
        st = DecodeStep(forest, pl, h_q, "bfloat16", head_begin=h0, head_end=h0 + h_local, device=dev,
                        flags=fl, tc_sm_budget=budget, concurrent=not serial)
        return pl, st, ms_plan

    # TC SM budget: the SMs the TC grid leaves free run the suffix kernel
    # from the start (programmatic dependent launch); tuned once per plan,
    # together with the routing of lightly shared nodes (17..128 rows): the
    # transposed tensor-core kernel takes them off the pair kernel's SMs
    # (a gain when the step is tensor-bound, cfg4) but adds to the HBM-bound
    # side (a loss when that is the long pole, cfg3)
    if budgets is None:
        budgets = [sms] if (serial or quick) else [sms] + list(range(136, 55, -8))
    routings = [flags]
    if not (flags & 4194304) and not blocks and not quick and len(budgets) > 1:
        has = torch.tensor([int(make((budgets[0], flags))[1].info.n_tct_groups > 0)], device=dev)
        if world > 1:  # every rank tunes the same candidates
            dist.all_reduce(has, op=dist.ReduceOp.MAX)
        if int(has.item()):
            routings.append(flags | 4194304)
    tune_ms, best = {}, None
    queue = [(b, fl) for fl in routings for b in budgets]
    refined = len(budgets) < 2
    while queue:
        cand = queue.pop(0)
        b = cand[0]
        pl, st, ms_plan = make(cand)
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
        tune_ms[f"{b}{'' if cand[1] & 4194304 == flags & 4194304 else '/notct'}"] = round(t_b, 4)
        if best is None or t_b < best[0]:
            best = (t_b, cand, pl, st, ms_plan)
        if not queue and not refined:  # a finer pass (+-4 SMs) around the coarse optimum
            refined = True
            b0, f0 = best[1]
            queue = [(x, f0) for x in (b0 - 4, b0 + 4) if 16 <= x < sms and x not in budgets]
    _, (budget, flags), plan, step, plan_ms = best
    return SimpleNamespace(cfg=cfg, config=config, dev=dev, rank=rank, world=world, partition=partition,
                           spec=spec, full=full, forest=forest, shard=shard, shards=shards, h0=h0,
                           h_local=h_local, hq_local=hq_local, g=g, kp=kp, vp=vp, q_host=q_host, q_dev=q_dev,
                           out=out, sms=sms, plan=plan, budget=budget, step=step, plan_ms=plan_ms,
                           tune_ms=tune_ms, table=table, blocks=blocks, flags=flags)


def library_reference(config):
    """FlashInfer's B200 decode and cascade kernels on this workload, from
    the committed same-box comparison (tools/library_baseline.py; not timed
    in this run -- `source` names the capture), or None."""
    p = ROOT / "profiles" / f"r02_library_baseline_{config}.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text().strip().splitlines()[-1])
    except Exception:
        return None
    out = {"source": str(p.relative_to(ROOT)), "note": "separate run on one B200; both arms in >= 3-s windows",
           "ours_us": d["ours"]["us"]}
    for k in ("trtllm_gen_decode", "cascade"):
        if "us" in d.get(k, {}):
            out[k + "_us"] = d[k]["us"]
            out[k + "_max_abs_vs_ours"] = d[k].get("max_abs_vs_ours")
    return out


def path_reference(forest, kp, vp, q, r):
    """Single-softmax attention of (local) request r over its root-to-leaf
    path (naive_attention, attention.py:164-187) in float64 on the device
    from the same bf16 values -- the bench's untimed self-check."""
    import torch
    toks = torch.cat([torch.arange(forest.token_offset[n], forest.token_offset[n] + forest.visible_count(n, r),
                                   device=kp.device) for n in forest.paths[r]])
    h_local = kp.shape[0]
    g = q.shape[1] // h_local
    k = kp[:, toks].double()
    v = vp[:, toks].double()
    qq = q[r].double().view(h_local, g, -1)
    s = torch.einsum("hgd,hld->hgl", qq, k) / math.sqrt(forest.d)
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hgl,hld->hgd", p, v).reshape(q.shape[1], -1)


def verify(ns, out, n=8, seed=0):
    """Sampled requests of `out` against path_reference: the bf16 bar of
    the north star (max-abs 2e-3 and max-norm rel 1e-2)."""
    bs = ns.forest.bs
    rng = np.random.default_rng(seed)
    reqs = sorted({0, bs - 1} | set(rng.choice(bs, size=min(n, bs), replace=False).tolist()))
    worst_abs = worst_rel = 0.0
    for r in reqs:
        ref = path_reference(ns.forest, ns.kp, ns.vp, ns.q_dev, r)
        err = float((out[r].double() - ref).abs().max())
        worst_abs = max(worst_abs, err)
        worst_rel = max(worst_rel, err / float(ref.abs().max()))
    ok = worst_abs <= 2e-3 and worst_rel <= 1e-2 and bool(out.isfinite().all())
    return {"requests": len(reqs), "max_abs": worst_abs, "max_rel": worst_rel, "ok": ok,
            "reference": "float64 softmax over each sampled request's path, on the device, same bf16 inputs"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--partition", default=None, choices=["heads", "trees"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--blocks", type=int, default=0, help="planner m (0: the device plan)")
    ap.add_argument("--ref-m", type=int, default=48, help="reference arm: planner m (the GPU plan's TC blocks)")
    ap.add_argument("--quick", action="store_true", help="profiling run: no e2e / clocks / cpu baseline / tuning")
    ap.add_argument("--serial", action="store_true", help="one stream: TC, GEMV and merge back to back")
    ap.add_argument("--no-graph", action="store_true", help="launch the step directly instead of a CUDA graph replay")
    ap.add_argument("--budget", type=int, default=0, help="fixed tensor-core SM budget (no tuning)")
    ap.add_argument("--gather", default="fused", choices=["fused", "nccl"],
                    help="N > 1 output gather: fused peer stores from the merge kernel (default) or NCCL all-gather")
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
    from paper_2505_17694_b200 import parallel as PL

    # CODEC_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo for the control
    # plane -- a single-GPU emulation of the multi-rank path (tests only;
    # the fused gather's peer stores and counters work across processes
    # sharing a GPU; the NCCL gather does not)
    one_gpu = os.environ.get("CODEC_BENCH_ONE_GPU") == "1"
    dev_index = 0 if one_gpu else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2505_17694_b200.executor import FLAG_MERGE_ALL
    fused = world > 1 and args.gather == "fused"
    gather_note = None
    if fused:
        # probe the peer mapping (CUDA IPC + peer access) once; every rank
        # takes the NCCL gather if any rank cannot map its peers' buffers
        err, probe = None, None
        try:
            probe = PL.PeerGather(1, 1, 1, dev)
        except Exception as e:  # noqa: BLE001 -- reported in the bench line
            err = f"{type(e).__name__}: {e}"
        bad = torch.tensor([1 if err else 0], dtype=torch.int32, device="cpu" if one_gpu else dev)
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if not int(bad.item()):
            probe.close()  # barriers inside: only when every rank holds a probe
        else:  # a probe a rank did map stays allocated (16 bytes)
            fused = False
            gather_note = "fused peer-store gather unavailable on this box (" + (err or "another rank failed") + \
                "); NCCL all-gather used"
    flags = args.flags | (FLAG_MERGE_ALL if fused else 0)
    ns = prepare(args.config, dev, rank, world, args.partition, flags, args.serial, args.blocks,
                 budgets=[args.budget] if args.budget else None, quick=args.quick)
    step, plan, budget = ns.step, ns.plan, ns.budget
    kp, vp, q_dev, q_host, out = ns.kp, ns.vp, ns.q_dev, ns.q_host, ns.out
    bs, hq_local, d = ns.forest.bs, ns.hq_local, ns.cfg["d"]
    full_bs, h_q = ns.full.bs, ns.cfg["h_q"]
    m = args.blocks or max(1, budget // 2)
    trees = ns.partition == "trees" and world > 1
    # receive buffers of the output gather (by head block or by request)
    n_max = max(s.bs for s in ns.shards) if trees else bs
    gathered = torch.empty((world, n_max, hq_local, d), dtype=torch.float32, device=dev) if world > 1 else None
    send = torch.zeros((n_max, hq_local, d), dtype=torch.float32, device=dev) if trees else None

    # fused gather: the merge kernel stores this rank's
    # rows into every rank's global output over NVLink and bumps their
    # arrival counters; no NCCL call on the data path
    peers = row_map = None
    head0 = ns.h0 * ns.g
    if fused:
        peers = PL.PeerGather(full_bs, h_q, d, dev, buffers=2)
        if trees:
            row_map = torch.tensor(list(ns.shard.requests), dtype=torch.int32, device=dev)
            head0 = 0

    def gather(o, buf):
        if world == 1:
            return o
        if trees:  # pad to the largest shard, one all-gather, scatter back by request
            send[:bs].copy_(o)
            dist.all_gather_into_tensor(buf.view(world * n_max, hq_local, d), send)
            return buf
        dist.all_gather_into_tensor(buf.view(world * bs, hq_local, d), o)
        return buf

    # the timed step replays a CUDA graph of the decode step (its three
    # launches recorded once; no per-step host work)
    if fused:
        replay = (step.capture_gather(q_dev, kp, vp, peers, head0, row_map, buf=0) if not args.no_graph else None)
    else:
        replay = step.capture(q_dev, kp, vp, out) if not args.no_graph else None

    def one_step():
        if fused:
            if replay is not None:
                replay()
            else:
                step.gather(q_dev, kp, vp, peers, head0, row_map, buf=0)
                peers.wait()
            return peers.output(0)
        if replay is not None:
            replay()
        else:
            step(q_dev, kp, vp, out=out)
        return gather(out, gathered)

    hbm, tf_burst, tf_sus, peak_kind = peaks()
    stream = torch.cuda.current_stream(dev)

    def all_done(local_done):
        """Stop a timing loop on every rank together (each rank's wall
        clock decides locally; the ranks' collectives must pair up)."""
        if world == 1:
            return local_done
        f = torch.tensor([1 if local_done else 0], device=dev)
        dist.all_reduce(f, op=dist.ReduceOp.MAX)
        return bool(f.item())

    def timed(n, fn, min_seconds=0.0):
        """ms per call over n calls between barrier+sync on both sides, CUDA
        events on the launching stream, max over ranks. The n-call window
        is repeated until min_seconds of wall time passed (so the clock
        sampler sees the load and the power cap settles) and the median
        window is used."""
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
            if all_done(time.perf_counter() - t_start >= min_seconds or len(windows) >= 5000):
                break
        return statistics.median(windows), len(windows)

    win_s = 0.0 if args.quick else MIN_WINDOW_S
    for _ in range(max(args.warmup, 3)):
        one_step()
    torch.cuda.synchronize(dev)
    clocks = None if args.quick else ClockSampler(local_rank)
    ms, windows = timed(args.steps, one_step, min_seconds=win_s)
    clock_rec = clocks.stop() if clocks else None

    # per-kernel device time: a twin step that records CUDA events around
    # each of its kernels (codec_kernel_timer) on the launching stream, in
    # the same >= 2 s windows. The events sit between the kernels, so the
    # twin runs them back to back (no early suffix launch): these times
    # attribute work to kernels; `value` is the overlapped step.
    step_ev = step.with_budget(budget, timer=True)
    for _ in range(3):
        step_ev(q_dev, kp, vp, out=out)
    torch.cuda.synchronize(dev)
    step_ev.kernel_times()  # drop the warm-up calls' events
    ms_ev = 0.0
    kt_all = []
    t_ev0 = time.perf_counter()
    while True:  # read the ring between windows (4096 calls)
        ms_w, _ = timed(args.steps, lambda: step_ev(q_dev, kp, vp, out=out))
        ms_ev = ms_w
        kt_all.append(step_ev.kernel_times())
        if all_done(time.perf_counter() - t_ev0 >= win_s):
            break
    kt = np.concatenate(kt_all) if kt_all else np.zeros((0, 3))
    info = step.info
    phases = {}
    if len(kt):
        for j, (name, present) in enumerate((("tc", info.n_tc_groups), ("gemv", info.n_gemv_groups),
                                             ("merge", info.n_merge))):
            if present:
                phases[name] = float(np.median(kt[:, j]))

    work_local = P.device_work(ns.forest, h_q, element_size=2, head_fraction=ns.h_local / ns.cfg["h_kv"])
    work_full = P.device_work(ns.full, h_q, element_size=2)
    total_bytes = work_full["unique_kv_bytes"]
    value = total_bytes / (ms * 1e-3) / 1e9
    g = ns.g
    from paper_2505_17694_b200.scheduler import node_kernel
    on_tc = [n for n in ns.forest.nodes[1:] if n.query_set and
             node_kernel(len(n.query_set) * g, len(n.query_set), not (ns.flags & 524288),
                         not (ns.flags & 4194304)) == "tc"]
    kv_tc = sum(n.len for n in on_tc) * ns.h_local * d * 2 * 2
    kernels = {}
    if "tc" in phases:
        fl = sum(n.len * len(n.query_set) for n in on_tc) * hq_local * 4 * d
        ach = fl / (phases["tc"] * 1e-3) / 1e12
        sms_tc = int(min(budget, ns.sms))
        # timed inside >= 2 s windows of back-to-back steps: the sustained
        # cuBLAS figure; the burst figure and the SM share are reported beside it
        kernels["tc"] = {"bound": "tensor", "achieved": ach, "peak": tf_sus, "peak_figure": "bf16_tflops_sustained",
                         "unit": "TFLOP/s", "ms": phases["tc"], "algorithmic_flops": fl, "kv_bytes": kv_tc,
                         "frac": ach / tf_sus, "frac_of_burst": ach / tf_burst, "sms": sms_tc,
                         "sm_share": sms_tc / ns.sms,
                         "note": "the TC grid holds `sms` SMs; the rest stream the suffixes concurrently"}
    if "gemv" in phases:
        kb = work_local["unique_kv_bytes"] - kv_tc
        kernels["gemv"] = {"bound": "hbm", "achieved": kb / (phases["gemv"] * 1e-3) / 1e9, "peak": hbm,
                           "unit": "GB/s", "ms": phases["gemv"], "algorithmic_bytes": kb}
        kernels["gemv"]["frac"] = kernels["gemv"]["achieved"] / hbm
    if "merge" in phases:
        kernels["merge"] = {"ms": phases["merge"]}
    # DRAM traffic per launch from the committed ncu --set full capture of
    # this workload at the benchmarked SM budget (profiles/ncu_summary.json)
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
            kernels[name]["traffic_budget"] = ncu.get("tc_sm_budget")
    dominant = max((k for k in kernels if "bound" in kernels[k]), key=lambda k: kernels[k]["ms"], default=None)
    roof = None
    if dominant:
        k = kernels[dominant]
        roof = {"bound": k["bound"], "achieved": k["achieved"], "peak": k["peak"], "unit": k["unit"],
                "frac": k["frac"], "traffic": k.get("traffic"), "kernel": dominant, "peak_kind": peak_kind,
                "peak_figure": k.get("peak_figure", "hbm_gbs"), "frac_of_burst": k.get("frac_of_burst"),
                "sms": k.get("sms")}

    e2e = None
    if not args.quick:
        # Serving-style pipeline through the public API (DecodeStep's
        # captured graphs): every step uploads its queries from pinned host
        # memory and reads its output back; step k's copies run on their
        # own streams, overlapping the compute of steps k - 1 / k + 1
        # (double-buffered device q / out, one captured graph per buffer
        # set). Same >= 2 s median windows as `value`.
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        qbuf = [torch.empty_like(q_dev) for _ in range(2)]
        obuf = [torch.empty_like(out) for _ in range(2)]
        gbuf = [torch.empty_like(gathered) for _ in range(2)] if world > 1 else [None, None]
        rows_out = full_bs if world > 1 else bs
        ohost = [torch.empty((rows_out, (h_q if (world > 1 and not trees) else hq_local), d),
                             dtype=torch.float32).pin_memory() for _ in range(2)]
        if fused:
            replays = [step.capture_gather(qbuf[i], kp, vp, peers, head0, row_map, buf=i) for i in range(2)]
        else:
            replays = [step.capture(qbuf[i], kp, vp, obuf[i]) for i in range(2)] if not args.no_graph else None
        ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("h2d", "comp", "d2h")}
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
            if fused:
                replays[sl]()
                res = peers.output(sl)
            elif replays is not None:
                replays[sl]()
                res = obuf[sl]
            else:
                step(qbuf[sl], kp, vp, out=obuf[sl], stream=stream)
                res = obuf[sl]
            if world > 1 and not fused:
                buf = gather(obuf[sl], gbuf[sl])
                res = PL.scatter_requests(buf, ns.shards, full_bs) if trees else PL.assemble_heads(buf)
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
            ms_w = e0.elapsed_time(e1) / n
            if world > 1:
                t = torch.tensor([ms_w], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms_w = float(t.item())
            return ms_w

        e2e_window(3)
        wins, t0 = [], time.perf_counter()
        while True:
            wins.append(e2e_window(args.steps))
            if all_done(time.perf_counter() - t0 >= win_s):
                break
        e2e_ms = statistics.median(wins)
        e2e = {"value": total_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
               "windows": len(wins),
               "h2d_bytes_per_step": q_host.numel() * q_host.element_size(),
               "d2h_bytes_per_step": ohost[0].numel() * ohost[0].element_size(),
               "pipeline": "per step: pinned H2D of q, decode step (graph replay), D2H of out; copies on their "
                           "own streams overlap the neighbouring steps' compute (double-buffered); >= 2 s "
                           "median windows like `value`"}

    # untimed self-check of the benchmarked step's output
    torch.cuda.synchronize(dev)
    if fused:
        res = one_step()  # the gathered global output
        step(q_dev, kp, vp, out=out)  # this rank's rows, written locally by the same kernels
    elif replay is not None:
        replay()
        res = gather(out, gathered)
    else:
        step(q_dev, kp, vp, out=out)
        res = gather(out, gathered)
    torch.cuda.synchronize(dev)
    check = verify(ns, out)
    if world > 1:  # the gathered output holds this rank's rows unchanged
        if fused:
            full_out = res
        else:
            full_out = PL.scatter_requests(res, ns.shards, full_bs) if trees else PL.assemble_heads(res)
        mine = full_out[list(ns.shard.requests)] if trees else full_out[:, ns.h0 * g:(ns.h0 + ns.h_local) * g]
        check["gather_ok"] = bool(torch.equal(mine, out))
        flag = torch.tensor([0 if (check["ok"] and check["gather_ok"]) else 1], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        check["all_ranks_ok"] = int(flag.item()) == 0

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        r = ReferenceRunner(ns.cfg, m=m)
        r.step()  # warm
        dt = min(r.step() for _ in range(2))
        cpu = {"value": r.bytes / dt / 1e9, "unit": "GB/s", "cores": r.workers, "kind": r.kind,
               "sample": r.desc, "seconds": dt, "plan_seconds": r.plan_s}

    run_rep = None
    if rank == 0 and ns.forest is ns.full:
        # the reference CLI's RunReport for this workload point (report.py;
        # schemas/report.schema.json admits the reference's four families)
        from paper_2505_17694_b200 import workloads as W
        from paper_2505_17694_b200.report import FAMILIES, check_report, run_report
        kw = W.CONFIGS[args.config]
        fam = kw["fn"].__name__
        if fam in FAMILIES:
            params = {k: v for k, v in kw["kw"].items() if k not in ("h_q", "h_kv", "d", "seed")}
            wl = {"family": fam, "params": params, "seed": int(kw["kw"].get("seed", 0)),
                  "dims": {"h_q": h_q, "h_kv": ns.cfg["h_kv"], "d": d}}
            run_rep = run_report(ns.full, plan, ns.table, m, wl, max_rel_err=check["max_rel"], element_size=2)
            check_report(run_rep)
    if rank == 0:
        traffic = P.traffic_report(ns.full, element_size=2)
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "timed_windows": windows, "us_per_step": ms * 1e3,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",  # the config's workload, split over N GPUs
            "data": "synthetic: N(0,1)/sqrt(d) K/V/Q generated on device (seeded), no checkpoint",
            "config": {"workload": ns.cfg["label"], "bs": full_bs, "h_q": h_q, "h_kv": ns.cfg["h_kv"], "d": d,
                       "kv_tokens": int(sum(ns.spec.length[1:])), "nodes": int(ns.spec.n_nodes - 1),
                       "parallelism": ((f"tree partition x{world}" if trees else f"kv-head split x{world}") +
                                       ("" if world == 1 else
                                        " + fused peer-store output gather (merge kernel -> NVLink)" if fused else
                                        (" + NCCL all-gather by request" if trees else " + NCCL all-gather"))),
                       **({"gather_note": gather_note} if gather_note else {}),
                       "l2": "inputs larger than L2 (KV pool %.0f MB > 126 MB)" % (2 * kp.numel() * 2 / 1e6),
                       "planner": {"m_tc": m, "subtasks": len(plan.subtasks), "makespan_ms": plan.makespan_ms,
                                   "truncated": plan.search_truncated, "ms": ns.plan_ms},
                       "launch": "CUDA graph replay of the step" if replay is not None else "direct launches",
                       "suffix_kernel": "mma.sync, early launch on the SMs the TC grid leaves (PDL)",
                       "tc_sm_budget": step.tc_sm_budget, "tc_ctas": step.info.n_tc_blocks * 2,
                       "lightly_shared": ("transposed tensor-core kernel (%d CTAs)" % (step.info.n_tct_groups * ns.h_local)
                                          if step.info.n_tct_groups else "pair kernel / mma.sync kernels"),
                       "autotune_ms": ns.tune_ms},
            "roofline": roof,
            "hbm_roofline_step": {"achieved": value / world, "peak": hbm, "unit": "GB/s",
                                  "frac": value / world / hbm, "frac_of_8tbs": value / world / 8000.0},
            "kernels": kernels,
            "kernels_window_ms_per_step": ms_ev,
            "work": work_full,
            "flashdecoding_bytes": {"bytes_baseline": traffic.bytes_baseline, "bytes_unique": total_bytes,
                                    "reduction": traffic.bytes_baseline / total_bytes,
                                    "dram_bytes_ncu": ncu.get("step_dram_bytes")},
            "verified": check,
            "library_reference": library_reference(args.config),
            "run_report": run_rep,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": step.launches * args.steps * windows,
            "clocks": clock_rec,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if not check["ok"] or not check.get("all_ranks_ok", True):
        raise SystemExit(f"bench output failed its self-check: {check}")


if __name__ == "__main__":
    main()
