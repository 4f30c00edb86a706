"""The decode-attention step on the B200 (reference-compatible `execute`).

`execute(forest, queries, plan, pool)` keeps the signature and error
behaviour of prefixdec/executor.py:296-308 and returns [bs, h_q, d]. The
reference runs the plan's subtasks on a host thread pool, barriers, and
folds each request's partials with por(); here the plan is expanded once
into a device task table (C++ codec_table_build: the row filter, the
per-row visible clip and the path-then-slice partial lists of
executor.py:145-231) and one call of codec_decode_attention runs
    tcgen05 shared-node kernel | GEMV suffix kernel | generic kernel
    -> LSE merge kernel
on the current CUDA stream.

`DecodeStep` is the prepared form (table + workspace uploaded once) that
serving code reuses across decode steps until the next re-plan
(DEFAULT_REPLAN_EVERY in scheduler.py), and that bench.py times.
`BlockPool` is accepted for API compatibility: the GPU's CTAs are the
blocks. `reduce_mode` "balanced" and "sequential" both map to the single
pass max-then-sum merge (same result up to rounding, test_attention.py:
160-180). The reference's simulated EventTrace is out of scope (CUDA
events and ncu replace simulated time).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .attention import torch_dtype
from .errors import DimensionMismatch
from .forest import Forest, QueryBatch, dtype_code

FLAG_NO_TC = 1
FLAG_FORCE_TC = 2
FLAG_NO_GEMV = 4
FLAG_NO_MULTI = 524288
FLAG_NO_TCT = 4194304  # no transposed tensor-core kernel (its slices on the pair kernel)
FLAG_TCT_WIDE = 8388608  # the transposed kernel also takes nodes of 65..128 rows (plan with tct_wide=True)
FLAG_MERGE_ALL = 2097152  # every output row through the merge kernel (the fused peer-store gather needs it)


@dataclass
class BlockPool:
    """API shim for prefixdec.executor.BlockPool (executor.py:35-44)."""

    worker_count: int = 1
    deterministic: bool = True

    def __post_init__(self):
        if self.worker_count < 1:
            raise ValueError(f"worker_count must be >= 1, got {self.worker_count}")


def _plan_arrays(plan):
    tasks = plan.tasks
    t_node = np.ascontiguousarray([t.node for t in tasks], dtype=np.int64)
    t_nq = np.ascontiguousarray([t.n_q for t in tasks], dtype=np.int64)
    s_task = np.ascontiguousarray([s.task_index for s in plan.subtasks], dtype=np.int32)
    s_start = np.ascontiguousarray([s.start for s in plan.subtasks], dtype=np.int64)
    s_stop = np.ascontiguousarray([s.stop for s in plan.subtasks], dtype=np.int64)
    s_block = np.ascontiguousarray(plan.assignment.block_of, dtype=np.int32)
    return t_node, t_nq, s_task, s_start, s_stop, s_block


def table_for(forest: Forest, plan, dims):
    """(codec_table_info, int32 blob) of a plan expanded for the device
    (codec_table_build): host-only, no GPU needed."""
    t_node, t_nq, s_task, s_start, s_stop, s_block = _plan_arrays(plan)
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.codec_table_build(forest._index, C.byref(dims), len(t_node), P(t_node, C.c_int64),
                                   P(t_nq, C.c_int64), len(s_task), P(s_task, C.c_int32),
                                   P(s_start, C.c_int64), P(s_stop, C.c_int64), P(s_block, C.c_int32),
                                   C.byref(h)))
    try:
        info = _lib.TableInfo()
        _lib.check(L.codec_table_info_get(h, C.byref(info)))
        blob = np.zeros(max(info.blob_len, 4), dtype=np.int32)
        _lib.check(L.codec_table_copy(h, P(blob, C.c_int32)))
    finally:
        L.codec_table_free(h)
    return info, blob


def make_dims(forest: Forest, h_q: int, dtype="bfloat16", head_begin=0, head_end=None, flags=0, sm_count=148,
              tc_sm_budget=0, page_size=0, page_table_ptr=None, pool_tokens=None):
    return _lib.Dims(forest.bs, int(h_q), forest.h_kv, forest.d, int(head_begin),
                     forest.h_kv if head_end is None else int(head_end), dtype_code(dtype), int(flags),
                     int(pool_tokens) if pool_tokens is not None else max(forest.total_tokens, 1), int(sm_count),
                     int(tc_sm_budget), int(page_size), 0, page_table_ptr)


class DecodeStep:
    """A plan expanded into a device task table for one forest, dtype and
    kv-head shard. Call with device queries [bs, h_q_local, d] and the
    head-major pools; returns [bs, h_q_local, d] (float32, or float64 for
    float64 inputs).

    Paged pools (paging.py): page_size > 0 with page_table (device int32,
    one physical page per logical page) and pool_tokens = the physical
    pools' token stride; the pools passed to each call are then the
    physical ones."""

    def __init__(self, forest: Forest, plan, h_q: int, dtype="bfloat16", head_begin=0, head_end=None,
                 device="cuda", flags=0, tc_sm_budget=0, concurrent=True, page_size=0, page_table=None,
                 pool_tokens=None, timer=False):
        import torch

        self.forest = forest
        self.h_q, self.h_kv, self.d = int(h_q), forest.h_kv, forest.d
        self.head_begin = int(head_begin)
        self.head_end = forest.h_kv if head_end is None else int(head_end)
        self.g = self.h_q // self.h_kv
        self.tdtype = torch_dtype(dtype)
        self.device = torch.device(device)
        if torch.cuda.is_available():
            _lib.bind_device(self.device)
        sm = torch.cuda.get_device_properties(self.device).multi_processor_count if torch.cuda.is_available() else 148
        self.plan, self.flags, self.tc_sm_budget = plan, int(flags), int(tc_sm_budget)
        self.page_size, self.page_table = int(page_size), page_table
        if self.page_size and page_table is None:
            raise ValueError("page_size without a page_table")
        self.pool_tokens = int(pool_tokens) if pool_tokens is not None else max(forest.total_tokens, 1)
        self.dims = _lib.Dims(forest.bs, self.h_q, self.h_kv, self.d, self.head_begin, self.head_end,
                              dtype_code(self.tdtype), int(flags), self.pool_tokens, int(sm),
                              int(tc_sm_budget), self.page_size, 0,
                              C.c_void_p(page_table.data_ptr()) if self.page_size else None)
        # GEMV/generic kernels run on an aux stream, concurrently with the
        # tensor-core kernel (event fork/join inside the library)
        self.aux = torch.cuda.Stream(self.device) if concurrent and torch.cuda.is_available() else None
        self.info, blob = table_for(forest, plan, self.dims)
        self.blob_host = blob
        self.table = torch.from_numpy(blob).to(self.device)
        # partials, then a 256-byte tail whose first word is the TC kernel's
        # per-step completion counter (reset by the library before each TC
        # launch; the merge waits on it)
        self.workspace = torch.zeros(max(int(self.info.workspace_bytes), 256), dtype=torch.uint8, device=self.device)
        self.out_dtype = torch.float64 if self.tdtype == torch.float64 else torch.float32
        self.h_local = self.head_end - self.head_begin
        self.hq_local = self.h_local * self.g
        self._graphs = []
        self._grown = 0
        # per-kernel CUDA-event timer (profiling); it serialises the kernels
        self._timer = None
        if timer:
            h = C.c_void_p()
            _lib.check(_lib.lib().codec_timer_create(C.byref(h)))
            self._timer = h

    def __del__(self):
        if getattr(self, "_timer", None):
            try:
                _lib.lib().codec_timer_free(self._timer)
            except Exception:
                pass
            self._timer = None

    def kernel_times(self):
        """[calls, 3] ms of the (TC, suffix, merge) kernels of every call
        since the last read (needs timer=True)."""
        if not self._timer:
            raise ValueError("DecodeStep built without timer=True")
        buf = (C.c_float * (3 * 4096))()
        n = C.c_int32()
        _lib.check(_lib.lib().codec_timer_read(self._timer, buf, 4096, C.byref(n)))
        return np.array(buf[:3 * n.value], dtype=np.float64).reshape(-1, 3)

    def _check(self, name, t, shape, dtype):
        import torch
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch tensor on {self.device}")
        if t.device != self.device and not (self.device.index is None and t.device.type == self.device.type):
            raise ValueError(f"{name} is on {t.device}, the step on {self.device}")
        if t.dtype != dtype:
            raise DimensionMismatch(f"{name} is {t.dtype}, the step computes in {dtype}")
        if tuple(t.shape) != tuple(shape):
            raise DimensionMismatch(f"{name} has shape {tuple(t.shape)}, the step needs {tuple(shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")

    @property
    def launches(self) -> int:
        """Kernels one call launches (for the bench's gpu_launches)."""
        i = self.info
        return (int(bool(i.n_tc_groups)) + int(bool(i.n_gemv_groups)) + int(bool(i.n_gen_groups)) +
                int(bool(i.n_multi_groups)) + int(bool(i.n_tct_groups - i.n_tct_wide)) + int(bool(i.n_tct_wide)) +
                int(bool(i.n_merge)))

    def __call__(self, q, k_pool, v_pool, out=None, stream=None):
        """q [bs, h_q_local, d] and the pools [h_local, pool_tokens, d] in
        the step's dtype on its device (checked: the kernels get raw
        pointers); returns / fills out [bs, h_q_local, d]."""
        import torch

        bs = self.forest.bs
        self._check("q", q, (bs, self.hq_local, self.d), self.tdtype)
        pool_shape = (self.h_local, self.pool_tokens, self.d)
        self._check("k_pool", k_pool, pool_shape, self.tdtype)
        self._check("v_pool", v_pool, pool_shape, self.tdtype)
        if out is None:
            out = torch.empty((bs, self.hq_local, self.d), dtype=self.out_dtype, device=self.device)
        else:
            self._check("out", out, (bs, self.hq_local, self.d), self.out_dtype)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.bind_device(self.device)
        _lib.check(_lib.lib().codec_decode_attention_ex(
            C.byref(self.dims), C.byref(self.info), C.c_void_p(self.table.data_ptr()), C.c_void_p(q.data_ptr()),
            C.c_void_p(k_pool.data_ptr()), C.c_void_p(v_pool.data_ptr()), C.c_void_p(out.data_ptr()),
            C.c_void_p(self.workspace.data_ptr()), self.workspace.numel(), C.c_void_p(st.cuda_stream),
            C.c_void_p(self.aux.cuda_stream) if self.aux is not None else None, self._timer))
        return out

    def gather(self, q, k_pool, v_pool, peers, head0=None, row_map=None, buf=0, stream=None):
        """The step with the fused multi-GPU output gather (parallel.PeerGather;
        SURVEY.md §8(e) K5): the merge kernel stores this rank's output rows
        straight into every rank's global output buffer `buf` and signals
        them; call peers.wait(stream) before reading peers.output(buf).
        head0: this rank's first q head in the global rows (default
        head_begin * g); row_map: device int32 [bs] global row of each local
        request (tree partition; None = identity). The step must be built
        with FLAG_MERGE_ALL."""
        import torch

        if not self.flags & FLAG_MERGE_ALL:
            raise ValueError("gather() needs a DecodeStep built with flags |= FLAG_MERGE_ALL")
        bs = self.forest.bs
        self._check("q", q, (bs, self.hq_local, self.d), self.tdtype)
        pool_shape = (self.h_local, self.pool_tokens, self.d)
        self._check("k_pool", k_pool, pool_shape, self.tdtype)
        self._check("v_pool", v_pool, pool_shape, self.tdtype)
        if row_map is not None:
            self._check("row_map", row_map, (bs,), torch.int32)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        pg = peers.struct(self.head_begin * self.g if head0 is None else int(head0), row_map, buf)
        _lib.bind_device(self.device)
        _lib.check(_lib.lib().codec_decode_attention_gather(
            C.byref(self.dims), C.byref(self.info), C.c_void_p(self.table.data_ptr()), C.c_void_p(q.data_ptr()),
            C.c_void_p(k_pool.data_ptr()), C.c_void_p(v_pool.data_ptr()), C.c_void_p(self.workspace.data_ptr()),
            self.workspace.numel(), C.c_void_p(st.cuda_stream),
            C.c_void_p(self.aux.cuda_stream) if self.aux is not None else None, C.byref(pg)))

    def capture_gather(self, q, k_pool, v_pool, peers, head0=None, row_map=None, buf=0):
        """CUDA graph of gather() + peers.wait() over these buffers; returns
        its replay function."""
        import torch

        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            self.gather(q, k_pool, v_pool, peers, head0, row_map, buf, stream=s)
            peers.wait(s)
        self._graphs.append(graph)
        return graph.replay

    def capture(self, q, k_pool, v_pool, out):
        """Record one decode step over these buffers into a CUDA graph and
        return its replay function: the serving loop re-runs the step with
        new query values written into `q` in place, without the per-step
        host work (tensor-map encoding, argument checks, launches)."""
        import torch

        if self.aux is not None and (self.flags & 2048):
            raise ValueError("capture() needs the single-stream launch (no aux-stream GEMV)")
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):  # warm the kernels' attributes outside the capture
            self(q, k_pool, v_pool, out=out, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            self(q, k_pool, v_pool, out=out, stream=s)
        self._graphs.append(graph)  # keep alive with the step (one per captured buffer set)
        return graph.replay

    def grow(self, delta: int = 1) -> None:
        """Decode-step growth between re-plans (the
        reference re-plans every DEFAULT_REPLAN_EVERY steps, scheduler.py:23;
        PlanCache below drives that cadence). Build the forest with spare
        leaf capacity (leaf length > visible_len), write each request's new
        token K/V into the pool at the leaf's next token, then call grow():
        every request's leaf sees `delta` more tokens. Only the suffix
        groups' row records change, in place in the device table, so a
        captured graph replays the grown step unchanged; shared nodes are
        untouched. The forest's visible counts (and its index) are updated
        to match. Works for contiguous and paged pools (the group records
        carry their slice start within the node). Raises ValueError when a
        leaf has no room left (re-plan with new capacity)."""
        import torch

        i, blob = self.info, self.blob_host
        leaf = {n.id for n in self.forest.nodes[1:] if not self.forest.children[n.id]}
        touched, grown = [], {}
        for off, count in ((i.off_gemv, i.n_gemv_groups), (i.off_gen, i.n_gen_groups),
                           (i.off_multi, i.n_multi_groups),
                           (i.off_multi + 8 * i.n_multi_groups, i.n_tct_groups)):
            for gidx in range(count):
                rec = off + 8 * gidx
                node = int(blob[rec + 5])
                if node not in leaf:
                    continue
                start_tok = int(blob[rec + 6])  # slice start within the node
                for k in range(int(blob[rec + 3])):
                    r = i.off_rows + 4 * (int(blob[rec + 2]) + k)
                    req, vis = int(blob[r]), int(blob[r + 1])
                    if start_tok + vis != self.forest.visible_count(node, req):
                        continue  # not the request's last slice of this leaf
                    if vis + delta > int(blob[rec + 1]):
                        raise ValueError(f"leaf {node} has no room for {delta} more tokens: re-plan")
                    blob[r + 1] = vis + delta
                    blob[rec + 4] = max(int(blob[rec + 4]), vis + delta)
                    touched += [r + 1, rec + 4]
                    grown[(node, req)] = start_tok + vis + delta
        self._grown += delta
        if grown:
            self.forest.set_visible(grown)
        if touched:
            lo, hi = min(touched), max(touched) + 1
            self.table[lo:hi].copy_(torch.from_numpy(blob[lo:hi]))

    def with_budget(self, tc_sm_budget: int, plan=None, flags=None, timer=False) -> "DecodeStep":
        return DecodeStep(self.forest, self.plan if plan is None else plan, self.h_q, self.tdtype, self.head_begin,
                          self.head_end, self.device, self.flags if flags is None else flags, tc_sm_budget,
                          self.aux is not None, self.page_size, self.page_table, self.pool_tokens, timer)


def autotune_step(step: DecodeStep, q, k_pool, v_pool, budgets=None, iters=10):
    """Pick the tensor-core SM budget (the SMs left to the concurrent GEMV
    kernel) by timing one decode step per candidate with CUDA events --
    done once per plan, like a cuDNN benchmark-mode choice. Returns
    (best_step, {budget: ms})."""
    import torch

    if step.info.n_tc_groups == 0 or step.info.n_gemv_groups == 0:
        return step, {}
    sms = step.dims.sm_count
    h_local = step.head_end - step.head_begin
    budgets = budgets or sorted({sms} | {int(sms * f) // 2 * 2 for f in (0.9, 0.8, 0.7, 0.6, 0.5, 0.45)}, reverse=True)
    out = torch.empty((step.forest.bs, step.hq_local, step.d), dtype=step.out_dtype, device=step.device)
    times = {}
    best, best_ms = step, None
    for b in budgets:
        if b < h_local:
            continue
        cand = step.with_budget(b)
        for _ in range(3):
            cand(q, k_pool, v_pool, out=out)
        torch.cuda.synchronize(step.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            cand(q, k_pool, v_pool, out=out)
        e1.record()
        torch.cuda.synchronize(step.device)
        ms = e0.elapsed_time(e1) / iters
        times[b] = ms
        if best_ms is None or ms < best_ms:
            best, best_ms = cand, ms
    return best, times


def execute(forest: Forest, queries: QueryBatch, plan, pool: BlockPool | None = None, trace=None,
            reduce_mode: str = "balanced", flags: int = 0):
    """Full decode-attention step (executor.py:296-308) on the GPU.
    Returns a torch CUDA tensor [bs, h_q, d]."""
    import torch

    if queries.bs != forest.bs:
        raise DimensionMismatch(f"{queries.bs} queries for {forest.bs} requests")
    if queries.d != forest.d or queries.h_kv != forest.h_kv:
        raise DimensionMismatch(
            f"queries d={queries.d} h_kv={queries.h_kv} vs forest d={forest.d} h_kv={forest.h_kv}")
    if reduce_mode not in ("balanced", "sequential"):
        raise ValueError(f"mode must be balanced or sequential, got {reduce_mode!r}")
    q = queries.queries
    qdt = str(q.dtype).replace("torch.", "")
    tdt = torch_dtype(qdt if qdt in ("float32", "float64", "bfloat16") else "float64")
    dev = torch.device("cuda", torch.cuda.current_device())
    key = ("step", id(plan), str(tdt), int(flags), queries.h_q, str(dev))
    cache = forest._pools.setdefault("_steps", {})
    step = cache.get(key)
    if step is None or step[0] is not plan:
        step = (plan, DecodeStep(forest, plan, queries.h_q, tdt, flags=flags, device=dev))
        cache[key] = step
        while len(cache) > 4:  # bounded: each step holds its table and workspace
            cache.pop(next(iter(cache)))
    step = step[1]
    kp, vp = forest.device_pool(tdt)
    qd = (q if isinstance(q, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(q)))
    qd = qd.to(device=step.device, dtype=tdt).contiguous()
    return step(qd, kp, vp)


class PlanCache:
    """Plan reuse across decode steps: the plan
    and its device table are rebuilt every `replan_every` decode steps
    (DEFAULT_REPLAN_EVERY = 4, scheduler.py:23) or when the
    forest changes; in between, `advance()` grows every request's leaf by
    one token in place (DecodeStep.grow), so a captured graph keeps
    replaying. `planner(forest)` returns the DivisionPlan (default: the
    device plan over the profile `table`)."""

    def __init__(self, h_q: int, table=None, replan_every: int | None = None, planner=None, **step_kw):
        from .scheduler import DEFAULT_REPLAN_EVERY
        self.h_q = int(h_q)
        self.replan_every = int(replan_every or DEFAULT_REPLAN_EVERY)
        if self.replan_every < 1:
            raise ValueError(f"replan_every must be >= 1, got {self.replan_every}")
        self.table = table
        self.planner = planner
        self.step_kw = step_kw
        self.step = None
        self.age = 0        # decode steps served by the current plan
        self.replans = 0

    def _plan(self, forest):
        if self.planner is not None:
            return self.planner(forest)
        from .cost_model import load_default_profile
        from .scheduler import plan_device
        table = self.table if self.table is not None else load_default_profile()
        h_kv = forest.h_kv
        lo = self.step_kw.get("head_begin", 0)
        hi = self.step_kw.get("head_end", h_kv) or h_kv
        return plan_device(forest, self.h_q // h_kv, table, hi - lo, tc_sm_budget=self.step_kw.get("tc_sm_budget", 0))

    def get(self, forest) -> DecodeStep:
        """The step for this decode step: the cached one while the plan is
        young and the forest unchanged, else a re-plan."""
        if self.step is None or self.step.forest is not forest or self.age >= self.replan_every:
            self.step = DecodeStep(forest, self._plan(forest), self.h_q, **self.step_kw)
            self.age = 0
            self.replans += 1
        return self.step

    def advance(self, delta: int = 1) -> None:
        """After a decode step: every request gained `delta` tokens in its
        leaf (already written to the pool)."""
        if self.step is None:
            raise ValueError("no step yet: call get(forest) first")
        self.age += 1
        if self.age < self.replan_every:
            self.step.grow(delta)
        else:
            # re-plan at the next get(): the forest carries the grown counts
            self.step.forest.set_visible(
                {(n, r): self.step.forest.visible_count(n, r) + delta
                 for r, p in enumerate(self.step.forest.paths) for n in p[-1:]})
