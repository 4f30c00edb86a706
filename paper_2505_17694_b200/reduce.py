"""Per-request reduction of split partials (reference executor.py:73-117,
:209-293): the merge-schedule contract and reduce_tree() on the device.

`merge_schedule` / `sequential_schedule` return the reference's integer
combination order (computed by the library, codec_merge_schedule).
`reduce_tree(partials, forest, pool)` folds a PartialTree -- per (node,
slice) PartialResults with their request rows, what the reference's split
phase produces -- into [bs, h_q, d] with the library's one-pass LSE merge
(codec_merge_partials): M = max m, L = sum s e^(m - M), out = sum out s
e^(m - M) / L, equal to the pairwise por() fold up to rounding
(test_attention.py:160-180). The decode step itself never materialises a
PartialTree (its partials live in the task table's workspace and
kern_merge.cu folds them); this is the API-level entry point.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import IncompletePartials, NoVisibleTokens
from .forest import prefix_path


def _schedule(mode, path_len, counts):
    L = _lib.lib()
    cnt = np.ascontiguousarray(counts, dtype=np.int64) if counts is not None else np.zeros(1, np.int64)
    n_counts = len(counts) if counts is not None else 0
    npairs, nrounds = C.c_int64(), C.c_int64()
    P64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
    _lib.check(L.codec_merge_schedule(mode, int(path_len), P64(cnt), n_counts, None, None, 0, C.byref(npairs),
                                      C.byref(nrounds)))
    pairs = np.zeros(2 * max(npairs.value, 1), np.int64)
    ptr = np.zeros(nrounds.value + 1, np.int64)
    _lib.check(L.codec_merge_schedule(mode, int(path_len), P64(cnt), n_counts, P64(pairs), P64(ptr), npairs.value,
                                      C.byref(npairs), C.byref(nrounds)))
    return [[(int(pairs[2 * k]), int(pairs[2 * k + 1])) for k in range(ptr[i], ptr[i + 1])]
            for i in range(nrounds.value)]


def merge_schedule(path_len: int, slices_per_node) -> list:
    """Balanced binary combination schedule over one request's partials
    numbered in path-then-slice order (executor.py:86-111)."""
    counts = [int(x) for x in slices_per_node]
    return _schedule(0, path_len, counts)


def sequential_schedule(total: int) -> list:
    """Left fold: P-1 single-merge rounds (executor.py:114-117)."""
    return _schedule(1, total, None)


@dataclass
class PartialTree:
    """Split-phase partials (executor.py:73-82): entries[(node, slice)] is a
    PartialResult over the request rows rows[(node, slice)];
    slice_count[node] = subtasks of the node."""

    entries: dict = field(default_factory=dict)
    rows: dict = field(default_factory=dict)
    slice_count: dict = field(default_factory=dict)


def reduce_tree(partials: PartialTree, forest, pool=None, trace=None, t0: float = 0.0,
                mode: str = "balanced"):
    """Merge each request's partials (path-then-slice order, like
    _reduce_one, executor.py:209-231) and finalize; returns a torch CUDA
    tensor [bs, h_q, d]. The reference's simulated merge trace is out of
    scope (trace must be None)."""
    import torch

    if mode not in ("balanced", "sequential"):
        raise ValueError(f"mode must be balanced or sequential, got {mode!r}")
    if trace is not None:
        raise ValueError("the simulated EventTrace is not produced on the GPU")
    some = next(iter(partials.entries.values()), None)
    if some is None:
        raise IncompletePartials("partial tree is empty")
    keys = list(partials.entries)
    index = {k: i for i, k in enumerate(keys)}
    # every entry's rows become slots: slot = row offset of the entry + row
    base, total = {}, 0
    for k in keys:
        base[k] = total
        total += partials.entries[k].out.shape[0]
    ptr, slots = [0], []
    for r in range(forest.bs):
        units = []
        for nid in prefix_path(forest, r):
            cnt = partials.slice_count.get(nid)
            if cnt is None:
                raise IncompletePartials(f"no subtasks recorded for node {nid}")
            for si in range(cnt):
                key = (nid, si)
                rows = partials.rows.get(key)
                if rows is not None and r in rows:
                    if key not in index:
                        raise IncompletePartials(f"partial {key} missing for request {r}")
                    units.append(base[key] + list(rows).index(r))
        if not units:
            raise NoVisibleTokens(f"request {r} has no visible tokens anywhere on its path")
        slots += units
        ptr.append(len(slots))
    dev = torch.device("cuda", torch.cuda.current_device())
    cat = lambda name: torch.cat([torch.as_tensor(getattr(partials.entries[k], name)).to(dev) for k in keys])
    po, pm, ps = cat("out"), cat("max_score"), cat("exp_sum")
    dt = po.dtype
    if dt not in (torch.float32, torch.float64):
        raise ValueError(f"partials must be float32 or float64, got {dt}")
    pm, ps = pm.to(dt).contiguous(), ps.to(dt).contiguous()
    po = po.contiguous()
    h_q, d = int(po.shape[1]), int(po.shape[2])
    ptr_d = torch.tensor(ptr, dtype=torch.int32, device=dev)
    slot_d = torch.tensor(slots, dtype=torch.int32, device=dev)
    out = torch.empty((forest.bs, h_q, d), dtype=dt, device=dev)
    out_s = torch.empty((forest.bs, h_q), dtype=dt, device=dev)
    _lib.check(_lib.lib().codec_merge_partials(
        1 if dt == torch.float64 else 0, forest.bs, h_q, d, C.c_void_p(ptr_d.data_ptr()),
        C.c_void_p(slot_d.data_ptr()), C.c_void_p(po.data_ptr()), C.c_void_p(pm.data_ptr()),
        C.c_void_p(ps.data_ptr()), C.c_void_p(out.data_ptr()), C.c_void_p(out_s.data_ptr()),
        C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    if bool((out_s <= 0).any()):
        raise NoVisibleTokens("some (query, head) saw no visible tokens")
    return out
