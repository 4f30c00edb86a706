"""The reference-side binding INTEGRATION.md §2 describes, runnable.

A maintainer of the reference (`prefixdec`) plugs the B200 path in at its
two boundaries:

* the kernel: `prefixdec._kernels.pac_kernel(q, k, v, visible, scale, out,
  max_score, exp_sum)` (_kernels.pyx:16-18), which
  attention._run_pac_kernel (attention.py:68-85) calls for every pac(),
  becomes a ctypes call of `codec_pac` (include/codec_b200.h) -- this
  module binds the shared library itself, with nothing from the
  paper_2505_17694_b200 package on that path;
* the operator: `prefixdec.execute(forest, queries, plan, pool)`
  (executor.py:296-308) becomes one decode step of the B200 package
  (index + device task table + codec_decode_attention), the reference's
  Forest / DivisionPlan translated at the boundary.

`install(mode)` patches an imported prefixdec in place ("kernel" or
"execute"); `integration/plugin.py` does it for pytest so the reference's
own test files run against the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB = Path(os.environ.get("CODEC_B200_LIB",
                          Path(__file__).resolve().parent.parent / "paper_2505_17694_b200" / "_codec_b200.so"))
_DT = {np.dtype("float32"): 0, np.dtype("float64"): 1}
_lib = None
CALLS = {"pac_kernel": 0, "execute": 0}


def lib():
    global _lib
    if _lib is None:
        h = C.CDLL(str(LIB))
        h.codec_pac.restype = C.c_int32
        h.codec_pac.argtypes = [C.c_int32] + [C.c_void_p] * 4 + [C.c_int64] * 5 + [C.c_double] + [C.c_void_p] * 4
        h.codec_last_error.restype = C.c_char_p
        _lib = h
    return _lib


def pac_kernel(q, k, v, visible, scale, out, max_score, exp_sum):
    """Same contract as prefixdec._kernels.pac_kernel: C-contiguous q
    [n_q,h_q,d], k/v [n,h_kv,d] (float32 or float64), visible int64 [n_q],
    scale = 1/sqrt(d); outputs preallocated by the caller in q's dtype."""
    import torch
    CALLS["pac_kernel"] += 1
    if q.dtype not in _DT:
        raise TypeError(f"unsupported dtype {q.dtype}")
    dq, dk, dv = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (q, k, v))
    dvis = torch.from_numpy(np.ascontiguousarray(visible, dtype=np.int64)).cuda()
    o = torch.empty_like(dq)
    m = torch.empty(q.shape[:2], dtype=dq.dtype, device="cuda")
    s = torch.empty_like(m)
    st = lib().codec_pac(_DT[q.dtype], dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), dvis.data_ptr(),
                         q.shape[0], q.shape[1], k.shape[0], k.shape[1], q.shape[2], float(scale),
                         o.data_ptr(), m.data_ptr(), s.data_ptr(), torch.cuda.current_stream().cuda_stream)
    if st:
        raise RuntimeError(lib().codec_last_error().decode())
    out[...] = o.cpu().numpy()
    max_score[...] = m.cpu().numpy()
    exp_sum[...] = s.cpu().numpy()


class _KernelModule:
    """Stands in for the compiled `prefixdec._kernels` module."""
    pac_kernel = staticmethod(pac_kernel)


def _to_b200_forest(forest, queries):
    import paper_2505_17694_b200 as B
    specs = [(n.parent, n.keys, n.values, n.visible_len) for n in forest.nodes[1:]]
    return B.build_forest(specs, forest.paths, B.QueryBatch(np.asarray(queries.queries), queries.h_kv))


def make_execute(ref_execute, errors):
    """execute() replacement: the whole decode step on the GPU. The
    reference's simulated EventTrace has no GPU counterpart (CUDA events /
    ncu replace simulated time), so trace= keeps the reference's own
    host path and is counted separately."""
    def execute(forest, queries, plan, pool, trace=None, reduce_mode="balanced"):
        import paper_2505_17694_b200 as B
        if trace is not None:
            return ref_execute(forest, queries, plan, pool, trace=trace, reduce_mode=reduce_mode)
        CALLS["execute"] += 1
        # the reference's own argument checks first (executor.py:301-306)
        if queries.bs != forest.bs:
            raise errors.DimensionMismatch(f"{queries.bs} queries for {forest.bs} requests")
        if queries.d != forest.d or queries.h_kv != forest.h_kv:
            raise errors.DimensionMismatch(
                f"queries d={queries.d} h_kv={queries.h_kv} vs forest d={forest.d} h_kv={forest.h_kv}")
        if reduce_mode not in ("balanced", "sequential"):
            raise ValueError(f"mode must be balanced or sequential, got {reduce_mode!r}")
        f = _to_b200_forest(forest, queries)
        q = B.QueryBatch(np.asarray(queries.queries), queries.h_kv)
        try:
            out = B.execute(f, q, plan, B.BlockPool(pool.worker_count))
        except B.PrefixDecError as e:  # same class names, the reference's classes
            raise getattr(errors, type(e).__name__)(str(e)) from None
        return out.cpu().numpy().astype(np.asarray(queries.queries).dtype, copy=False)
    return execute


def install(mode: str = "kernel"):
    """Patch the imported prefixdec: mode "kernel" swaps the compiled
    kernel module for codec_pac; "execute" also swaps execute()."""
    import prefixdec
    import prefixdec.attention as A
    import prefixdec.errors as E
    import prefixdec.executor as X
    A._kernels = _KernelModule
    if mode == "execute":
        ex = make_execute(X.execute, E)
        X.execute = ex
        prefixdec.execute = ex
    elif mode != "kernel":
        raise ValueError(f"mode must be kernel or execute, got {mode!r}")
