"""Split-attention primitives on the GPU (reference-compatible API).

`pac`, `por`, `empty_partial`, `finalize` and `PartialResult` keep the
signatures and semantics of prefixdec/attention.py:46-161, but compute on
the B200 through the C ABI (codec_pac / codec_por in the shared
library). Inputs may be numpy arrays or torch tensors (host or device);
results are torch CUDA tensors: float64 for float64 inputs, float32 for
float32 and bfloat16 inputs (fp32 accumulation).

There is no backend switch and no CPU path: without a CUDA device or the
built library these functions raise.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch, EmptyVisibleSet, NoVisibleTokens, ShapeMismatch


def torch_dtype(dt):
    import torch

    s = str(dt).replace("torch.", "")
    return {"float32": torch.float32, "float64": torch.float64, "bfloat16": torch.bfloat16}[s]


def _code(t) -> int:
    return {"torch.float32": 0, "torch.float64": 1, "torch.bfloat16": 2}[str(t.dtype)]


def _dev(x, device="cuda", dtype=None):
    import torch

    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.asarray(x)
        if a.dtype == np.float16 or a.dtype.kind not in "f":
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device).contiguous()


def _stream(t):
    import torch

    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


@dataclass
class PartialResult:
    """(normalised out [n_q,h_q,d], running max [n_q,h_q], exp-sum [n_q,h_q]);
    s = 0 with m = -inf marks an empty entry (attention.py:46-65)."""

    out: object
    max_score: object
    exp_sum: object

    @property
    def n_q(self) -> int:
        return int(self.out.shape[0])

    def copy(self) -> "PartialResult":
        return PartialResult(self.out.clone(), self.max_score.clone(), self.exp_sum.clone())

    def row(self, i: int) -> "PartialResult":
        return PartialResult(self.out[i:i + 1], self.max_score[i:i + 1], self.exp_sum[i:i + 1])


def pac(queries, keys, values, visible=None) -> PartialResult:
    """Partial attention of queries [n_q,h_q,d] over one KV chunk
    [n,h_kv,d]; score q.k/sqrt(d) over tokens j < visible[i]; query head h
    reads kv head h // g (attention.py:88-117). Runs codec_pac."""
    import torch

    q = _dev(queries)
    k = _dev(keys, dtype=q.dtype)
    v = _dev(values, dtype=q.dtype)
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3 or k.shape != v.shape:
        raise DimensionMismatch(
            f"expected q [n_q,h_q,d], k/v [n,h_kv,d]; got {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    if q.shape[2] != k.shape[2]:
        raise DimensionMismatch(f"head dim mismatch: q d={q.shape[2]}, k d={k.shape[2]}")
    if k.shape[0] < 1 or q.shape[0] < 1:
        raise DimensionMismatch("need n >= 1 tokens and n_q >= 1 queries")
    if k.shape[1] < 1 or q.shape[1] % k.shape[1] != 0:
        raise DimensionMismatch(f"h_q={q.shape[1]} not a multiple of h_kv={k.shape[1]}")
    n_q, h_q, d = (int(s) for s in q.shape)
    n, h_kv = int(k.shape[0]), int(k.shape[1])
    vis_t = None
    if visible is not None:
        vis = np.asarray(visible.cpu() if hasattr(visible, "cpu") else visible, dtype=np.int64).reshape(n_q)
        if (vis < 1).any() or (vis > n).any():
            raise EmptyVisibleSet(f"visible counts must lie in 1..{n}, got {vis.tolist()}")
        vis_t = torch.from_numpy(vis).to(q.device)
    odt = torch.float64 if q.dtype == torch.float64 else torch.float32
    out = torch.empty((n_q, h_q, d), dtype=odt, device=q.device)
    m = torch.empty((n_q, h_q), dtype=odt, device=q.device)
    s = torch.empty((n_q, h_q), dtype=odt, device=q.device)
    scale = 1.0 / math.sqrt(d)
    _lib.check(_lib.lib().codec_pac(
        _code(q), C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
        C.c_void_p(vis_t.data_ptr()) if vis_t is not None else None, n_q, h_q, n, h_kv, d, scale,
        C.c_void_p(out.data_ptr()), C.c_void_p(m.data_ptr()), C.c_void_p(s.data_ptr()), _stream(q)))
    return PartialResult(out, m, s)


def empty_partial(n_q: int, h_q: int, d: int, dtype=np.float64, device="cuda") -> PartialResult:
    """Neutral element of por (attention.py:120-128)."""
    import torch

    if n_q < 1 or h_q < 1 or d < 1:
        raise DimensionMismatch(f"dimensions must be positive, got ({n_q}, {h_q}, {d})")
    tdt = torch_dtype(np.dtype(dtype).name if not str(dtype).startswith("torch") else dtype)
    return PartialResult(torch.zeros((n_q, h_q, d), dtype=tdt, device=device),
                         torch.full((n_q, h_q), float("-inf"), dtype=tdt, device=device),
                         torch.zeros((n_q, h_q), dtype=tdt, device=device))


def por(a: PartialResult, b: PartialResult) -> PartialResult:
    """LSE merge of two partials; a wholly empty side returns the other
    unchanged, empty entries merge elementwise (attention.py:131-153).
    Elementwise math runs in codec_por."""
    import torch

    if tuple(a.out.shape) != tuple(b.out.shape) or tuple(a.max_score.shape) != tuple(b.max_score.shape):
        raise ShapeMismatch(f"partial shapes differ: {tuple(a.out.shape)} vs {tuple(b.out.shape)}")
    if not bool(b.exp_sum.any()):
        return a.copy()
    if not bool(a.exp_sum.any()):
        return b.copy()
    ao, am, as_ = (_dev(x) for x in (a.out, a.max_score, a.exp_sum))
    bo, bm, bs = (_dev(x, dtype=ao.dtype) for x in (b.out, b.max_score, b.exp_sum))
    ro, rm, rs = torch.empty_like(ao), torch.empty_like(am), torch.empty_like(as_)
    count = int(am.numel())
    d = int(ao.shape[-1])
    _lib.check(_lib.lib().codec_por(
        _code(ao), count, d, *(C.c_void_p(t.data_ptr()) for t in (ao, am, as_, bo, bm, bs, ro, rm, rs)),
        _stream(ao)))
    return PartialResult(ro, rm, rs)


def finalize(p: PartialResult):
    """The output tensor; NoVisibleTokens if any entry is empty
    (attention.py:156-161)."""
    if bool((p.exp_sum <= 0).any()):
        raise NoVisibleTokens("some (query, head) saw no visible tokens")
    return p.out.clone()
