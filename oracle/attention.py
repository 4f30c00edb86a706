"""Oracle: split-attention partials (PAC), their log-sum-exp merge (POR),
the split/merge executor and the single-softmax reference.

Restates reference prefixdec/attention.py, prefixdec/_kernels_py.py and
prefixdec/executor.py in numpy. Partials use the reference convention:
`out` already normalised by the exp-sum `s`, `m` the running max, and
(m=-inf, s=0) marks an empty entry.
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .index import preorder_offsets, children_lists, query_sets, visible_count

CHUNK = 2048  # token chunk of the streaming pass (_kernels_py.py:13)


def pac(q, k, v, visible=None):
    """Partial attention of q [n_q,h_q,d] over one KV chunk k/v [n,h_kv,d]
    with per-query visible prefix counts; score scale 1/sqrt(d); q head h
    reads kv head h // (h_q/h_kv). Streams ascending token chunks with an
    online softmax in the storage dtype (_kernels_py.py:16-52,
    attention.py:88-117). Returns (out, m, s)."""
    n_q, h_q, d = q.shape
    n, h_kv, _ = k.shape
    g = h_q // h_kv
    dt = q.dtype
    vis = np.full(n_q, n, dtype=np.int64) if visible is None else np.asarray(visible, np.int64)
    scale = dt.type(1.0 / math.sqrt(d))
    qg = q.reshape(n_q, h_kv, g, d)
    m = np.full((n_q, h_kv, g), -np.inf, dtype=dt)
    s = np.zeros((n_q, h_kv, g), dtype=dt)
    acc = np.zeros((n_q, h_kv, g, d), dtype=dt)
    stop_all = int(vis.max())
    for lo in range(0, stop_all, CHUNK):
        hi = min(lo + CHUNK, stop_all)
        sc = np.einsum("akgd,ckd->akgc", qg, k[lo:hi]) * scale
        dead = np.arange(lo, hi)[None, :] >= vis[:, None]
        sc[np.broadcast_to(dead[:, None, None, :], sc.shape)] = -np.inf
        new_m = np.maximum(m, sc.max(axis=3))
        p = np.exp(sc - new_m[..., None])
        rescale = np.exp(m - new_m)
        s = s * rescale + p.sum(axis=3)
        acc = acc * rescale[..., None] + np.einsum("akgc,ckd->akgd", p, v[lo:hi])
        m = new_m
    out = acc / s[..., None]
    return out.reshape(n_q, h_q, d), m.reshape(n_q, h_q), s.reshape(n_q, h_q)


def empty(n_q, h_q, d, dtype=np.float64):
    """Neutral element of por (attention.py:120-128)."""
    return (np.zeros((n_q, h_q, d), dtype), np.full((n_q, h_q), -np.inf, dtype),
            np.zeros((n_q, h_q), dtype))


def por(a, b):
    """Merge two partials in a common max frame; a wholly empty side
    returns the other unchanged, empty entries merge elementwise
    (attention.py:131-153)."""
    ao, am, as_ = a
    bo, bm, bs = b
    if not bs.any():
        return ao.copy(), am.copy(), as_.copy()
    if not as_.any():
        return bo.copy(), bm.copy(), bs.copy()
    m = np.maximum(am, bm)
    with np.errstate(invalid="ignore"):
        wa = np.where(as_ > 0, as_ * np.exp(am - m), 0.0)
        wb = np.where(bs > 0, bs * np.exp(bm - m), 0.0)
    s = wa + wb
    den = np.where(s > 0, s, 1.0)
    out = np.where(s[..., None] > 0, (ao * wa[..., None] + bo * wb[..., None]) / den[..., None], 0.0)
    m = np.where(s > 0, m, -np.inf)
    dt = ao.dtype
    return out.astype(dt, copy=False), m.astype(dt, copy=False), s.astype(dt, copy=False)


def merge_rounds(counts):
    """Balanced adjacent pairing over P = sum(counts) partials in
    path-then-slice order; ceil(log2 P) rounds (executor.py:86-111)."""
    live = list(range(sum(counts)))
    rounds = []
    while len(live) > 1:
        pairs = [(live[i], live[i + 1]) for i in range(0, len(live) - 1, 2)]
        keep = live[0::2]
        rounds.append(pairs)
        live = keep
    return rounds


class ForestData:
    """Minimal forest container for the oracle: node tensors plus the
    structural description used by oracle.index."""

    def __init__(self, parent, keys, values, paths, visible=None):
        self.parent = list(parent)          # parent[0] = 0 (virtual root)
        self.keys = list(keys)              # keys[0] is an empty [0,h_kv,d]
        self.values = list(values)
        self.paths = [tuple(p) for p in paths]
        self.visible = visible if visible is not None else [None] * len(self.parent)
        self.length = [int(k.shape[0]) for k in self.keys]
        self.qsets = query_sets(self.paths, len(self.length))
        self.offsets = preorder_offsets(self.length, children_lists(self.parent, len(self.length)))

    @property
    def bs(self):
        return len(self.paths)

    def vis(self, nid, rid):
        return visible_count(self.length, self.visible, nid, rid)


def naive_attention(queries, fd: ForestData):
    """One shift-stabilised softmax per request over the concatenated
    visible path (attention.py:164-187)."""
    bs, h_q, d = queries.shape
    h_kv = fd.keys[1].shape[1]
    kv_of = np.arange(h_q) // (h_q // h_kv)
    out = np.zeros((bs, h_q, d), dtype=queries.dtype)
    scale = 1.0 / math.sqrt(d)
    for r in range(bs):
        ks = [fd.keys[n][: fd.vis(n, r)] for n in fd.paths[r]]
        vs = [fd.values[n][: fd.vis(n, r)] for n in fd.paths[r]]
        k = np.concatenate(ks)[:, kv_of, :]
        v = np.concatenate(vs)[:, kv_of, :]
        sc = np.einsum("hd,lhd->hl", queries[r], k) * scale
        w = np.exp(sc - sc.max(axis=1, keepdims=True))
        out[r] = np.einsum("hl,lhd->hd", w, v) / w.sum(axis=1)[:, None]
    return out


def execute(fd: ForestData, queries, subtasks, workers=1):
    """Split phase over plan subtasks (rows with visible > start,
    per-row visible clipped to the slice), then per-request balanced
    merge in path-then-slice order and finalize
    (executor.py:145-206, :209-264, :296-308).

    subtasks: sequence of (node, start, stop) in plan order."""
    slice_no = {}
    jobs = []
    for node, start, stop in subtasks:
        si = slice_no.get(node, 0)
        slice_no[node] = si + 1
        rows = tuple(r for r in fd.qsets[node] if fd.vis(node, r) > start)
        jobs.append(((node, si), rows, start, stop))

    def run(job):
        key, rows, start, stop = job
        if not rows:
            return key, rows, None
        vis = np.array([min(fd.vis(key[0], r), stop) - start for r in rows], dtype=np.int64)
        part = pac(queries[list(rows)], fd.keys[key[0]][start:stop],
                   fd.values[key[0]][start:stop], vis)
        return key, rows, part

    if workers > 1:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            results = list(ex.map(run, jobs))
    else:
        results = [run(j) for j in jobs]
    parts = {key: (rows, p) for key, rows, p in results if p is not None}

    bs, h_q, d = queries.shape
    out = np.zeros((bs, h_q, d), dtype=queries.dtype)
    for r in range(bs):
        units, counts = [], []
        for node in fd.paths[r]:
            c = 0
            for si in range(slice_no[node]):
                got = parts.get((node, si))
                if got is not None and r in got[0]:
                    i = got[0].index(r)
                    p = got[1]
                    units.append((p[0][i:i + 1], p[1][i:i + 1], p[2][i:i + 1]))
                    c += 1
            counts.append(c)
        acc = dict(enumerate(units))
        for rnd in merge_rounds(counts):
            for i, j in rnd:
                acc[i] = por(acc[i], acc[j])
        if (acc[0][2] <= 0).any():
            raise ValueError(f"request {r} saw no visible tokens")
        out[r] = acc[0][0][0]
    return out
