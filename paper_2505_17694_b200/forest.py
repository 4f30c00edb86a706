"""Tree-of-tensors KV cache: the prefix forest (K0 on the host, KV pool on
the device).

API-compatible with the reference's prefixdec/forest.py: `QueryBatch`,
`KvNode`, `Forest`, `build_forest(node_specs, request_paths, queries)`,
`prefix_path`, `node_query_set`, `validate`. Node ids are 1..N in spec
order under a virtual root 0; each request's path is a parent->child
chain; query sets are ascending; nodes are flattened in preorder
(kappa, forest.py:148-157).

B200 specifics:
  * the integer index (query-set CSR, preorder offsets, visible counts)
    is built by the C++ indexer of the shared library
    (csrc/host_index.cpp) -- the same arrays the device task table is
    expanded from;
  * the KV tensors live on the GPU as one head-major pool per K and V,
    [h_kv][T][d] with node n at tokens [kappa(n), kappa(n)+len), so a
    node slice of one head is a single contiguous run for TMA.
    `Forest.device_pool()` packs host node tensors into it once;
    `forest_from_pool()` adopts a pool already resident in HBM.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import (
    CycleDetected,
    DanglingParent,
    DimensionMismatch,
    PathNotPrefixChain,
    UnknownNode,
    UnknownRequest,
)

ROOT = 0


def _shape(x):
    return tuple(int(s) for s in x.shape)


def _dtype_name(x):
    return str(x.dtype).replace("torch.", "")


@dataclass(frozen=True)
class QueryBatch:
    """One decode-step query row per request, [bs, h_q, d] (numpy or torch),
    plus the kv head count for grouped-query mapping (forest.py:29-65)."""

    queries: object
    h_kv: int

    def __post_init__(self):
        q = self.queries
        if not hasattr(q, "shape"):
            q = np.asarray(q)
        if len(q.shape) != 3:
            raise DimensionMismatch(f"queries must be [bs, h_q, d], got shape {tuple(q.shape)}")
        if self.h_kv < 1 or q.shape[1] % self.h_kv != 0:
            raise DimensionMismatch(f"h_q={q.shape[1]} must be a positive multiple of h_kv={self.h_kv}")
        object.__setattr__(self, "queries", q)

    @property
    def bs(self) -> int:
        return int(self.queries.shape[0])

    @property
    def h_q(self) -> int:
        return int(self.queries.shape[1])

    @property
    def d(self) -> int:
        return int(self.queries.shape[2])

    @property
    def group_size(self) -> int:
        return self.h_q // self.h_kv

    @property
    def dtype(self):
        return self.queries.dtype


@dataclass
class KvNode:
    """A node: a run of tokens, K/V [len, h_kv, d] (None when the forest
    adopted a device pool), ascending query set, optional visible_len
    (forest.py:68-85)."""

    id: int
    parent: int
    keys: object
    values: object
    query_set: tuple = ()
    visible_len: dict | None = None
    length: int = 0

    @property
    def len(self) -> int:
        return self.length


@dataclass(frozen=True)
class Violation:
    code: str
    message: str
    node: int | None = None
    request: int | None = None


@dataclass
class Forest:
    nodes: list
    children: list
    paths: list
    h_kv: int
    d: int
    token_offset: list = field(default_factory=list)
    kv_dtype: str = "float64"
    _index: object = None          # codec_index* (owned)
    _pools: dict = field(default_factory=dict)

    def __del__(self):
        if self._index:
            try:
                _lib.lib().codec_index_free(self._index)
            except Exception:
                pass
            self._index = None

    @property
    def bs(self) -> int:
        return len(self.paths)

    @property
    def total_tokens(self) -> int:
        return sum(n.len for n in self.nodes)

    @property
    def dtype(self):
        return self.kv_dtype

    def node(self, node_id: int) -> KvNode:
        if not 0 <= node_id < len(self.nodes):
            raise UnknownNode(f"no node {node_id}")
        return self.nodes[node_id]

    def non_root_ids(self) -> list:
        return [n.id for n in self.nodes[1:]]

    def visible_count(self, node_id: int, request: int) -> int:
        node = self.node(node_id)
        if node.visible_len and request in node.visible_len:
            return node.visible_len[request]
        return node.len

    def request_len(self, request: int) -> int:
        return sum(self.visible_count(n, request) for n in prefix_path(self, request))

    def flatten_index(self, node_id: int, local: int) -> int:
        """1-based global token index under preorder flattening
        (forest.py:139-145)."""
        node = self.node(node_id)
        if node_id == ROOT or not 0 <= local < node.len:
            raise UnknownNode(f"token {local} not in node {node_id}")
        return self.token_offset[node_id] + local + 1

    # ---------------------------------------------------------- device pool
    def device_pool(self, dtype=None, device="cuda", head_begin=0, head_end=None):
        """(K, V) head-major pools [h_local][T][d] on `device`, packed from
        the host node tensors once and cached (heads [head_begin,
        head_end) only, for kv-head sharding)."""
        import torch

        from .attention import torch_dtype

        head_end = self.h_kv if head_end is None else head_end
        tdt = torch_dtype(dtype if dtype is not None else self.kv_dtype)
        key = (str(tdt), str(device), head_begin, head_end)
        if key in self._pools:
            return self._pools[key]
        if any(n.keys is None for n in self.nodes[1:]):
            raise DimensionMismatch("forest has no host tensors; adopt a device pool with forest_from_pool")
        h_local = head_end - head_begin
        T = self.total_tokens
        kp = torch.zeros((h_local, max(T, 1), self.d), dtype=tdt, device=device)
        vp = torch.zeros_like(kp)
        stream = torch.cuda.current_stream(kp.device).cuda_stream
        code = dtype_code(tdt)
        L = _lib.lib()
        for n in self.nodes[1:]:
            for src, pool in ((n.keys, kp), (n.values, vp)):
                t = torch.as_tensor(src).to(device=device, dtype=tdt).contiguous()
                _lib.check(L.codec_pool_pack(code, C.c_void_p(t.data_ptr()), n.len, self.h_kv, self.d, head_begin,
                                             h_local, C.c_void_p(pool.data_ptr()), max(T, 1),
                                             self.token_offset[n.id], C.c_void_p(stream)))
        self._pools[key] = (kp, vp)
        return kp, vp

    def set_visible(self, updates: dict) -> None:
        """Set visible_len[request] of nodes ({(node, request): count}, each
        count in 1..len) -- decode-step growth of partially filled leaves --
        and rebuild the integer index to match."""
        for (nid, rid), cnt in updates.items():
            node = self.node(nid)
            if rid not in node.query_set:
                raise UnknownRequest(f"request {rid} does not run through node {nid}")
            if not 1 <= cnt <= node.len:
                raise ValueError(f"node {nid} visible_len[{rid}]={cnt} outside 1..{node.len}")
            if node.visible_len is None:
                node.visible_len = {}
            node.visible_len[rid] = int(cnt)
        old = self._index
        self._index = _index_build([n.parent for n in self.nodes], [n.len for n in self.nodes], self.paths,
                                   [n.visible_len if n.id else None for n in self.nodes], self.bs)[0]
        if old:
            _lib.lib().codec_index_free(old)

    def adopt_pool(self, k_pool, v_pool, head_begin=0, head_end=None):
        head_end = self.h_kv if head_end is None else head_end
        key = (str(k_pool.dtype), str(k_pool.device), head_begin, head_end)
        self._pools[key] = (k_pool, v_pool)


def dtype_code(dt) -> int:
    s = str(dt).replace("torch.", "")
    return {"float32": 0, "float64": 1, "bfloat16": 2}[s]


def _index_build(parent, length, paths, visible, bs):
    n_nodes = len(parent)
    par = np.ascontiguousarray(parent, dtype=np.int32)
    ln = np.ascontiguousarray(length, dtype=np.int64)
    pptr = np.zeros(bs + 1, dtype=np.int64)
    for r, p in enumerate(paths):
        pptr[r + 1] = pptr[r] + len(p)
    pidx = np.ascontiguousarray([x for p in paths for x in p], dtype=np.int32)
    vn, vr, vc = [], [], []
    for nid, vis in enumerate(visible):
        if vis:
            for rid, cnt in vis.items():
                vn.append(nid)
                vr.append(int(rid))
                vc.append(int(cnt))
    vn = np.ascontiguousarray(vn, dtype=np.int32)
    vr = np.ascontiguousarray(vr, dtype=np.int32)
    vc = np.ascontiguousarray(vc, dtype=np.int64)
    h = C.c_void_p()
    L = _lib.lib()
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    _lib.check(L.codec_index_build(n_nodes, P(par, C.c_int32), P(ln, C.c_int64), bs, P(pptr, C.c_int64),
                                   P(pidx, C.c_int32), len(vn), P(vn, C.c_int32), P(vr, C.c_int32),
                                   P(vc, C.c_int64), C.byref(h)))
    info = _lib.IndexInfo()
    _lib.check(L.codec_index_info_get(h, C.byref(info)))
    off = np.zeros(n_nodes, np.int64)
    qptr = np.zeros(n_nodes + 1, np.int64)
    qidx = np.zeros(max(info.qset_nnz, 1), np.int32)
    cptr = np.zeros(n_nodes + 1, np.int64)
    cidx = np.zeros(max(n_nodes - 1, 1), np.int32)
    _lib.check(L.codec_index_read(h, P(off, C.c_int64), P(qptr, C.c_int64), P(qidx, C.c_int32), None,
                                  P(cptr, C.c_int64), P(cidx, C.c_int32)))
    return h, off, qptr, qidx, cptr, cidx


def _assemble(parent, length, keys, values, visible, paths, h_kv, d, kv_dtype):
    paths = [tuple(int(x) for x in p) for p in paths]
    for rid, p in enumerate(paths):
        if not p:
            raise PathNotPrefixChain(f"request {rid} has an empty path")
    h, off, qptr, qidx, cptr, cidx = _index_build(parent, length, paths, visible, len(paths))
    nodes = []
    for nid in range(len(parent)):
        qs = tuple(int(x) for x in qidx[qptr[nid]:qptr[nid + 1]]) if nid else ()
        nodes.append(KvNode(nid, int(parent[nid]), keys[nid], values[nid], qs,
                            visible[nid] if nid else None, int(length[nid])))
    children = [[int(x) for x in cidx[cptr[i]:cptr[i + 1]]] for i in range(len(parent))]
    return Forest(nodes=nodes, children=children, paths=paths, h_kv=h_kv, d=d,
                  token_offset=[int(x) for x in off], kv_dtype=kv_dtype, _index=h)


def build_forest(node_specs, request_paths, queries: QueryBatch | None = None) -> Forest:
    """Assemble a forest from (parent, keys, values[, visible_len]) specs
    and per-request node paths (forest.py:160-251); same checks, same
    exception classes and messages."""
    if not node_specs:
        raise DimensionMismatch("forest needs at least one node")
    k0 = node_specs[0][1]
    if not hasattr(k0, "shape"):
        k0 = np.asarray(k0)
    if len(k0.shape) != 3:
        raise DimensionMismatch(f"keys must be [len, h_kv, d], got shape {_shape(k0)}")
    h_kv, d = int(k0.shape[1]), int(k0.shape[2])
    dtype = _dtype_name(k0)
    parent, length, keys, values, visible = [0], [0], [None], [None], [None]
    for spec in node_specs:
        p, k, v = spec[0], spec[1], spec[2]
        vis = spec[3] if len(spec) > 3 else None
        if not hasattr(k, "shape"):
            k = np.asarray(k)
        if not hasattr(v, "shape"):
            v = np.asarray(v)
        nid = len(parent)
        if p == nid:
            raise CycleDetected(f"node {nid} is its own parent")
        if not 0 <= p < nid:
            raise DanglingParent(f"node {nid} references undeclared parent {p}")
        if _shape(k) != _shape(v) or len(k.shape) != 3:
            raise DimensionMismatch(f"node {nid}: keys {_shape(k)} and values {_shape(v)} must be equal 3-d shapes")
        if _shape(k)[1:] != (h_kv, d) or _dtype_name(k) != dtype:
            raise DimensionMismatch(f"node {nid}: expected [*, {h_kv}, {d}] {dtype}, got {_shape(k)} {_dtype_name(k)}")
        if k.shape[0] < 1:
            raise DimensionMismatch(f"node {nid} has no tokens")
        parent.append(int(p))
        length.append(int(k.shape[0]))
        keys.append(k)
        values.append(v)
        visible.append(dict(vis) if vis else None)
    if queries is not None:
        if queries.bs != len(request_paths):
            raise DimensionMismatch(f"{queries.bs} query rows for {len(request_paths)} request paths")
        if queries.d != d or queries.h_kv != h_kv:
            raise DimensionMismatch(f"queries d={queries.d} h_kv={queries.h_kv} vs forest d={d} h_kv={h_kv}")
    return _assemble(parent, length, keys, values, visible, request_paths, h_kv, d, dtype)


def forest_from_pool(parent, lengths, request_paths, h_kv, d, k_pool=None, v_pool=None, visible=None,
                     kv_dtype="bfloat16") -> Forest:
    """Forest over KV already resident in HBM: `parent[i]`/`lengths[i]` for
    nodes 1..N (index 0 = virtual root), the pools [h_kv][T][d] laid out
    at the preorder offsets this function returns in forest.token_offset.
    Pools may be attached later with Forest.adopt_pool()."""
    parent = [0] + [int(p) for p in parent]
    length = [0] + [int(x) for x in lengths]
    n = len(parent)
    for nid in range(1, n):
        if parent[nid] == nid:
            raise CycleDetected(f"node {nid} is its own parent")
        if not 0 <= parent[nid] < nid:
            raise DanglingParent(f"node {nid} references undeclared parent {parent[nid]}")
        if length[nid] < 1:
            raise DimensionMismatch(f"node {nid} has no tokens")
    vis = [None] * n if visible is None else [None] + [dict(v) if v else None for v in visible]
    f = _assemble(parent, length, [None] * n, [None] * n, vis, request_paths, h_kv, d, kv_dtype)
    if k_pool is not None:
        f.adopt_pool(k_pool, v_pool)
    return f


def prefix_path(forest: Forest, request: int) -> tuple:
    if not 0 <= request < forest.bs:
        raise UnknownRequest(f"no request {request}")
    return forest.paths[request]


def node_query_set(forest: Forest, node: int) -> tuple:
    if node == ROOT:
        raise UnknownNode("virtual root has no query set")
    return forest.node(node).query_set


_VIOLATION_CODES = ("BadNodeIndex", "NonEmptyRoot", "EmptyNonRootNode", "DimensionMismatch", "CycleDetected",
                    "DanglingParent", "AdjacencyMismatch", "PathNotPrefixChain", "QuerySetUnsorted",
                    "QuerySetPathMismatch", "VisibleLenOutOfRange", "FlattenMismatch")


_NONE = -(2 ** 63)  # codec_report_get's None


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(x) for x in lists]) if lists else []
    idx = np.fromiter((int(v) for x in lists for v in x), dtype=np.int64, count=int(ptr[-1]))
    return ptr, (idx if len(idx) else np.zeros(1, np.int64))


def validate(forest: Forest) -> list:
    """Every structural invariant, reported as a list of violations instead
    of raised -- the contract of the reference's validate()
    (forest.py:266-363): same codes, messages and order. The checks run in
    the library (codec_forest_validate, csrc/host_validate.cpp) over a flat
    snapshot of the forest object."""
    nodes = forest.nodes
    n = len(nodes)
    ids = np.array([nd.id for nd in nodes] or [0], dtype=np.int64)
    parent = np.array([nd.parent for nd in nodes] or [0], dtype=np.int64)
    length = np.array([nd.len for nd in nodes] or [0], dtype=np.int64)
    kv_state = np.zeros(max(n, 1), dtype=np.int32)
    tails = [()] * n
    for i, nd in enumerate(nodes[1:], start=1):
        if nd.keys is None:
            continue
        if _shape(nd.keys) != _shape(nd.values):
            kv_state[i] = 1
        else:
            kv_state[i], tails[i] = 2, _shape(nd.keys)[1:]
    t_ptr, t_idx = _csr(tails)
    c_ptr, c_idx = _csr(list(forest.children) + [[]] * max(0, n - len(forest.children)))
    p_ptr, p_idx = _csr(forest.paths)
    q_ptr, q_idx = _csr([nd.query_set for nd in nodes])
    vn, vr, vc = [], [], []
    for i, nd in enumerate(nodes[1:], start=1):
        for rid, cnt in (nd.visible_len or {}).items():
            vn.append(i)  # position; the message uses that node's id and len
            vr.append(int(rid))
            vc.append(int(cnt))
    n_vis = len(vn)
    vn, vr, vc = (np.array(x or [0], dtype=np.int64) for x in (vn, vr, vc))
    off = np.array(list(forest.token_offset) or [0], dtype=np.int64)
    P64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.codec_forest_validate(n, P64(ids), P64(parent), P64(length),
                                       kv_state.ctypes.data_as(C.POINTER(C.c_int32)), P64(t_ptr), P64(t_idx),
                                       forest.h_kv, forest.d, P64(c_ptr), P64(c_idx), forest.bs, P64(p_ptr),
                                       P64(p_idx), P64(q_ptr), P64(q_idx), n_vis, P64(vn), P64(vr), P64(vc),
                                       P64(off), len(forest.token_offset), C.byref(h)))
    try:
        cnt = C.c_int64()
        _lib.check(L.codec_report_count(h, C.byref(cnt)))
        out = []
        code, node, req = C.c_int32(), C.c_int64(), C.c_int64()
        msg = C.create_string_buffer(4096)
        for i in range(cnt.value):
            _lib.check(L.codec_report_get(h, i, C.byref(code), C.byref(node), C.byref(req), msg, len(msg)))
            out.append(Violation(_VIOLATION_CODES[code.value], msg.value.decode(),
                                 node=None if node.value == _NONE else int(node.value),
                                 request=None if req.value == _NONE else int(req.value)))
        return out
    finally:
        L.codec_report_free(h)
