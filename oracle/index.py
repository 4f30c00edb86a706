"""Oracle: integer indexing of a KV forest (the K0 metadata).

Restates the index arithmetic of reference `forest.py` on plain integer
arrays so the product's C++ indexer can be compared array-for-array.
A forest here is described structurally:

    parent[i]  parent id of node i (i = 1..N, node 0 is the virtual root)
    length[i]  token count of node i (length[0] == 0)
    paths[r]   root-to-leaf node ids of request r
    visible[i] {request: visible token count} or None
"""
from __future__ import annotations

import numpy as np


def children_lists(parent, n_nodes):
    """Children in declaration order (reference forest.py:195-206: each
    new node is appended to its parent's list as it is declared)."""
    kids = [[] for _ in range(n_nodes)]
    for nid in range(1, n_nodes):
        kids[parent[nid]].append(nid)
    return kids


def preorder_offsets(length, kids):
    """Start token of every node under preorder flattening: iterative DFS
    from the root, children visited in declaration order
    (reference forest.py:148-157)."""
    n = len(length)
    off = [0] * n
    cursor = 0
    todo = [0]
    while todo:
        nid = todo.pop()
        off[nid] = cursor
        cursor += length[nid]
        # push in reverse so the first-declared child is popped first
        for c in reversed(kids[nid]):
            todo.append(c)
    return off


def query_sets(paths, n_nodes):
    """I_n: ascending ids of the requests whose path crosses node n
    (reference forest.py:229, :236-237)."""
    members = [set() for _ in range(n_nodes)]
    for rid, path in enumerate(paths):
        for nid in path:
            members[nid].add(rid)
    return [tuple(sorted(m)) for m in members]


def visible_count(length, visible, nid, rid):
    """Tokens of node `nid` request `rid` may attend to
    (reference forest.py:128-132)."""
    vis = visible[nid] if visible is not None else None
    if vis and rid in vis:
        return vis[rid]
    return length[nid]


def csr(lists):
    """Flatten a list of int sequences into (ptr, idx) int32 arrays."""
    ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    for i, lst in enumerate(lists):
        ptr[i + 1] = ptr[i] + len(lst)
    idx = np.fromiter((x for lst in lists for x in lst), dtype=np.int64, count=int(ptr[-1]))
    return ptr, idx


def forest_index(parent, length, paths, visible=None):
    """All K0 arrays for one forest, in the layout the product emits:
    node_off (preorder kappa), qset CSR, path CSR and the per-(node,
    request) visible count aligned with the qset CSR."""
    n = len(length)
    kids = children_lists(parent, n)
    off = preorder_offsets(length, kids)
    qs = query_sets(paths, n)
    qptr, qidx = csr(qs)
    pptr, pidx = csr([tuple(p) for p in paths])
    vis = np.array(
        [visible_count(length, visible, nid, rid) for nid in range(n) for rid in qs[nid]],
        dtype=np.int64,
    )
    return {
        "node_off": np.asarray(off, dtype=np.int64),
        "node_len": np.asarray(length, dtype=np.int64),
        "qset_ptr": qptr,
        "qset_idx": qidx,
        "qset_vis": vis,
        "path_ptr": pptr,
        "path_idx": pidx,
    }
