"""Seeded synthetic prefix forests (the benchmark inputs).

Draw-for-draw compatible with the reference generator
(prefixdec/workloads.py:104-233): one `numpy.random.default_rng(seed)`
stream, per node keys then values as N(0,1)/sqrt(d) float64 draws, the
query batch last. Equal seeds therefore give the reference's exact
inputs (pinned by tests/golden/workloads.json), which is what lets the
parity tests compare against the CPU oracle on identical data.

Besides the reference's four families this module adds the structures
BASELINE.json names for configs 3 and 4; those are
new recipes, not reference generators.

Generators return a `Spec`: node parents, per-node tensors (or only
lengths when `tensors=False`, for planning/indexing at sizes that do
not fit host RAM as float64) and request paths.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Spec:
    h_q: int
    h_kv: int
    d: int
    parent: list = field(default_factory=lambda: [0])   # index 0 = virtual root
    length: list = field(default_factory=lambda: [0])
    keys: list = field(default_factory=lambda: [None])
    values: list = field(default_factory=lambda: [None])
    paths: list = field(default_factory=list)
    queries: np.ndarray | None = None
    visible: list | None = None   # per node {request: visible count} or None

    @property
    def n_nodes(self):
        return len(self.parent)

    @property
    def bs(self):
        return len(self.paths)

    def node_specs(self):
        """(parent, keys, values) tuples in the reference build_forest
        format (forest.py:160-167)."""
        vis = self.visible or [None] * self.n_nodes
        return [(self.parent[i], self.keys[i], self.values[i], vis[i]) for i in range(1, self.n_nodes)]


class _Draw:
    """One seeded stream, fixed draw order (workloads.py:104-122)."""

    def __init__(self, spec: Spec, seed: int, tensors: bool, dtype):
        self.rng = np.random.default_rng(seed)
        self.spec = spec
        self.scale = 1.0 / math.sqrt(spec.d)
        self.tensors = tensors
        self.dtype = np.dtype(dtype) if dtype is not None else None

    def _one(self, shape):
        x = self.rng.standard_normal(shape) * self.scale
        return x if self.dtype is None else x.astype(self.dtype)

    def node(self, parent: int, n: int) -> int:
        s = self.spec
        if self.tensors:
            shape = (n, s.h_kv, s.d)
            k = self._one(shape)
            v = self._one(shape)
        else:
            k = v = None
        s.parent.append(parent)
        s.length.append(n)
        s.keys.append(k)
        s.values.append(v)
        return s.n_nodes - 1

    def queries(self):
        s = self.spec
        if self.tensors:
            s.queries = self._one((s.bs, s.h_q, s.d))


def two_level(shared_len, leaf_len, batch, h_q=1, h_kv=1, d=16, seed=0,
              tensors=True, dtype=None) -> Spec:
    """One shared root, one private leaf per request
    (workloads.py:125-137)."""
    spec = Spec(h_q, h_kv, d)
    dr = _Draw(spec, seed, tensors, dtype)
    root = dr.node(0, shared_len)
    for _ in range(batch):
        leaf = dr.node(root, leaf_len)
        spec.paths.append((root, leaf))
    dr.queries()
    return spec


def full_tree(arity, depth, node_len, h_q=1, h_kv=1, d=16, seed=0,
              tensors=True, dtype=None) -> Spec:
    """Complete arity-ary tree, one request per leaf, BFS ids
    (workloads.py:140-174)."""
    spec = Spec(h_q, h_kv, d)
    dr = _Draw(spec, seed, tensors, dtype)
    level = [dr.node(0, node_len)]
    for _ in range(depth - 1):
        level = [dr.node(p, node_len) for p in level for _ in range(arity)]
    for leaf in level:
        chain = []
        cur = leaf
        while cur:
            chain.append(cur)
            cur = spec.parent[cur]
        spec.paths.append(tuple(reversed(chain)))
    dr.queries()
    return spec


def degenerate(depth, node_len, h_q=1, h_kv=1, d=16, seed=0,
               tensors=True, dtype=None) -> Spec:
    """Spine of depth-1 nodes, one leaf per spine node, two on the last
    (workloads.py:177-199)."""
    spec = Spec(h_q, h_kv, d)
    dr = _Draw(spec, seed, tensors, dtype)
    for i in range(depth - 1):
        dr.node(i, node_len)
    for i in range(1, depth - 1):
        leaf = dr.node(i, node_len)
        spec.paths.append(tuple(range(1, i + 1)) + (leaf,))
    for _ in range(2):
        leaf = dr.node(depth - 1, node_len)
        spec.paths.append(tuple(range(1, depth)) + (leaf,))
    dr.queries()
    return spec


def shared_ratio(total_len, ratio, batch, h_q=1, h_kv=1, d=16, seed=0,
                 tensors=True, dtype=None) -> Spec:
    """Two-level tree sized by the shared-token fraction
    (workloads.py:202-233)."""
    shared = math.floor(total_len * ratio + 1e-9)
    rest = total_len - shared
    spec = Spec(h_q, h_kv, d)
    dr = _Draw(spec, seed, tensors, dtype)
    root = dr.node(0, shared)
    if rest == 0:
        spec.paths = [(root,)] * batch
    else:
        base, extra = divmod(rest, batch)
        for r in range(batch):
            leaf = dr.node(root, base + (1 if r < extra else 0))
            spec.paths.append((root, leaf))
    dr.queries()
    return spec


def tot_tree(root_len=8192, branching=4, levels=4, lo=64, hi=2049, h_q=32, h_kv=8, d=128,
             seed=3, tensors=True, dtype=None) -> Spec:
    """Config 3: tree-of-thought / beam tree. Root of root_len tokens, then
    levels-1 levels of `branching` children; non-root lengths from
    default_rng(seed).integers(lo, hi) in BFS creation order; tensors from
    a separate stream seeded `seed`."""
    lens = np.random.default_rng(seed).integers(lo, hi, size=sum(branching ** i for i in range(1, levels)))
    spec = Spec(h_q, h_kv, d)
    dr = _Draw(spec, seed, tensors, dtype)
    level = [dr.node(0, root_len)]
    it = iter(int(x) for x in lens)
    for _ in range(levels - 1):
        level = [dr.node(p, next(it)) for p in level for _ in range(branching)]
    for leaf in level:
        chain = []
        cur = leaf
        while cur:
            chain.append(cur)
            cur = spec.parent[cur]
        spec.paths.append(tuple(reversed(chain)))
    dr.queries()
    return spec


def forest_of_trees(n_trees=64, suffix=512, h_q=32, h_kv=8, d=128, seed=4,
                    tensors=True, dtype=None, only_trees=None) -> Spec:
    """Config 4: imbalanced forest. Tree t has a shared prefix of
    P = round(exp(U(ln 512, ln 131072))) tokens and R = round(exp(U(0,
    ln 512))) requests, each with a private `suffix`-token leaf; shapes
    from default_rng(seed); tensors of tree t from their own stream
    seeded 1000+t (root, suffixes, then that tree's queries) so any tree
    regenerates alone. `only_trees` keeps a subset
    (original tree seeds preserved) for bounded CPU-oracle samples."""
    shape_rng = np.random.default_rng(seed)
    shapes = []
    for _ in range(n_trees):
        p = int(round(math.exp(shape_rng.uniform(math.log(512), math.log(131072)))))
        r = int(round(math.exp(shape_rng.uniform(0.0, math.log(512)))))
        shapes.append((p, max(r, 1)))
    spec = Spec(h_q, h_kv, d)
    qs = []
    for t, (p, r) in enumerate(shapes):
        if only_trees is not None and t not in only_trees:
            continue
        dr = _Draw(spec, 1000 + t, tensors, dtype)
        root = dr.node(0, p)
        for _ in range(r):
            leaf = dr.node(root, suffix)
            spec.paths.append((root, leaf))
        if tensors:
            qs.append(dr._one((r, h_q, d)))
    if tensors:
        spec.queries = np.concatenate(qs)
    return spec


def cast(spec: Spec, dtype) -> Spec:
    """Re-type every tensor after generation (workloads.py:247-258)."""
    dt = np.dtype(dtype)
    out = Spec(spec.h_q, spec.h_kv, spec.d, list(spec.parent), list(spec.length),
               [None] + [k.astype(dt) for k in spec.keys[1:]],
               [None] + [v.astype(dt) for v in spec.values[1:]],
               list(spec.paths), None if spec.queries is None else spec.queries.astype(dt),
               spec.visible)
    return out


# Named benchmark configurations (BASELINE.json "configs")
CONFIGS = {
    "cfg1": dict(fn=two_level, kw=dict(shared_len=1024, leaf_len=64, batch=16, h_q=8, h_kv=8, d=128, seed=0)),
    "cfg2": dict(fn=two_level, kw=dict(shared_len=32768, leaf_len=512, batch=256, h_q=32, h_kv=8, d=128, seed=0)),
    "cfg3": dict(fn=tot_tree, kw=dict()),
    "cfg4": dict(fn=forest_of_trees, kw=dict()),
    "cfg5": dict(fn=two_level, kw=dict(shared_len=65536, leaf_len=512, batch=1024, h_q=64, h_kv=8, d=128, seed=0)),
}


def make_config(name, tensors=True, dtype=None, **over) -> Spec:
    c = CONFIGS[name]
    kw = dict(c["kw"])
    kw.update(over)
    return c["fn"](tensors=tensors, dtype=dtype, **kw)
