"""Seeded test-input recipes shared by the golden generator and the tests.

They reproduce, draw for draw, the input factories of the reference test
suite -- conftest.random_forest (pkg/tests/conftest.py:21-82),
conftest.random_micro_instance (:85-98) and test_kernels.make_inputs
(pkg/tests/test_kernels.py:16-33) -- so the golden outputs recorded from
the reference apply to inputs regenerated here (or on the GPU box)
without storing the tensors.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2505_17694_b200.workloads import Spec

PAC_SHAPES = [
    # (n, n_q, h_q, h_kv, d)
    (1, 1, 1, 1, 4),
    (7, 3, 2, 1, 16),
    (33, 5, 4, 2, 64),
    (2049, 2, 4, 4, 32),
    (512, 8, 8, 2, 128),
]


def random_forest_spec(seed, *, max_depth=6, max_arity=5, max_len=64, max_bs=16, with_masks=False):
    rng = np.random.default_rng(seed)
    d = int(rng.choice([4, 16, 64]))
    g = int(rng.choice([1, 2, 4]))
    h_kv = int(rng.integers(1, 3))
    h_q = h_kv * g
    scale = 1.0 / math.sqrt(d)
    depth = int(rng.integers(1, max_depth + 1))
    spec = Spec(h_q, h_kv, d)

    def grow(parent):
        n = int(rng.integers(1, max_len + 1))
        k = rng.standard_normal((n, h_kv, d)) * scale
        v = rng.standard_normal((n, h_kv, d)) * scale
        spec.parent.append(parent)
        spec.length.append(n)
        spec.keys.append(k)
        spec.values.append(v)
        return spec.n_nodes - 1

    frontier = [grow(0)]
    for _ in range(depth - 1):
        nxt = []
        for nid in frontier:
            for _ in range(int(rng.integers(0, max_arity + 1))):
                nxt.append(grow(nid))
        if not nxt:
            break
        frontier = nxt

    inner = set(spec.parent[1:])
    leaves = [nid for nid in range(1, spec.n_nodes) if nid not in inner]
    bs = int(rng.integers(1, min(max_bs, len(leaves)) + 1))
    chosen = sorted(rng.choice(len(leaves), size=bs, replace=False).tolist())
    for i in chosen:
        chain = []
        cur = leaves[i]
        while cur:
            chain.append(cur)
            cur = spec.parent[cur]
        spec.paths.append(tuple(reversed(chain)))

    spec.visible = [None] * spec.n_nodes
    if with_masks:
        for rid, path in enumerate(spec.paths):
            for nid in path:
                ln = spec.length[nid]
                if ln > 1 and rng.random() < 0.25:
                    if spec.visible[nid] is None:
                        spec.visible[nid] = {}
                    spec.visible[nid][rid] = int(rng.integers(1, ln + 1))
    spec.queries = rng.standard_normal((bs, h_q, d)) * scale
    return spec


def random_micro_tasks(seed):
    """(tasks, m) of conftest.random_micro_instance; tasks as
    (node, n_q, n) tuples."""
    gen = np.random.default_rng(seed)
    t = int(gen.integers(1, 5))
    m = int(gen.integers(1, 5))
    tasks = []
    for j in range(t):
        n_q = int(gen.integers(1, 9))
        n = int(gen.integers(1, 20001))
        tasks.append((j + 1, n_q, n))
    return tasks, m


def pac_inputs(shape, dtype=np.float64, seed=7, masked=False):
    n, n_q, h_q, h_kv, d = shape
    rng = np.random.default_rng(seed)
    q = (rng.standard_normal((n_q, h_q, d)) / math.sqrt(d)).astype(dtype)
    k = (rng.standard_normal((n, h_kv, d)) / math.sqrt(d)).astype(dtype)
    v = rng.standard_normal((n, h_kv, d)).astype(dtype)
    vis = rng.integers(1, n + 1, size=n_q) if masked else None
    return q, k, v, vis


def multi_tree_spec(seed, n_trees=5, h_q=8, h_kv=4, d=16, with_masks=True):
    """Several independent trees under the virtual root (forest.py:26):
    random depth / fan-out / lengths per tree, optional per-request
    visible_len masks. The tree partition tests' input."""
    rng = np.random.default_rng(seed)
    scale = 1.0 / math.sqrt(d)
    spec = Spec(h_q, h_kv, d)

    def grow(parent):
        n = int(rng.integers(1, 96))
        spec.parent.append(parent)
        spec.length.append(n)
        spec.keys.append(rng.standard_normal((n, h_kv, d)) * scale)
        spec.values.append(rng.standard_normal((n, h_kv, d)) * scale)
        return spec.n_nodes - 1

    for _ in range(n_trees):
        root = grow(0)
        frontier, tree = [root], [root]
        for _ in range(int(rng.integers(0, 3))):
            nxt = [grow(p) for p in frontier for _ in range(int(rng.integers(1, 4)))]
            tree += nxt
            frontier = nxt
        inner = {spec.parent[n] for n in tree}
        leaves = [n for n in tree if n not in inner]
        for leaf in leaves:
            for _ in range(int(rng.integers(1, 3))):  # some leaves serve two requests
                chain, cur = [], leaf
                while cur:
                    chain.append(cur)
                    cur = spec.parent[cur]
                spec.paths.append(tuple(reversed(chain)))
    # interleave the trees' requests (a shard's requests are then scattered)
    spec.paths = [spec.paths[i] for i in rng.permutation(len(spec.paths))]
    spec.visible = [None] * spec.n_nodes
    if with_masks:
        for rid, path in enumerate(spec.paths):
            for nid in path:
                ln = spec.length[nid]
                if ln > 1 and rng.random() < 0.25:
                    spec.visible[nid] = spec.visible[nid] or {}
                    spec.visible[nid][rid] = int(rng.integers(1, ln + 1))
    spec.queries = rng.standard_normal((spec.bs, h_q, d)) * scale
    return spec


# Corruptions applied to a built forest object (reference or ours) for the
# validate() goldens: (name, fn(forest)). Each breaks one or more of the
# invariants reference forest.py:266-363 reports.
def _mut(name):
    def apply(f):
        import numpy as _np
        if name == "bad_id":
            f.nodes[2].id = 7
        elif name == "cycle":
            f.nodes[1].parent = 2
        elif name == "dangling":
            f.nodes[3].parent = 40
        elif name == "path_break":
            f.paths[0] = (2, 1)
        elif name == "qset_unsorted":
            f.nodes[2].query_set = (1, 0)
        elif name == "qset_foreign":
            f.nodes[3].query_set = (5,)
        elif name == "qset_negative":
            f.nodes[3].query_set = (-1,)
        elif name == "visible_range":
            f.nodes[3].visible_len = {2: 9, 1: 0}
        elif name == "flatten":
            f.token_offset[2] = 99
        elif name == "adjacency":
            f.children[1] = [3]
        elif name == "kv_tail":
            f.nodes[2].keys = _np.zeros((3, 3, 4))
            f.nodes[2].values = _np.zeros((3, 3, 4))
        elif name == "kv_differ":
            f.nodes[2].values = _np.zeros((2, 2, 4))
        elif name == "kv_2d":
            f.nodes[3].keys = _np.zeros((4, 8))
            f.nodes[3].values = _np.zeros((4, 8))
        elif name == "many":
            f.nodes[1].parent = 3
            f.paths[1] = (1, 9)
            f.nodes[2].query_set = (0, 0)
        elif name != "clean":
            raise ValueError(name)
    return apply


VALIDATE_CASES = ["clean", "bad_id", "cycle", "dangling", "path_break", "qset_unsorted", "qset_foreign",
                  "qset_negative", "visible_range", "flatten", "adjacency", "kv_tail", "kv_differ", "kv_2d", "many"]


def validate_forest_specs(seed=0):
    """the small forest the validate() goldens corrupt: (specs, paths)"""
    rng = np.random.default_rng(seed)
    t = lambda n: rng.standard_normal((n, 2, 4))
    specs = [(0, t(5), t(5)), (1, t(3), t(3), {0: 2}), (1, t(4), t(4))]
    return specs, [(1, 2), (1, 3), (1,)]


def mutate(forest, name):
    _mut(name)(forest)
    return forest


# Profile CSVs the reference's load_profile / CostTable reject (or accept),
# for the error-contract goldens (cost_model.py:39-53, :102-150).
PROFILE_CASES = {
    "ok": "# src=x\n# a=1\nn_q,n,cost_ms\n1,512,0.5\n2,512,0.75\n1,1024,1.0\n2,1024,1.5\n",
    "no_body": "# only=meta\n\n",
    "bad_header": "n,n_q,cost_ms\n1,512,0.5\n",
    "bad_int": "n_q,n,cost_ms\n1,512,0.5\nx,1024,1.0\n",
    "short_row": "n_q,n,cost_ms\n1,512\n",
    "duplicate": "n_q,n,cost_ms\n1,512,0.5\n2,512,-1\n1,512,0.7\n",
    "non_positive": "n_q,n,cost_ms\n1,512,0.5\n2,512,-0.25\n2,512,0.7\n",
    "non_positive_int": "n_q,n,cost_ms\n1,512,0\n",
    "missing": "n_q,n,cost_ms\n1,512,0.5\n2,512,0.75\n1,1024,1.0\n",
    "knot_zero": "n_q,n,cost_ms\n0,512,0.5\n",
    "extra_field": "n_q,n,cost_ms\n1,512,0.5,9\n",
}
