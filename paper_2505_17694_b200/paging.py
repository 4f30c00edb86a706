"""Paged KV pools (block tables instead of one
contiguous node pool, as a PagedAttention-style serving engine keeps them).

Layout: every node's tokens are cut into pages of `page_size` tokens
(a power of two >= 128); node n owns the logical pages
[base[n], base[n + 1]) in node-id order (`page_layout`, computed by the
library's `codec_page_layout` so Python and the kernels agree). The pools
are physical: k, v [h_local][n_phys_pages * page_size][d], and
page_table[logical page] names the physical page that holds it. The kernels
translate every 128-token tile / 32-token chunk start through the table
(kern_tc.cu `prow`, kern_mma.cu), so a step over a paged pool computes
exactly what it computes over the contiguous pool: the same tiles in the
same order, bit for bit (tests/test_gpu_parity.py::TestPaged).

The reference keeps each node's K/V as one array (forest.py:68-85) and
has no paged layout; this is the serving-side extension the paper's kernel
assumes.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def page_layout(forest, page_size: int):
    """(node_page_base int64[n_nodes + 1], n_logical_pages)."""
    base = np.zeros(len(forest.nodes) + 1, dtype=np.int64)
    n = C.c_int64()
    _lib.check(_lib.lib().codec_page_layout(forest._index, int(page_size),
                                            base.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
    return base, int(n.value)


def paged_pools(forest, k_pool, v_pool, page_size: int, n_phys_pages: int | None = None, generator=None):
    """Scatter contiguous head-major pools [h][T][d] (nodes at their
    preorder offsets) into physical paged pools under a random page
    permutation. Returns (k_phys, v_phys, page_table int32 on the pools'
    device). Physical pages not named by the table hold zeros."""
    import torch

    base, n_pages = page_layout(forest, page_size)
    n_phys = max(n_pages, n_phys_pages or 0)
    dev = k_pool.device
    perm = torch.randperm(n_phys, generator=generator)[:n_pages].to(torch.int32)
    h, _, d = k_pool.shape
    k_phys = torch.zeros((h, n_phys * page_size, d), dtype=k_pool.dtype, device=dev)
    v_phys = torch.zeros_like(k_phys)
    for node in forest.nodes:
        if node.len == 0:
            continue
        src0 = forest.token_offset[node.id]
        for i in range((node.len + page_size - 1) // page_size):
            lo, hi = i * page_size, min(node.len, (i + 1) * page_size)
            dst0 = int(perm[base[node.id] + i]) * page_size
            k_phys[:, dst0:dst0 + hi - lo] = k_pool[:, src0 + lo:src0 + hi]
            v_phys[:, dst0:dst0 + hi - lo] = v_pool[:, src0 + lo:src0 + hi]
    return k_phys, v_phys, perm.to(dev)
