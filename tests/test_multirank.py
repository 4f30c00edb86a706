"""Multi-rank plumbing on CPU: world_size 2 over gloo.

The CUDA kernels cannot run here, so each rank computes its kv-head
shard's output with the CPU oracle and the product code does the rest:
head_shard() ranges, the all-gather and assemble_heads() reassembly, and
tree_partition(). The result must equal the unsharded oracle exactly
(sharding changes no arithmetic: attention is independent per head)."""
from __future__ import annotations

import io
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_table_text


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sliced_oracle(spec, h0, h1):
    from oracle import attention as OA
    g = spec.h_q // spec.h_kv
    z = np.zeros((0, h1 - h0, spec.d))
    fd = OA.ForestData(spec.parent, [z] + [k[:, h0:h1] for k in spec.keys[1:]],
                       [z] + [v[:, h0:h1] for v in spec.values[1:]], spec.paths)
    return OA.naive_attention(spec.queries[:, h0 * g:h1 * g], fd)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_17694_b200 import workloads as W
        from paper_2505_17694_b200.parallel import assemble_heads, head_shard
        spec = W.two_level(64, 8, 5, h_q=8, h_kv=4, d=16, seed=3)
        h0, h1 = head_shard(spec.h_kv, world, rank)
        local = torch.from_numpy(_sliced_oracle(spec, h0, h1))
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(bufs, local)
        full = assemble_heads(torch.stack(bufs)).numpy()
        if rank == 0:
            q.put(full)
    finally:
        dist.destroy_process_group()


def test_head_split_gather_world2():
    from paper_2505_17694_b200 import workloads as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = W.two_level(64, 8, 5, h_q=8, h_kv=4, d=16, seed=3)
    ref = _sliced_oracle(spec, 0, spec.h_kv)
    assert np.array_equal(full, ref)


def test_head_shard_ranges():
    from paper_2505_17694_b200.parallel import head_shard
    assert [head_shard(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        head_shard(8, 3, 0)


def test_tree_partition_balances_cfg4():
    import paper_2505_17694_b200 as P
    from paper_2505_17694_b200 import workloads as W
    from paper_2505_17694_b200.parallel import tree_partition
    spec = W.make_config("cfg4", tensors=False)
    f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, spec.h_kv, spec.d)
    table = P.load_default_profile()
    part = tree_partition(f, table, 8, head_multiplicity=4)
    assert len(part.trees) == 64 and set(part.rank_of_tree) <= set(range(8))
    assert max(part.loads) <= 1.35 * (sum(part.loads) / 8) or max(part.loads) == max(
        P.estimate(table, 1, 1) for _ in [0])
    reqs = sorted(r for k in range(8) for r in part.requests_of(f, k))
    assert reqs == list(range(f.bs))
