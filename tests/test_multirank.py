"""Multi-rank plumbing on CPU: world_size 2 over gloo.

The CUDA kernels cannot run here, so each rank's local attention is the CPU
oracle (test infrastructure); everything around it is the product code a
multi-GPU step runs: head_shard() ranges and all_gather_heads() for the
kv-head split; tree_partition(), shard_trees() (sub-forest build, request
and node renumbering, pool token map) and gather_requests() (padded
all-gather + scatter back into request order) for the tree partition.
The result must equal the unsharded oracle exactly: sharding changes no
arithmetic (attention is independent per head and per tree)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


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
                       [z] + [v[:, h0:h1] for v in spec.values[1:]], spec.paths, spec.visible)
    return OA.naive_attention(spec.queries[:, h0 * g:h1 * g], fd)


def _multi_tree(seed):
    from recipes import multi_tree_spec
    return multi_tree_spec(seed, n_trees=7)


def _full_forest(spec):
    import paper_2505_17694_b200 as P
    return P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, spec.h_kv, spec.d,
                              visible=(spec.visible or [None] * spec.n_nodes)[1:])


def _shard_oracle(spec, shard, forest, sub):
    """The rank's local step, restated by the oracle over the shard's own
    sub-forest and a pool gathered through shard.token_map()."""
    from oracle import attention as OA
    # full pools in the head-major [h][T][d] layout of the product
    T = forest.total_tokens
    kp = np.zeros((spec.h_kv, T, spec.d))
    vp = np.zeros_like(kp)
    for n in range(1, spec.n_nodes):
        o = forest.token_offset[n]
        kp[:, o:o + spec.length[n]] = spec.keys[n].transpose(1, 0, 2)
        vp[:, o:o + spec.length[n]] = spec.values[n].transpose(1, 0, 2)
    idx = shard.token_map(forest, sub)
    skp, svp = kp[:, idx], vp[:, idx]
    z = np.zeros((0, spec.h_kv, spec.d))
    keys, vals = [z], [z]
    for j in range(len(shard.nodes)):
        o, ln = sub.token_offset[j + 1], shard.lengths[j]
        keys.append(skp[:, o:o + ln].transpose(1, 0, 2))
        vals.append(svp[:, o:o + ln].transpose(1, 0, 2))
    vis = [None] + list(shard.visible) if shard.visible else None
    fd = OA.ForestData([0] + list(shard.parent), keys, vals, shard.paths, vis)
    return OA.naive_attention(spec.queries[list(shard.requests)], fd)


def _worker(rank, world, port, q, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2505_17694_b200 as P
        from paper_2505_17694_b200 import workloads as W
        from paper_2505_17694_b200 import parallel as PL
        if mode == "heads":
            spec = W.two_level(64, 8, 5, h_q=8, h_kv=4, d=16, seed=3)
            h0, h1 = PL.head_shard(spec.h_kv, world, rank)
            local = torch.from_numpy(_sliced_oracle(spec, h0, h1))
            full = PL.all_gather_heads(local).numpy()
        else:
            spec = _multi_tree(11)
            forest = _full_forest(spec)
            part = PL.tree_partition(forest, P.load_default_profile(), world, head_multiplicity=2)
            shards = [PL.shard_trees(forest, part, r) for r in range(world)]
            me = shards[rank]
            sub = me.forest(spec.h_kv, spec.d)
            local = torch.from_numpy(_shard_oracle(spec, me, forest, sub))
            full = PL.gather_requests(local, shards, forest.bs).numpy()
        if rank == 0:
            q.put(full)
    finally:
        dist.destroy_process_group()


def _run_world2(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    import queue
    full = None
    while full is None:
        try:
            full = q.get(timeout=5)
        except queue.Empty:
            assert all(p.is_alive() or p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return full


def test_head_split_gather_world2():
    from paper_2505_17694_b200 import workloads as W
    full = _run_world2("heads")
    spec = W.two_level(64, 8, 5, h_q=8, h_kv=4, d=16, seed=3)
    assert np.array_equal(full, _sliced_oracle(spec, 0, spec.h_kv))


def test_tree_partition_gather_world2():
    full = _run_world2("trees")
    spec = _multi_tree(11)
    assert np.array_equal(full, _sliced_oracle(spec, 0, spec.h_kv))


def test_shard_trees_structure():
    """Sub-forests: every request and node lands on exactly one rank; local
    paths / visible counts / pool tokens map back onto the global ones."""
    import paper_2505_17694_b200 as P
    from paper_2505_17694_b200 import parallel as PL
    spec = _multi_tree(5)
    forest = _full_forest(spec)
    for world in (1, 2, 3, 4):
        part = PL.tree_partition(forest, P.load_default_profile(), world)
        shards = [PL.shard_trees(forest, part, r) for r in range(world)]
        assert sorted(r for s in shards for r in s.requests) == list(range(forest.bs))
        assert sorted(n for s in shards for n in s.nodes) == list(range(1, spec.n_nodes))
        for s in shards:
            sub = s.forest(spec.h_kv, spec.d)
            for i, r in enumerate(s.requests):
                assert tuple(s.nodes[j - 1] for j in s.paths[i]) == tuple(forest.paths[r])
                for j in s.paths[i]:
                    assert sub.visible_count(j, i) == forest.visible_count(s.nodes[j - 1], r)
            tm = s.token_map(forest, sub)
            assert len(tm) == max(sub.total_tokens, 1)
            assert len(set(tm.tolist())) == len(tm)
        # an unsharded partition is the identity
        if world == 1:
            assert shards[0].requests == tuple(range(forest.bs))
            assert np.array_equal(shards[0].token_map(forest, shards[0].forest(spec.h_kv, spec.d)),
                                  np.arange(forest.total_tokens))


def test_scatter_requests_rejects_bad_cover():
    from paper_2505_17694_b200 import parallel as PL
    s0 = PL.TreeShard(0, (0, 2), (), (), (), (), None)
    s1 = PL.TreeShard(1, (2,), (), (), (), (), None)
    with pytest.raises(ValueError, match="exactly once"):
        PL.scatter_requests([torch.zeros(2, 1, 1), torch.zeros(1, 1, 1)], [s0, s1], 3)


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
    # LPT bound: makespan <= mean + largest single tree
    assert max(part.loads) <= sum(part.loads) / 8 + max(part.tree_cost)
    assert sum(part.loads) == pytest.approx(sum(part.tree_cost))
    reqs = sorted(r for k in range(8) for r in part.requests_of(f, k))
    assert reqs == list(range(f.bs))
