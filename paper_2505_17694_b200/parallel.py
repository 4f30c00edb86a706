"""Multi-GPU partitioning of the decode-attention step.

Attention is independent per kv head (a query head h reads kv head h // g,
attention.py:91-92) and per tree under the virtual root (forest.py:26),
so the step shards with no cross-GPU reduction:

  * kv-head split (tensor-parallel): rank r owns kv heads
    [r*h_kv/G, (r+1)*h_kv/G) of every node -- a contiguous slab of the
    head-major pool -- and the matching contiguous block of query heads;
    every rank runs the same plan on 1/G of the bytes and FLOPs. The only
    collective is one all-gather of the [bs, h_q/G, d] outputs.
  * tree partition: whole trees (children of the virtual root) are
    LPT-assigned to ranks by their summed cost estimate
    (greedy_assign, scheduler.py:142-155); each rank plans its own
    sub-forest; outputs are gathered by request.

The collective goes through torch.distributed, NCCL over NVLink on the
B200 box and gloo in the CPU tests of the reassembly logic.
"""
from __future__ import annotations

from dataclasses import dataclass


def head_shard(h_kv: int, world: int, rank: int) -> tuple:
    """[begin, end) kv heads of `rank`; h_kv must split evenly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if h_kv % world:
        raise ValueError(f"{h_kv} kv heads do not split over {world} ranks")
    per = h_kv // world
    return rank * per, (rank + 1) * per


def assemble_heads(gathered):
    """[G, bs, h_q/G, d] (rank-major all-gather) -> [bs, h_q, d]."""
    G, bs, hl, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(bs, G * hl, d)


def all_gather_heads(local_out, group=None):
    """All-gather this rank's [bs, h_q/G, d] output into [bs, h_q, d]."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    buf = torch.empty((world,) + tuple(local_out.shape), dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(buf, local_out.contiguous(), group=group)
    return assemble_heads(buf)


@dataclass(frozen=True)
class TreePartition:
    trees: tuple         # root node id of each tree
    rank_of_tree: tuple  # rank owning each tree
    loads: tuple         # summed estimate per rank (ms)

    def requests_of(self, forest, rank):
        """Requests whose path starts in a tree owned by `rank`, ascending."""
        own = {t for t, r in zip(self.trees, self.rank_of_tree) if r == rank}
        return [i for i, p in enumerate(forest.paths) if p[0] in own]


def tree_partition(forest, table, world: int, head_multiplicity: int = 1) -> TreePartition:
    """LPT-assign whole trees to ranks by the summed cost estimate of their
    node tasks (each node task costed unsplit)."""
    from .cost_model import estimate
    from .scheduler import greedy_assign

    roots = [n.id for n in forest.nodes[1:] if n.parent == 0]
    root_of = {}
    for n in forest.nodes[1:]:
        root_of[n.id] = n.id if n.parent == 0 else root_of[n.parent]
    cost = {r: 0.0 for r in roots}
    for n in forest.nodes[1:]:
        if n.query_set:
            cost[root_of[n.id]] += estimate(table, len(n.query_set) * head_multiplicity, n.len)
    a = greedy_assign([cost[r] for r in roots], world)
    return TreePartition(tuple(roots), tuple(a.block_of), tuple(a.loads))
