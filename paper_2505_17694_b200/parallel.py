"""Multi-GPU partitioning of the decode-attention step.

Attention is independent per kv head (a query head h reads kv head h // g,
attention.py:91-92) and per tree under the virtual root (forest.py:26;
PAPER.md:506), so the step shards with no cross-GPU reduction:

  * kv-head split (tensor-parallel): rank r owns kv heads
    [r*h_kv/G, (r+1)*h_kv/G) of every node -- a contiguous slab of the
    head-major pool -- and the matching contiguous block of query heads;
    every rank runs the same plan on 1/G of the bytes and FLOPs. The only
    collective is one all-gather of the [bs, h_q/G, d] outputs
    (`all_gather_heads`).
  * tree partition: whole trees (children of the virtual root) are
    LPT-assigned to ranks by their summed cost estimate (greedy_assign,
    scheduler.py:142-155). `shard_trees` cuts a rank's sub-forest (its
    trees' nodes renumbered in global id order, its requests renumbered
    in ascending global order); the rank plans and runs it alone over a
    pool holding only its trees' KV, and `gather_requests` all-gathers
    the per-rank outputs and scatters them back into global request order.

The collective goes through torch.distributed: NCCL over NVLink on the
B200 box, gloo in the CPU tests of the partition / reassembly logic --
or, fused (`PeerGather`), through peer memory: every
rank's merge kernel stores its output rows straight into all ranks'
global output buffers over NVLink / NVSwitch and bumps one arrival
counter per rank; no NCCL call on the data path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


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


def all_gather_heads(local_out, group=None, out=None):
    """All-gather this rank's [bs, h_q/G, d] output into [bs, h_q, d]
    (`out`, when given, is the [G, bs, h_q/G, d] receive buffer)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    buf = out if out is not None else torch.empty((world,) + tuple(local_out.shape), dtype=local_out.dtype,
                                                  device=local_out.device)
    # rank-major concatenation along dim 0 (the form every backend accepts)
    flat = buf.view((world * local_out.shape[0],) + tuple(local_out.shape[1:]))
    dist.all_gather_into_tensor(flat, local_out.contiguous(), group=group)
    return assemble_heads(buf)


# ------------------------------------------------------------ tree partition
@dataclass(frozen=True)
class TreePartition:
    trees: tuple         # root node id of each tree
    rank_of_tree: tuple  # rank owning each tree
    loads: tuple         # summed estimate per rank (ms)
    tree_cost: tuple = ()  # summed estimate per tree (ms)

    @property
    def world(self) -> int:
        return len(self.loads)

    def requests_of(self, forest, rank):
        """Requests whose path starts in a tree owned by `rank`, ascending."""
        own = {t for t, r in zip(self.trees, self.rank_of_tree) if r == rank}
        return [i for i, p in enumerate(forest.paths) if p[0] in own]


def tree_roots(forest) -> dict:
    """node id -> root of its tree (the child of the virtual root above it)."""
    root_of = {}
    for n in forest.nodes[1:]:  # parents precede children (forest.py:160-216)
        root_of[n.id] = n.id if n.parent == 0 else root_of[n.parent]
    return root_of


def tree_partition(forest, table, world: int, head_multiplicity: int = 1) -> TreePartition:
    """LPT-assign whole trees to ranks by the summed cost estimate of their
    node tasks (each node task costed unsplit)."""
    from .cost_model import estimate
    from .scheduler import greedy_assign

    if world < 1:
        raise ValueError(f"need world >= 1, got {world}")
    roots = [n.id for n in forest.nodes[1:] if n.parent == 0]
    root_of = tree_roots(forest)
    cost = {r: 0.0 for r in roots}
    for n in forest.nodes[1:]:
        if n.query_set:
            cost[root_of[n.id]] += estimate(table, len(n.query_set) * head_multiplicity, n.len)
    a = greedy_assign([cost[r] for r in roots], world)
    return TreePartition(tuple(roots), tuple(a.block_of), tuple(a.loads), tuple(cost[r] for r in roots))


@dataclass(frozen=True)
class TreeShard:
    """One rank's part of a tree partition.

    requests[i] is the global id of local request i (ascending); nodes[j]
    the global id of local node j + 1 (ascending, so parents still precede
    children); parent / lengths / paths / visible describe the sub-forest
    in local ids, the forest_from_pool argument form."""

    rank: int
    requests: tuple
    nodes: tuple
    parent: tuple
    lengths: tuple
    paths: tuple
    visible: tuple | None

    @property
    def bs(self) -> int:
        return len(self.requests)

    def forest(self, h_kv: int, d: int, kv_dtype: str = "bfloat16"):
        """The sub-forest (no tensors; adopt or pack a pool for it)."""
        from .forest import forest_from_pool
        return forest_from_pool(self.parent, self.lengths, self.paths, h_kv, d, visible=self.visible,
                                kv_dtype=kv_dtype)

    def token_map(self, full_forest, sub_forest) -> np.ndarray:
        """int64 [T_sub]: global pool token of every sub-forest pool token
        (the sub-forest's own preorder layout)."""
        idx = np.zeros(max(sub_forest.total_tokens, 1), dtype=np.int64)
        for j, gn in enumerate(self.nodes):
            ln = self.lengths[j]
            lo = sub_forest.token_offset[j + 1]
            g0 = full_forest.token_offset[gn]
            idx[lo:lo + ln] = np.arange(g0, g0 + ln, dtype=np.int64)
        return idx

    def slice_pool(self, full_forest, sub_forest, k_pool, v_pool):
        """This shard's head-major pools [h][T_sub][d] cut from the full
        forest's pools (tests, single-GPU emulation of a sharded run)."""
        import torch
        idx = torch.from_numpy(self.token_map(full_forest, sub_forest)).to(k_pool.device)
        return k_pool.index_select(1, idx).contiguous(), v_pool.index_select(1, idx).contiguous()


def shard_trees(forest, part: TreePartition, rank: int) -> TreeShard:
    """Rank `rank`'s sub-forest under a tree partition."""
    if not 0 <= rank < part.world:
        raise ValueError(f"bad rank {rank} of {part.world}")
    own = {t for t, r in zip(part.trees, part.rank_of_tree) if r == rank}
    root_of = tree_roots(forest)
    nodes = [n.id for n in forest.nodes[1:] if root_of[n.id] in own]
    local = {gn: j + 1 for j, gn in enumerate(nodes)}
    reqs = [r for r, p in enumerate(forest.paths) if p[0] in own]
    rloc = {r: i for i, r in enumerate(reqs)}
    parent = tuple(0 if forest.nodes[gn].parent == 0 else local[forest.nodes[gn].parent] for gn in nodes)
    lengths = tuple(forest.nodes[gn].len for gn in nodes)
    paths = tuple(tuple(local[gn] for gn in forest.paths[r]) for r in reqs)
    vis = []
    any_vis = False
    for gn in nodes:
        v = forest.nodes[gn].visible_len
        if v:
            any_vis = True
            vis.append({rloc[r]: c for r, c in v.items() if r in rloc})
        else:
            vis.append(None)
    return TreeShard(rank, tuple(reqs), tuple(nodes), parent, lengths, paths, tuple(vis) if any_vis else None)


def request_index(shards) -> np.ndarray:
    """Global request id of every row of the rank-major concatenation of
    the shards' outputs."""
    return np.concatenate([np.asarray(s.requests, dtype=np.int64) for s in shards]) if shards else \
        np.zeros(0, np.int64)


def scatter_requests(per_rank, shards, bs: int):
    """Reassemble rank-ordered outputs ([n_r, h_q, d] each, or a padded
    [G, max n_r, h_q, d] gather buffer) into global request order."""
    import torch
    rows = torch.cat([per_rank[r][:s.bs] for r, s in enumerate(shards)])
    idx = torch.from_numpy(request_index(shards)).to(rows.device)
    if idx.numel() != bs or not torch.equal(torch.sort(idx).values, torch.arange(bs, device=rows.device)):
        raise ValueError("the shards do not cover every request exactly once")
    out = torch.empty((bs,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    out.index_copy_(0, idx, rows)
    return out


def gather_requests(local_out, shards, bs: int, group=None, buf=None):
    """All-gather every rank's [n_r, h_q, d] output (padded to the largest
    shard, one all_gather_into_tensor) and return [bs, h_q, d] in global
    request order. `shards` = every rank's TreeShard (all ranks derive the
    same partition)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if len(shards) != world:
        raise ValueError(f"{len(shards)} shards for {world} ranks")
    n_max = max(s.bs for s in shards)
    send = local_out
    if local_out.shape[0] != n_max:
        send = torch.zeros((n_max,) + tuple(local_out.shape[1:]), dtype=local_out.dtype, device=local_out.device)
        send[:local_out.shape[0]] = local_out
    if buf is None:
        buf = torch.empty((world,) + tuple(send.shape), dtype=send.dtype, device=send.device)
    dist.all_gather_into_tensor(buf.view((world * n_max,) + tuple(send.shape[1:])), send.contiguous(), group=group)
    return scatter_requests(buf, shards, bs)


# ------------------------------------------------------------ fused gather
class _DevArray:
    """__cuda_array_interface__ view of a raw device allocation."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerGather:
    """Symmetric output buffers for the fused output gather
    (codec_decode_attention_gather, include/codec_b200.h): `buffers` global
    outputs float32 [rows, hq_global, d] and one int32 [world] arrival
    counter array per rank, allocated by the library (cudaMalloc + CUDA IPC
    handle) and mapped into every rank of `group` (handles exchanged with
    all_gather_object -- gloo or NCCL). Works across GPUs (peer stores
    over NVLink) and across processes sharing one GPU (the tests).

    Per step: DecodeStep.gather(..., peers=self, buf=b) on every rank, then
    wait(stream); output(b) then holds every rank's rows. A buffer is
    rewritten by the next step that targets it: consumers double-buffer."""

    def __init__(self, rows: int, hq_global: int, d: int, device, group=None, buffers: int = 1):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib

        L = _lib.lib()
        self.device = torch.device(device)
        _lib.bind_device(self.device)  # allocations and peer mappings on this rank's GPU
        self.rows, self.hq_global, self.d = int(rows), int(hq_global), int(d)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        nbytes = max(self.rows * self.hq_global * self.d * 4, 16)
        self._own, self._opened = [], []

        def alloc(n):
            ptr, h = C.c_void_p(), (C.c_char * 64)()
            _lib.check(L.codec_ipc_alloc(n, C.byref(ptr), h))
            self._own.append(ptr.value)
            return ptr.value, bytes(h)

        mine = [alloc(nbytes) for _ in range(int(buffers))] + [alloc(max(4 * self.world, 16))]
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, [h for _, h in mine], group=group)
        else:
            allh = [[h for _, h in mine]]
        ptrs = []  # ptrs[p][j]: rank p's allocation j mapped here
        for p in range(self.world):
            if p == self.rank:
                ptrs.append([ptr for ptr, _ in mine])
                continue
            row = []
            for h in allh[p]:
                ptr = C.c_void_p()
                _lib.check(L.codec_ipc_open(C.create_string_buffer(h, 64), C.byref(ptr)))
                self._opened.append(ptr.value)
                row.append(ptr.value)
            ptrs.append(row)
        self.buffers = int(buffers)
        self._peer_out = [torch.tensor([ptrs[p][b] for p in range(self.world)], dtype=torch.int64, device=self.device)
                          for b in range(self.buffers)]
        self._peer_flags = torch.tensor([ptrs[p][-1] for p in range(self.world)], dtype=torch.int64,
                                        device=self.device)
        self._flags_local = mine[-1][0]
        self._done = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._expected = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._out_views = [torch.as_tensor(_DevArray(mine[b][0], (self.rows, self.hq_global, self.d), "<f4"),
                                           device=self.device) for b in range(self.buffers)]

    def struct(self, head0: int, row_map=None, buf: int = 0):
        import ctypes as C

        from . import _lib

        return _lib.PeerGatherC(self.world, self.rank, self.hq_global, int(head0),
                                C.c_void_p(self._peer_out[buf].data_ptr()), C.c_void_p(self._peer_flags.data_ptr()),
                                C.c_void_p(row_map.data_ptr()) if row_map is not None else None,
                                C.c_void_p(self._done.data_ptr()))

    def wait(self, stream=None):
        """Make `stream` wait until every rank's rows of the next step
        arrived here."""
        import ctypes as C

        import torch

        from . import _lib

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.bind_device(self.device)
        _lib.check(_lib.lib().codec_peer_wait(C.c_void_p(self._flags_local), self.world,
                                              C.c_void_p(self._expected.data_ptr()), C.c_void_p(st.cuda_stream)))

    def output(self, buf: int = 0):
        """The gathered global output [rows, hq_global, d] (float32) of `buf`."""
        return self._out_views[buf]

    def close(self):
        """Unmap the peers' buffers and free this rank's (after a barrier:
        no peer may still be storing into them)."""
        import torch
        import torch.distributed as dist

        from . import _lib

        if not (self._own or self._opened):
            return
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(group=self.group)
        L = _lib.lib()
        for ptr in self._opened:
            L.codec_ipc_close(ptr)
        if self.world > 1:
            dist.barrier(group=self.group)
        for ptr in self._own:
            L.codec_ipc_free(ptr)
        self._own, self._opened, self._out_views = [], [], []
