"""The library's device task tables against the Python statement of the
device balancer (tests/device_table_model.py): kernel routing (tensor
cores / multi-request / per-request suffix kernels) and the stream-K cut of
tensor-core work into per-CTA-pair pieces, record for record, over forests,
SM budgets and kv-head shards. CPU only (the table is built on the host)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.executor import FLAG_FORCE_TC, FLAG_NO_MULTI, FLAG_NO_TCT, make_dims, table_for

from device_table_model import groups_of, tc_pieces


def _forests():
    yield "cfg2", W.make_config("cfg2", tensors=False)
    yield "cfg3", W.make_config("cfg3", tensors=False)
    rng = np.random.default_rng(7)
    for k in range(4):
        parent, length, paths = [0], [0], []
        for _ in range(int(rng.integers(2, 6))):
            root = len(parent)
            parent.append(0)
            length.append(int(rng.integers(200, 9000)))
            for _ in range(int(rng.integers(1, 90))):
                parent.append(root)
                length.append(int(rng.integers(10, 700)))
                paths.append((root, len(parent) - 1))
        yield f"rand{k}", W.Spec(32, 8, 128, parent, length, None, None,
                                 [paths[i] for i in rng.permutation(len(paths))], None, None)


FORESTS = list(_forests())


@pytest.mark.parametrize("name,spec", FORESTS, ids=[n for n, _ in FORESTS])
@pytest.mark.parametrize("budget", [0, 96, 40])
@pytest.mark.parametrize("heads", [(0, 8), (2, 4)])
@pytest.mark.parametrize("flags", [0, FLAG_NO_MULTI, FLAG_FORCE_TC, FLAG_NO_TCT])
def test_pieces_match_model(name, spec, budget, heads, flags):
    f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, spec.h_kv, spec.d)
    g = spec.h_q // spec.h_kv
    h0, h1 = heads
    multi, tct = not (flags & FLAG_NO_MULTI), not (flags & FLAG_NO_TCT)
    plan = P.plan_device(f, g, P.load_default_profile(), h1 - h0, 148, budget, multi=multi, tct=tct)
    info, blob = table_for(f, plan, make_dims(f, spec.h_q, "bfloat16", h0, h1, flags, 148, budget))
    recs = blob[info.off_tc:info.off_tc + 8 * info.n_tc_groups].reshape(-1, 8)
    got = [(int(r[0]), int(r[1]), int(r[3]), int(r[4]), int(r[5]), int(r[6]), int(r[7])) for r in recs]
    want, n_pairs = tc_pieces(f, plan, g, h1 - h0, 148, budget, multi=multi, force_tc=bool(flags & FLAG_FORCE_TC),
                              tct=tct)
    assert got == want
    assert info.n_tc_blocks == (n_pairs if want else 0)
    # per-pair unit CSR covers the pieces in order
    bp = blob[info.off_tc_block_ptr:info.off_tc_block_ptr + info.n_tc_blocks + 1]
    if want:
        assert bp[0] == 0 and bp[-1] == len(want)
        assert all(want[i][5] == b for b in range(info.n_tc_blocks) for i in range(bp[b], bp[b + 1]))
    # every pair has work and the balance bound holds: no pair over T tiles
    tiles = {}
    for kv, ln, nr, mv, q0, pair, h in want:
        tiles[pair] = tiles.get(pair, 0) + (mv + 127) // 128
    if tiles:
        total = sum(tiles.values())
        assert max(tiles.values()) <= -(-total // len(tiles)) * 2 + 1
    # routing: the other kinds' group counts
    kinds = [x[0] for x in groups_of(f, plan, g, multi, bool(flags & FLAG_FORCE_TC), tct)]
    assert info.n_multi_groups == kinds.count("multi")
    assert info.n_tct_groups == kinds.count("tct")
    assert info.n_gemv_groups == kinds.count("gemv")
