"""Forest on-disk format (serialize.py) against fixtures written by the
reference's own dump_forest (tests/golden/make_forest_fixture.py,
forest.py:386-441): our loader reads them, our writer produces the same
document, and bf16 / pool-backed forests round-trip."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2505_17694_b200 as P

GOLD = Path(__file__).resolve().parent / "golden"


def _same_forest(a, b):
    assert a.h_kv == b.h_kv and a.d == b.d and a.paths == b.paths
    assert [n.parent for n in a.nodes] == [n.parent for n in b.nodes]
    assert [n.len for n in a.nodes] == [n.len for n in b.nodes]
    assert [n.query_set for n in a.nodes] == [n.query_set for n in b.nodes]
    assert [n.visible_len for n in a.nodes] == [n.visible_len for n in b.nodes]


@pytest.mark.parametrize("mode", ["sidecar", "inline"])
def test_reads_reference_files(mode):
    f = P.load_forest(GOLD / f"ref_forest_{mode}.json")
    assert f.h_kv == 2 and f.d == 4 and f.bs == 3
    assert [n.len for n in f.nodes[1:]] == [5, 3, 2]
    assert f.nodes[2].visible_len == {1: 2}
    assert f.visible_count(2, 1) == 2 and f.visible_count(2, 0) == 3
    rng = np.random.default_rng(17)  # the fixture script's draws, in order
    for nid, n in ((1, 5), (2, 3), (3, 2)):
        k, v = rng.standard_normal((n, 2, 4)), rng.standard_normal((n, 2, 4))
        assert np.array_equal(f.nodes[nid].keys, k) and np.array_equal(f.nodes[nid].values, v)


@pytest.mark.parametrize("mode", ["sidecar", "inline"])
def test_writes_the_reference_document(tmp_path, mode):
    ref_path = GOLD / f"ref_forest_{mode}.json"
    f = P.load_forest(ref_path)
    out = tmp_path / f"ref_forest_{mode}.json"
    P.dump_forest(f, out, tensors=mode)
    assert json.loads(out.read_text()) == json.loads(ref_path.read_text())
    if mode == "sidecar":
        a, b = np.load(out.with_suffix(".npz")), np.load(ref_path.with_suffix(".npz"))
        assert sorted(a.files) == sorted(b.files)
        assert all(np.array_equal(a[x], b[x]) for x in a.files)


def test_float32_roundtrip_and_execute(tmp_path):
    from paper_2505_17694_b200 import workloads as W
    spec = W.two_level(40, 7, 3, h_q=4, h_kv=2, d=8, seed=3)
    specs = [(p, k.astype(np.float32), v.astype(np.float32), vis) for p, k, v, vis in spec.node_specs()]
    f = P.build_forest(specs, spec.paths)
    P.dump_forest(f, tmp_path / "f.json")
    g = P.load_forest(tmp_path / "f.json")
    _same_forest(f, g)
    assert all(np.array_equal(a.keys, b.keys) for a, b in zip(f.nodes[1:], g.nodes[1:]))
    assert str(g.dtype) == "float32"


def test_bfloat16_roundtrip(tmp_path):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    t = lambda n: torch.from_numpy(rng.standard_normal((n, 2, 8)).astype(np.float32)).to(torch.bfloat16)
    f = P.build_forest([(0, t(6), t(6)), (1, t(3), t(3))], [(1, 2), (1,)])
    P.dump_forest(f, tmp_path / "b.json", tensors="inline")
    assert json.loads((tmp_path / "b.json").read_text())["dims"]["dtype"] == "bfloat16"
    g = P.load_forest(tmp_path / "b.json")
    _same_forest(f, g)
    for a, b in zip(f.nodes[1:], g.nodes[1:]):
        assert b.keys.dtype == torch.bfloat16 and torch.equal(a.keys, b.keys) and torch.equal(a.values, b.values)


def test_pool_backed_forest(tmp_path):
    torch = pytest.importorskip("torch")
    from paper_2505_17694_b200 import workloads as W
    spec = W.two_level(20, 5, 2, h_q=2, h_kv=2, d=8, seed=1, tensors=False)
    f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 2, 8)
    T = f.total_tokens
    # the pool forest is bfloat16: small integers are exact
    kp = (torch.arange(2 * T * 8) % 97).to(torch.bfloat16).reshape(2, T, 8)
    vp = -kp
    with pytest.raises(ValueError, match="k_pool"):
        P.dump_forest(f, tmp_path / "p.json")
    P.dump_forest(f, tmp_path / "p.json", k_pool=kp, v_pool=vp)
    g = P.load_forest(tmp_path / "p.json")
    _same_forest(f, g)
    for n in g.nodes[1:]:
        lo = f.token_offset[n.id]
        assert torch.equal(n.keys, kp[:, lo:lo + n.len].permute(1, 0, 2))
        assert torch.equal(n.values, vp[:, lo:lo + n.len].permute(1, 0, 2))
