"""K0 parity (C++ forest indexer vs the reference's Forest, via goldens),
build_forest error behaviour, and the C-ABI surface. CPU only."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden_json
from recipes import random_forest_spec
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import _lib
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.errors import (CycleDetected, DanglingParent, DimensionMismatch, PathNotPrefixChain,
                                          UnknownNode, UnknownRequest)


def build(spec):
    return P.build_forest(spec.node_specs(), spec.paths,
                          P.QueryBatch(spec.queries, spec.h_kv) if spec.queries is not None else None)


class TestIndexGolden:
    def test_random_forests(self):
        for doc in golden_json("index.json")["random"]:
            spec = random_forest_spec(doc["seed"], with_masks=doc["masks"])
            f = build(spec)
            assert [list(n.query_set) for n in f.nodes][1:] == doc["query_sets"][1:]
            assert f.token_offset == doc["token_offset"]
            assert [list(p) for p in f.paths] == doc["paths"]
            assert f.children == doc["children"]
            assert [[t.node, t.n_q, t.n] for t in P.tasks_from_forest(f)] == doc["tasks"]
            assert [f.request_len(r) for r in range(f.bs)] == doc["request_len"]
            assert P.validate(f) == []

    def test_config_structures(self):
        import hashlib
        for doc in golden_json("index.json")["configs"]:
            spec = W.make_config(doc["config"], tensors=False)
            f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, spec.h_kv, spec.d)
            assert hashlib.sha256(np.asarray(f.token_offset, np.int64).tobytes()).hexdigest() == doc["token_offset_sha"]
            qs = np.concatenate([np.asarray(n.query_set, np.int64) for n in f.nodes[1:]])
            assert hashlib.sha256(qs.tobytes()).hexdigest() == doc["qset_sha"]
            t = np.asarray([[x.node, x.n_q, x.n] for x in P.tasks_from_forest(f)], np.int64)
            assert hashlib.sha256(t.tobytes()).hexdigest() == doc["tasks_sha"]

    def test_traffic(self):
        for cname, doc in golden_json("traffic.json").items():
            spec = W.make_config(cname, tensors=False)
            f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, spec.h_kv, spec.d)
            rep = P.traffic_report(f, element_size=2)
            assert rep.kv_rows_codec == doc["rows_codec"]
            assert rep.kv_rows_baseline == doc["rows_baseline"]
            assert rep.nq_bar == float(doc["nq_bar"])


def kv(n, h_kv=1, d=4, seed=0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, h_kv, d)), rng.standard_normal((n, h_kv, d))


class TestBuildErrors:
    """Same classes and messages as reference test_forest.py:63-118."""

    def test_parent_must_be_declared_first(self):
        with pytest.raises(DanglingParent, match="undeclared parent"):
            P.build_forest([(2, *kv(2))], [(1,)])

    def test_self_parent_is_a_cycle(self):
        with pytest.raises(CycleDetected, match="own parent"):
            P.build_forest([(1, *kv(2))], [(1,)])

    def test_kv_shape_mismatch(self):
        k, _ = kv(2)
        _, v = kv(3)
        with pytest.raises(DimensionMismatch, match="equal 3-d shapes"):
            P.build_forest([(0, k, v)], [(1,)])

    def test_empty_node(self):
        with pytest.raises(DimensionMismatch, match="no tokens"):
            P.build_forest([(0, *kv(0))], [(1,)])

    def test_path_chain(self):
        specs = [(0, *kv(4)), (1, *kv(2)), (1, *kv(2))]
        with pytest.raises(PathNotPrefixChain, match="not a parent->child edge"):
            P.build_forest(specs, [(2, 3)])
        with pytest.raises(PathNotPrefixChain, match="empty path"):
            P.build_forest(specs, [()])
        with pytest.raises(PathNotPrefixChain, match="missing node 9"):
            P.build_forest(specs, [(1, 9)])

    def test_visible_len(self):
        k, v = kv(4)
        with pytest.raises(DimensionMismatch, match="outside 1..4"):
            P.build_forest([(0, k, v, {0: 5})], [(1,)])
        with pytest.raises(PathNotPrefixChain, match="not routed"):
            P.build_forest([(0, k, v, {3: 2})], [(1,)])

    def test_queries_checked(self):
        q = P.QueryBatch(np.zeros((2, 2, 4)), h_kv=2)
        with pytest.raises(DimensionMismatch, match="query rows"):
            P.build_forest([(0, *kv(4, h_kv=2, d=4))], [(1,)], q)

    def test_lookups(self):
        f = P.build_forest([(0, *kv(8)), (1, *kv(2)), (1, *kv(2))], [(1, 2), (1, 3)])
        with pytest.raises(UnknownRequest, match="no request 9"):
            P.prefix_path(f, 9)
        with pytest.raises(UnknownNode, match="virtual root"):
            P.node_query_set(f, 0)
        assert f.flatten_index(1, 7) < f.flatten_index(2, 0)


class TestAbiSurface:
    def test_library_exports_every_declared_symbol(self):
        header = (ROOT / "include" / "codec_b200.h").read_text()
        declared = set(re.findall(r"CODEC_API [\w\s\*]*?\b(codec_\w+)\(", header))
        assert declared, "no declarations parsed"
        lib = _lib.lib()
        for name in declared:
            assert hasattr(lib, name), name
        assert declared == set(_lib.exported_symbols())
        assert lib.codec_abi_version() == 8

    def test_library_is_sm100a(self):
        import subprocess
        out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                             capture_output=True, text=True).stdout
        assert "sm_100a" in out

    def test_status_maps_to_reference_errors(self):
        with pytest.raises(PathNotPrefixChain):
            P.build_forest([(0, *kv(4))], [(2,)])


def test_validate_goldens():
    """validate() (codec_forest_validate) on corrupted forests reports what
    the reference's validate() reported (tests/golden/validate.json: codes,
    messages, node / request, order)."""
    from conftest import golden_json
    from recipes import VALIDATE_CASES, mutate, validate_forest_specs
    gold = golden_json("validate.json")
    for case in VALIDATE_CASES:
        specs, paths = validate_forest_specs()
        f = mutate(P.build_forest(specs, paths), case)
        got = [[v.code, v.message, v.node, v.request] for v in P.validate(f)]
        assert got == gold[case], case
