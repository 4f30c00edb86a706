"""Generate the forest on-disk fixtures with the REFERENCE's dump_forest
(run in the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_forest_fixture.py

Writes ref_forest_sidecar.json + .npz and ref_forest_inline.json: a
3-node tree (root 5 tokens, two children of 3 and 2 tokens, one with a
visible_len), h_kv = 2, d = 4, float64, 3 requests.
"""
from pathlib import Path

import numpy as np
from prefixdec.forest import build_forest, dump_forest

here = Path(__file__).resolve().parent
rng = np.random.default_rng(17)
kv = lambda n: (rng.standard_normal((n, 2, 4)), rng.standard_normal((n, 2, 4)))
k1, v1 = kv(5)
k2, v2 = kv(3)
k3, v3 = kv(2)
specs = [(0, k1, v1), (1, k2, v2, {1: 2}), (1, k3, v3)]
forest = build_forest(specs, [(1, 2), (1, 2), (1, 3)])
dump_forest(forest, here / "ref_forest_sidecar.json", tensors="sidecar")
dump_forest(forest, here / "ref_forest_inline.json", tensors="inline")
print("wrote", here / "ref_forest_sidecar.json", here / "ref_forest_inline.json")
