"""Forest on-disk format: a JSON document of the
structure -- dims, nodes (id, parent, len, optional visible_len), request
paths -- with the K/V matrices either inline (nested row-major lists) or in
an .npz sidecar (arrays k<id>, v<id>). Files are interchangeable with the
reference's `dump_forest` / `load_forest` (forest.py:386-441): same keys,
same sidecar naming, so fixtures written by either side load in the other.

Beyond the reference: bfloat16 forests (torch tensors) are written with
dims.dtype = "bfloat16" and float32 payloads (exact: bf16 widens to fp32
losslessly) and load back as bfloat16 tensors; forests built on a device
pool (forest_from_pool, no per-node tensors) are written from that pool.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .forest import Forest, build_forest


def _host_array(x):
    if hasattr(x, "detach"):  # torch tensor
        import torch
        t = x.detach().cpu()
        if t.dtype == torch.bfloat16:
            t = t.float()
        return t.numpy()
    return np.asarray(x)


def _node_kv(forest: Forest, node, k_pool, v_pool):
    if node.keys is not None:
        return _host_array(node.keys), _host_array(node.values)
    if k_pool is None or v_pool is None:
        raise ValueError(f"node {node.id} has no tensors: pass the forest's k_pool / v_pool")
    lo = forest.token_offset[node.id]
    # head-major pools [h][T][d] -> the node's [len, h, d]
    k = _host_array(k_pool[:, lo:lo + node.len]).transpose(1, 0, 2)
    v = _host_array(v_pool[:, lo:lo + node.len]).transpose(1, 0, 2)
    return np.ascontiguousarray(k), np.ascontiguousarray(v)


def dump_forest(forest: Forest, path, tensors: str = "sidecar", k_pool=None, v_pool=None) -> None:
    """Write `forest` to `path` (JSON) with its K/V inline or in
    `path.with_suffix('.npz')`."""
    if tensors not in ("inline", "sidecar"):
        raise ValueError(f"tensors must be 'inline' or 'sidecar', got {tensors!r}")
    path = Path(path)
    nodes = forest.nodes[1:]
    kv = {n.id: _node_kv(forest, n, k_pool, v_pool) for n in nodes}
    dtype = "bfloat16" if "bfloat16" in str(forest.dtype) else str(np.dtype(next(iter(kv.values()))[0].dtype))
    doc = {
        "dims": {"h_kv": forest.h_kv, "d": forest.d, "dtype": dtype},
        "nodes": [dict(id=n.id, parent=n.parent, len=n.len,
                       **({"visible_len": {str(r): int(c) for r, c in n.visible_len.items()}} if n.visible_len else {}))
                  for n in nodes],
        "paths": [list(p) for p in forest.paths],
    }
    if tensors == "inline":
        doc["tensors"] = {str(i): {"keys": k.tolist(), "values": v.tolist()} for i, (k, v) in kv.items()}
    else:
        side = path.with_suffix(".npz")
        np.savez(side, **{f"{c}{i}": a for i, (k, v) in kv.items() for c, a in (("k", k), ("v", v))})
        doc["tensor_file"] = side.name
    path.write_text(json.dumps(doc, sort_keys=True) + "\n", encoding="utf-8")


def load_forest(path) -> Forest:
    """Read a forest written by `dump_forest` (ours or the reference's)."""
    path = Path(path)
    doc = json.loads(path.read_text(encoding="utf-8"))
    name = doc["dims"]["dtype"]
    bf16 = name == "bfloat16"
    dtype = np.float32 if bf16 else np.dtype(name)
    npz = np.load(path.parent / doc["tensor_file"]) if "tensor_file" in doc else None
    specs = []
    for e in sorted(doc["nodes"], key=lambda e: e["id"]):
        i = e["id"]
        if npz is not None:
            k, v = npz[f"k{i}"], npz[f"v{i}"]
        else:
            t = doc["tensors"][str(i)]
            k, v = np.asarray(t["keys"], dtype=dtype), np.asarray(t["values"], dtype=dtype)
        k, v = k.astype(dtype, copy=False), v.astype(dtype, copy=False)
        if bf16:
            import torch
            k, v = torch.from_numpy(np.ascontiguousarray(k)).to(torch.bfloat16), \
                torch.from_numpy(np.ascontiguousarray(v)).to(torch.bfloat16)
        vis = e.get("visible_len")
        specs.append((e["parent"], k, v, {int(r): c for r, c in vis.items()} if vis is not None else None))
    return build_forest(specs, [tuple(p) for p in doc["paths"]])
