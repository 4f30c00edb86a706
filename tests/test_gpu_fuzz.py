"""GPU stress: randomly shaped mid-size forests through the device plan at
several tensor-core SM budgets (each budget re-cuts the stream-K pieces, so
units of 1..n tiles, partly padded row tiles and pooled lane tails all
occur), concurrent suffix kernel on. Every step must be (a) bit-for-bit
repeatable and (b) within the bf16 bar of a float64 reference over the same
bf16 values, for every request. CODEC_FUZZ_SEEDS=n widens the sweep."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import paper_2505_17694_b200 as P
from paper_2505_17694_b200.executor import DecodeStep

pytestmark = pytest.mark.gpu


def _forest(rng):
    """two-level or three-level tree with random lengths and fan-out"""
    kind = rng.integers(0, 2)
    if kind == 0:
        bs = int(rng.integers(20, 150))
        parent = [0, 0] + [1] * bs
        length = [0, int(rng.integers(900, 6000))] + [int(x) for x in rng.integers(40, 420, size=bs)]
        paths = [(1, 2 + r) for r in range(bs)]
    else:
        parent, length, paths = [0, 0], [0, int(rng.integers(1000, 4000))], []
        for _ in range(int(rng.integers(2, 5))):
            mid = len(parent)
            parent.append(1)
            length.append(int(rng.integers(128, 1500)))
            for _ in range(int(rng.integers(4, 40))):
                parent.append(mid)
                length.append(int(rng.integers(20, 300)))
                paths.append((1, mid, len(parent) - 1))
    return parent, length, paths


def _reference(f, kp, vp, q, r):
    import torch
    toks = torch.cat([torch.arange(f.token_offset[n], f.token_offset[n] + f.visible_count(n, r), device="cuda")
                      for n in f.paths[r]])
    g = q.shape[1] // f.h_kv
    k, v = kp[:, toks].double(), vp[:, toks].double()
    s = torch.einsum("hgd,hld->hgl", q[r].double().view(f.h_kv, g, -1), k) / math.sqrt(f.d)
    return torch.einsum("hgl,hld->hgd", torch.softmax(s, dim=-1), v).reshape(q.shape[1], -1)


@pytest.mark.parametrize("seed", range(int(os.environ.get("CODEC_FUZZ_SEEDS", 6))))
def test_random_forests_all_budgets(seed):
    import torch
    rng = np.random.default_rng(500 + seed)
    parent, length, paths = _forest(rng)
    f = P.forest_from_pool(parent[1:], length[1:], paths, 8, 128)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    T = f.total_tokens
    kp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
    vp = (torch.randn((8, T, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
    q = (torch.randn((f.bs, 32, 128), generator=gen, device="cuda") * 0.088).to(torch.bfloat16)
    ref = torch.stack([_reference(f, kp, vp, q, r) for r in range(f.bs)])
    table = P.load_default_profile()
    for budget in (148, 120, 96, 64, 40):
        plan = P.plan_device(f, 4, table, 8, 148, budget)
        # the opt-in per-entry counted merge on alternate budgets
        flags = 1048576 if budget in (120, 64) else 0
        step = DecodeStep(f, plan, 32, "bfloat16", tc_sm_budget=budget, concurrent=True, flags=flags)
        a = step(q, kp, vp)
        b = step(q, kp, vp)
        torch.cuda.synchronize()
        assert torch.equal(a, b), (seed, budget, "not repeatable")
        err = float((a.double() - ref).abs().max())
        rel = err / float(ref.abs().max())
        assert err <= 2e-3 and rel <= 1e-2, (seed, budget, err, rel)
