"""Paged KV pools (paging.py, codec_dims.page_size / page_table): the page
layout and the table builder's checks on CPU; on the GPU, a step over
randomly permuted physical pages equals the step over the contiguous pool
bit for bit (same tiles, same order, same arithmetic) and the float64
oracle within the bf16 bar."""
from __future__ import annotations

import ctypes as C
import io

import numpy as np
import pytest

from conftest import golden_table_text
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import _lib, workloads as W
from paper_2505_17694_b200.errors import PrefixDecError
from paper_2505_17694_b200.executor import _plan_arrays
from paper_2505_17694_b200.forest import dtype_code
from paper_2505_17694_b200.paging import page_layout


@pytest.fixture(scope="module")
def table():
    return P.load_profile(io.StringIO(golden_table_text("a100_d128.csv")))


def build_table(forest, plan, h_q, page_size, dtype=13, flags=0):
    """codec_table_build with a dummy (never dereferenced) page table."""
    dummy = (C.c_int32 * 4)()
    dims = _lib.Dims(forest.bs, h_q, forest.h_kv, forest.d, 0, forest.h_kv, dtype, flags, 1 << 20, 148, 0,
                     page_size, 0, C.cast(dummy, C.c_void_p) if page_size else None)
    t_node, t_nq, s_task, s_start, s_stop, s_block = _plan_arrays(plan)
    Pt = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    h = C.c_void_p()
    _lib.check(_lib.lib().codec_table_build(forest._index, C.byref(dims), len(t_node), Pt(t_node, C.c_int64),
                                            Pt(t_nq, C.c_int64), len(s_task), Pt(s_task, C.c_int32),
                                            Pt(s_start, C.c_int64), Pt(s_stop, C.c_int64), Pt(s_block, C.c_int32),
                                            C.byref(h)))
    _lib.lib().codec_table_free(h)


class TestLayout:
    @pytest.mark.parametrize("page", [128, 256, 1024])
    def test_node_page_bases(self, page):
        spec = W.two_level(3000, 333, 5, h_q=8, h_kv=2, d=128, seed=1, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 2, 128)
        base, n = page_layout(f, page)
        want = np.concatenate([[0], np.cumsum([-(-node.len // page) for node in f.nodes])])
        assert np.array_equal(base, want) and n == want[-1]


class TestTableChecks:
    def test_aligned_plan_builds(self, table):
        spec = W.two_level(3000, 333, 24, h_q=32, h_kv=8, d=128, seed=2, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        plan = P.plan_device(f, 4, table, 8, 148, page_size=128)
        build_table(f, plan, 32, 128, dtype_code("bfloat16"))

    @pytest.mark.parametrize("page", [64, 100, 129])
    def test_page_size_must_be_pow2_at_least_128(self, table, page):
        spec = W.two_level(3000, 333, 24, h_q=32, h_kv=8, d=128, seed=2, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        plan = P.plan_device(f, 4, table, 8, 148)
        with pytest.raises((PrefixDecError, ValueError), match="power of two"):
            build_table(f, plan, 32, page, dtype_code("bfloat16"))

    def test_float32_pool_is_unsupported(self, table):
        spec = W.two_level(3000, 333, 24, h_q=32, h_kv=8, d=128, seed=2, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        plan = P.plan_device(f, 4, table, 8, 148)
        with pytest.raises((PrefixDecError, ValueError), match="paged KV"):
            build_table(f, plan, 32, 128, dtype_code("float32"))

    def test_unaligned_suffix_slice_is_rejected(self, table):
        # a reference plan that cuts a lightly shared 5000-token node into
        # ceil(n / b)-token slices: 5000 / 3 -> 1667, not a multiple of 32
        spec = W.two_level(5000, 100, 2, h_q=32, h_kv=8, d=128, seed=2, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        tasks = P.tasks_from_forest(f)
        plan = P.plan_uniform_bk(tasks, table, 8, 3)
        with pytest.raises((PrefixDecError, ValueError), match="not a multiple"):
            build_table(f, plan, 32, 128, dtype_code("bfloat16"))

    def test_contiguous_mode_unchanged(self, table):
        spec = W.two_level(5000, 100, 2, h_q=32, h_kv=8, d=128, seed=2, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 8, 3)
        build_table(f, plan, 32, 0, dtype_code("bfloat16"))


@pytest.mark.gpu
class TestPaged:
    @pytest.mark.parametrize("page,shape", [(128, "two_level"), (256, "two_level"), (128, "forest"),
                                             (512, "forest")])
    def test_paged_equals_contiguous(self, table, page, shape):
        import torch
        from paper_2505_17694_b200.executor import DecodeStep
        from paper_2505_17694_b200.paging import paged_pools
        if shape == "two_level":
            spec = W.two_level(4200, 300, 40, h_q=32, h_kv=8, d=128, seed=11, tensors=False)
        else:
            # three independent trees of different depth, odd node lengths
            parent = [0, 0, 1, 1, 0, 4, 4, 4, 0, 8]
            length = [0, 1000, 700, 130, 2600, 77, 300, 511, 900, 260]
            paths = [(1, 2), (1, 3), (1, 2), (4, 5), (4, 6), (4, 7), (4, 7), (8, 9), (8, 9), (8, 9), (8,)]
            spec = W.Spec(32, 8, 128, parent, length, None, None, paths, None, None)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        gen = torch.Generator().manual_seed(page)
        T = f.total_tokens
        kp = (torch.randn((8, T, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        vp = (torch.randn((8, T, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        q = (torch.randn((f.bs, 32, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        kx, vx, pt = paged_pools(f, kp, vp, page, n_phys_pages=page_layout(f, page)[1] + 7, generator=gen)
        plan = P.plan_device(f, 4, table, 8, 148, page_size=page)
        for concurrent in (False, True):
            ref = DecodeStep(f, plan, 32, "bfloat16", concurrent=concurrent)(q, kp, vp)
            got = DecodeStep(f, plan, 32, "bfloat16", concurrent=concurrent, page_size=page, page_table=pt,
                             pool_tokens=kx.shape[1])(q, kx, vx)
            torch.cuda.synchronize()
            assert torch.isfinite(ref).all()
            assert torch.equal(ref, got), (page, shape, concurrent, float((ref - got).abs().max()))
        # and the paged output against the float64 restatement of the
        # reference's single-softmax attention (oracle/attention.py
        # naive_attention, attention.py:164-187) on the same bf16 values,
        # every request: the bf16 bar of the north star
        from oracle import attention as OA
        up = lambda t: t.double().cpu().numpy()
        kp_h, vp_h = up(kp), up(vp)
        z = np.zeros((0, 8, 128))
        node_k = [z] + [kp_h[:, f.token_offset[n]:f.token_offset[n] + f.nodes[n].len].transpose(1, 0, 2)
                        for n in range(1, len(f.nodes))]
        node_v = [z] + [vp_h[:, f.token_offset[n]:f.token_offset[n] + f.nodes[n].len].transpose(1, 0, 2)
                        for n in range(1, len(f.nodes))]
        fd = OA.ForestData(spec.parent, node_k, node_v, spec.paths)
        want = OA.naive_attention(up(q), fd)
        err = np.abs(got.double().cpu().numpy() - want)
        assert err.max() <= 2e-3 and err.max() / np.abs(want).max() <= 1e-2, (page, shape, float(err.max()))

    @pytest.mark.parametrize("page", [128, 256])
    def test_paged_head_shard(self, table, page):
        """A kv-head shard (heads [2, 6) of 8) over a paged
        pool: the shard's slab of the physical pages with the shared page
        table equals the contiguous shard step bit for bit, and its q heads
        [8, 24) match the float64 oracle of the whole forest."""
        import torch
        from paper_2505_17694_b200.executor import DecodeStep
        from paper_2505_17694_b200.paging import paged_pools
        spec = W.two_level(3000, 260, 24, h_q=32, h_kv=8, d=128, seed=5, tensors=False)
        f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128)
        gen = torch.Generator().manual_seed(page + 1)
        T = f.total_tokens
        kp = (torch.randn((8, T, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        vp = (torch.randn((8, T, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        q = (torch.randn((f.bs, 32, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        kx, vx, pt = paged_pools(f, kp, vp, page, n_phys_pages=page_layout(f, page)[1] + 3, generator=gen)
        h0, h1, g = 2, 6, 4
        plan = P.plan_device(f, g, table, h1 - h0, 148, page_size=page)
        qs = q[:, h0 * g:h1 * g].contiguous()
        ref = DecodeStep(f, plan, 32, "bfloat16", head_begin=h0, head_end=h1)(
            qs, kp[h0:h1].contiguous(), vp[h0:h1].contiguous())
        got = DecodeStep(f, plan, 32, "bfloat16", head_begin=h0, head_end=h1, page_size=page, page_table=pt,
                         pool_tokens=kx.shape[1])(qs, kx[h0:h1].contiguous(), vx[h0:h1].contiguous())
        torch.cuda.synchronize()
        assert torch.isfinite(ref).all()
        assert torch.equal(ref, got), (page, float((ref - got).abs().max()))
        from oracle import attention as OA
        up = lambda t: t.double().cpu().numpy()
        kp_h, vp_h = up(kp), up(vp)
        z = np.zeros((0, 8, 128))
        node_k = [z] + [kp_h[:, f.token_offset[n]:f.token_offset[n] + f.nodes[n].len].transpose(1, 0, 2)
                        for n in range(1, len(f.nodes))]
        node_v = [z] + [vp_h[:, f.token_offset[n]:f.token_offset[n] + f.nodes[n].len].transpose(1, 0, 2)
                        for n in range(1, len(f.nodes))]
        want = OA.naive_attention(up(q), OA.ForestData(spec.parent, node_k, node_v, spec.paths))[:, h0 * g:h1 * g]
        err = np.abs(got.double().cpu().numpy() - want)
        assert err.max() <= 2e-3 and err.max() / np.abs(want).max() <= 1e-2, (page, float(err.max()))
