"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the golden vectors recorded from the reference. Needs a B200."""
from __future__ import annotations

import io
import math

import numpy as np
import pytest

from conftest import golden_json, golden_npz, golden_table_text, rel_err
from recipes import PAC_SHAPES, pac_inputs, random_forest_spec
from oracle import attention as OA
import paper_2505_17694_b200 as P
from paper_2505_17694_b200 import workloads as W
from paper_2505_17694_b200.executor import (FLAG_FORCE_TC, FLAG_NO_GEMV, FLAG_NO_MULTI, FLAG_NO_TC, FLAG_NO_TCT,
                                            FLAG_TCT_WIDE, DecodeStep)

pytestmark = pytest.mark.gpu

BF16_ABS, BF16_REL = 2e-3, 1e-2   # north-star tolerance for bf16 KV (BASELINE.json)


@pytest.fixture(scope="module")
def table():
    return P.load_profile(io.StringIO(golden_table_text("a100_d128.csv")))


def np_(t):
    return t.detach().double().cpu().numpy()


def oracle_forest(spec):
    z = np.zeros((0, spec.h_kv, spec.d))
    return OA.ForestData(spec.parent, [z] + [np.asarray(k, np.float64) for k in spec.keys[1:]],
                         [z] + [np.asarray(v, np.float64) for v in spec.values[1:]], spec.paths, spec.visible)


def build(spec, dtype=None):
    specs = spec.node_specs()
    q = spec.queries
    if dtype is not None:
        import torch
        tdt = {"bfloat16": torch.bfloat16, "float32": torch.float32}[dtype]
        specs = [(p, torch.from_numpy(np.ascontiguousarray(k)).to(tdt), torch.from_numpy(np.ascontiguousarray(v)).to(tdt), vis)
                 for p, k, v, vis in specs]
        q = torch.from_numpy(np.ascontiguousarray(q)).to(tdt)
    qb = P.QueryBatch(q, spec.h_kv)
    return P.build_forest(specs, spec.paths, qb), qb


def upcast_spec(spec, dtype="bfloat16"):
    """The spec's tensors rounded to `dtype` and back to float64: the
    oracle then sees exactly the values the GPU sees."""
    import torch
    tdt = {"bfloat16": torch.bfloat16, "float32": torch.float32}[dtype]
    r = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(tdt).double().numpy()
    out = W.Spec(spec.h_q, spec.h_kv, spec.d, list(spec.parent), list(spec.length),
                 [None] + [r(k) for k in spec.keys[1:]], [None] + [r(v) for v in spec.values[1:]],
                 list(spec.paths), r(spec.queries), spec.visible)
    return out


def assert_bf16_close(out, ref):
    out, ref = np.asarray(out, np.float64), np.asarray(ref, np.float64)
    assert np.isfinite(out).all()
    err = float(np.max(np.abs(out - ref)))
    assert err <= BF16_ABS, err
    assert rel_err(out, ref) <= BF16_REL, rel_err(out, ref)


# ----------------------------------------------------------------- pac / por
class TestPacGolden:
    def test_known_answers(self, cuda_ok):
        a = lambda *x: np.asarray(x, np.float64).reshape(-1, 1, 1)
        p = P.pac(a(2.0), a(3.0), a(7.0))
        assert (np_(p.out).item(), np_(p.max_score).item(), np_(p.exp_sum).item()) == (7.0, 6.0, 1.0)
        p = P.pac(a(1.0), a(0.0, 0.0), a(2.0, 4.0))
        assert np_(p.out).item() == pytest.approx(3.0, abs=1e-15)
        p = P.pac(a(2.0), a(3.0, 5.0), a(7.0, 11.0))
        assert np_(p.out).item() == pytest.approx(10.928055160152, rel=1e-12)
        assert np_(p.max_score).item() == 10.0
        assert np_(p.exp_sum).item() == pytest.approx(1.0183156388887, rel=1e-12)
        d = 16
        p = P.pac(np.ones((1, 1, d)), np.ones((1, 1, d)), np.ones((1, 1, d)))
        assert np_(p.max_score).item() == pytest.approx(4.0, rel=1e-15)

    def test_extreme_scores(self, cuda_ok):
        a = lambda *x: np.asarray(x, np.float64).reshape(-1, 1, 1)
        p = P.pac(np.ones((1, 1, 1)), a(500.0, -500.0, 250.0, -250.0, 0.0), a(1.0, 2.0, 3.0, 4.0, 5.0))
        assert np.isfinite(np_(p.out)).all() and np_(p.out).item() == pytest.approx(1.0, rel=1e-8)
        lo = P.pac(np.ones((1, 1, 1)), a(-500.0), a(2.0))
        hi = P.pac(np.ones((1, 1, 1)), a(500.0), a(3.0))
        m = P.por(lo, hi)
        assert np_(m.out).item() == pytest.approx(3.0, rel=1e-12) and np_(m.max_score).item() == 500.0

    @pytest.mark.parametrize("i", range(len(PAC_SHAPES)))
    @pytest.mark.parametrize("masked", [False, True])
    def test_float64_goldens(self, cuda_ok, i, masked):
        z = golden_npz()
        q, k, v, vis = pac_inputs(PAC_SHAPES[i], masked=masked)
        p = P.pac(q, k, v, visible=vis)
        tag = f"{i}_{int(masked)}"
        assert rel_err(np_(p.out), z[f"pac_out_{tag}"]) <= 1e-12
        assert rel_err(np_(p.max_score), z[f"pac_m_{tag}"]) <= 1e-12
        assert rel_err(np_(p.exp_sum), z[f"pac_s_{tag}"]) <= 1e-12

    @pytest.mark.parametrize("i", [1, 2, 4])
    def test_float32(self, cuda_ok, i):
        z = golden_npz()
        q, k, v, vis = pac_inputs(PAC_SHAPES[i], dtype=np.float32, masked=True)
        p = P.pac(q, k, v, visible=vis)
        assert rel_err(np_(p.out), z[f"pac_out_{i}_1"]) <= 1e-4

    def test_gqa_equals_expanded(self, cuda_ok):
        rng = np.random.default_rng(1234)
        h_kv, g, d, n = 2, 4, 8, 12
        q = rng.standard_normal((3, h_kv * g, d))
        k = rng.standard_normal((n, h_kv, d))
        v = rng.standard_normal((n, h_kv, d))
        kvmap = np.arange(h_kv * g) // g
        a, b = P.pac(q, k, v), P.pac(q, k[:, kvmap, :], v[:, kvmap, :])
        assert np.array_equal(np_(a.out), np_(b.out))

    def test_errors(self, cuda_ok):
        from paper_2505_17694_b200.errors import DimensionMismatch, EmptyVisibleSet, NoVisibleTokens, ShapeMismatch
        a = lambda *x: np.asarray(x, np.float64).reshape(-1, 1, 1)
        with pytest.raises(EmptyVisibleSet, match="1..2"):
            P.pac(a(1.0), a(0.0, 0.0), a(1.0, 2.0), visible=[0])
        with pytest.raises(DimensionMismatch, match="multiple"):
            P.pac(np.zeros((1, 3, 4)), np.zeros((2, 2, 4)), np.zeros((2, 2, 4)))
        with pytest.raises(ShapeMismatch, match="shapes differ"):
            P.por(P.empty_partial(1, 1, 2), P.empty_partial(1, 1, 3))
        with pytest.raises(NoVisibleTokens):
            P.finalize(P.empty_partial(1, 1, 1))


class TestPor:
    def test_matches_concatenation(self, cuda_ok):
        rng = np.random.default_rng(5)
        k = rng.standard_normal((10, 2, 8))
        v = rng.standard_normal((10, 2, 8))
        q = rng.standard_normal((3, 4, 8))
        whole = P.pac(q, k, v)
        split = P.por(P.pac(q, k[:4], v[:4]), P.pac(q, k[4:], v[4:]))
        assert rel_err(np_(split.out), np_(whole.out)) <= 1e-12
        assert np.array_equal(np_(split.max_score), np_(whole.max_score))

    def test_identity_and_elementwise_empty(self, cuda_ok):
        rng = np.random.default_rng(6)
        x = P.pac(rng.standard_normal((2, 2, 4)), rng.standard_normal((5, 2, 4)), rng.standard_normal((5, 2, 4)))
        e = P.empty_partial(2, 2, 4)
        for mgd in (P.por(x, e), P.por(e, x)):
            assert np.array_equal(np_(mgd.out), np_(x.out))
        y = x.copy()
        y.exp_sum[0, 1] = 0.0
        y.max_score[0, 1] = float("-inf")
        y.out[0, 1] = 0.0
        r = P.por(y, P.pac(rng.standard_normal((2, 2, 4)), rng.standard_normal((3, 2, 4)),
                           rng.standard_normal((3, 2, 4))))
        assert np.isfinite(np_(r.out)).all()


# ----------------------------------------------------------------- execute
class TestExecuteGolden:
    """execute() on the reference's random forests vs the reference's own
    execute/naive outputs (test_executor.py:104-110, acceptance :40-59)."""

    def test_float64(self, cuda_ok, table):
        z = golden_npz()
        worst = 0.0
        for doc in golden_json("forests.json")["forests"]:
            spec = random_forest_spec(doc["seed"], with_masks=doc["masks"])
            f, q = build(spec)
            tasks = P.tasks_from_forest(f)
            plan_u = P.plan_uniform_bk(tasks, table, 4, doc["bk"])
            plan_a = P.divide_and_schedule(tasks, table, 4)
            for plan, key in ((plan_u, "exec_u"), (plan_a, "exec_a")):
                out = np_(P.execute(f, q, plan, P.BlockPool(4)))
                worst = max(worst, rel_err(out, z[f"{key}_{doc['seed']}"]))
                assert rel_err(out, z[f"naive_{doc['seed']}"]) <= 1e-10
        assert worst <= 1e-10

    def test_float32(self, cuda_ok, table):
        z = golden_npz()
        for doc in golden_json("forests.json")["forests"]:
            spec = random_forest_spec(doc["seed"], with_masks=doc["masks"])
            f, q = build(spec, "float32")
            plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 4, doc["bk"])
            out = np_(P.execute(f, q, plan))
            assert rel_err(out, z[f"naive_{doc['seed']}"]) <= 1e-3
            assert rel_err(out, z[f"exec32_{doc['seed']}"]) <= 1e-3

    def test_float32_generic_kernel(self, cuda_ok, table):
        z = golden_npz()
        for doc in golden_json("forests.json")["forests"][:12]:
            spec = random_forest_spec(doc["seed"], with_masks=doc["masks"])
            f, q = build(spec, "float32")
            plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 4, doc["bk"])
            out = np_(P.execute(f, q, plan, flags=FLAG_NO_GEMV))
            assert rel_err(out, z[f"naive_{doc['seed']}"]) <= 1e-3


def d128_forest(seed, with_masks):
    """random_forest recipe with d=128, g=4, h_kv=2: the head shape the
    tensor-core and GEMV kernels specialise on."""
    rng = np.random.default_rng(10_000 + seed)
    spec = random_forest_spec(seed, with_masks=with_masks, max_bs=16)
    h_kv, g, d = 2, 4, 128
    sc = 1.0 / math.sqrt(d)
    spec.h_q, spec.h_kv, spec.d = h_kv * g, h_kv, d
    spec.keys = [None] + [rng.standard_normal((n, h_kv, d)) * sc for n in spec.length[1:]]
    spec.values = [None] + [rng.standard_normal((n, h_kv, d)) * sc for n in spec.length[1:]]
    spec.queries = rng.standard_normal((spec.bs, h_kv * g, d)) * sc
    return spec


class TestBf16Kernels:
    @pytest.mark.parametrize("flags", [0, FLAG_FORCE_TC, FLAG_NO_TC, FLAG_NO_MULTI, FLAG_NO_TC | FLAG_NO_MULTI,
                                       FLAG_NO_TCT, FLAG_NO_MULTI | FLAG_NO_TCT, 1048576, FLAG_FORCE_TC | 1048576])
    def test_random_forests(self, cuda_ok, table, flags):
        for seed in range(24):
            spec = d128_forest(seed, with_masks=(seed % 2 == 1))
            f, q = build(spec, "bfloat16")
            plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 4, 1 + seed % 3)
            out = np_(P.execute(f, q, plan, flags=flags))
            ups = upcast_spec(spec)
            ref = OA.naive_attention(ups.queries, oracle_forest(ups))
            assert_bf16_close(out, ref)

    def test_cfg1_float32(self, cuda_ok, table):
        spec = W.make_config("cfg1", dtype=np.float32)
        f, q = build(spec)
        plan = P.divide_and_schedule(P.tasks_from_forest(f), table, 8)
        out = np_(P.execute(f, q, plan))
        ref = OA.naive_attention(np.asarray(spec.queries, np.float64), oracle_forest(spec))
        assert rel_err(out, ref) <= 1e-3

    def test_shared_root_device_plan(self, cuda_ok, table):
        """cfg2 shape at reduced size: TC kernel on the split root, GEMV on
        suffixes, LSE merge; device-level (row-chunk) plan."""
        spec = W.two_level(4096, 128, 64, h_q=32, h_kv=8, d=128, seed=1, dtype=None)
        f, q = build(spec, "bfloat16")
        tasks = P.device_tasks(f, group_size=4)
        plan = P.divide_and_schedule(tasks, table, 18)
        step = DecodeStep(f, plan, 32, "bfloat16")
        assert step.info.n_tc_groups > 0 and step.info.n_gemv_groups > 0
        out = np_(P.execute(f, q, plan))
        ups = upcast_spec(spec)
        ref = OA.naive_attention(ups.queries, oracle_forest(ups))
        assert_bf16_close(out, ref)

    def test_repeatable_bitwise(self, cuda_ok, table):
        spec = d128_forest(3, with_masks=True)
        f, q = build(spec, "bfloat16")
        plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 4, 2)
        a = np_(P.execute(f, q, plan, flags=FLAG_FORCE_TC))
        b = np_(P.execute(f, q, plan, flags=FLAG_FORCE_TC))
        assert np.array_equal(a, b)

    def test_plan_mismatch_errors(self, cuda_ok, table):
        from paper_2505_17694_b200.errors import PlanForestMismatch
        big = P.build_forest([(0, *[np.random.default_rng(0).standard_normal((8, 1, 8))] * 2),
                              (1, *[np.random.default_rng(1).standard_normal((8, 1, 8))] * 2)], [(1, 2)])
        small = P.build_forest([(0, *[np.random.default_rng(0).standard_normal((8, 1, 8))] * 2)], [(1,)])
        q = P.QueryBatch(np.zeros((1, 1, 8)), 1)
        plan = P.plan_uniform_bk(P.tasks_from_forest(small), table, 1, 1)
        with pytest.raises(PlanForestMismatch, match="plan covers nodes"):
            P.execute(big, q, plan)
        donor = P.build_forest([(0, *[np.zeros((10, 1, 8))] * 2)], [(1,)])
        target = P.build_forest([(0, *[np.zeros((12, 1, 8))] * 2)], [(1,)])
        plan = P.plan_uniform_bk(P.tasks_from_forest(donor), table, 1, 2)
        with pytest.raises(PlanForestMismatch, match="do not tile"):
            P.execute(target, q, plan)


class TestConcurrency:
    def test_aux_stream_and_budgets(self, cuda_ok, table):
        """The aux stream changes scheduling only (bit-identical results);
        a different TC SM budget re-cuts the stream-K pieces, which changes
        the partial-merge rounding only."""
        spec = W.two_level(2048, 200, 96, h_q=32, h_kv=8, d=128, seed=4)
        f, q = build(spec, "bfloat16")
        plan = P.divide_and_schedule(P.device_tasks(f, group_size=4), table, 37)
        kp, vp = f.device_pool("bfloat16")
        qd = q.queries.cuda()
        serial = DecodeStep(f, plan, 32, "bfloat16", concurrent=False)
        base = np_(serial(qd, kp, vp))
        conc = DecodeStep(f, plan, 32, "bfloat16", concurrent=True)
        assert np.array_equal(np_(conc(qd, kp, vp)), base)
        for budget in (120, 64):
            other = np_(DecodeStep(f, plan, 32, "bfloat16", concurrent=True, tc_sm_budget=budget)(qd, kp, vp))
            # other piece boundaries: other bf16 roundings of P (well inside the bf16 bar)
            assert np.max(np.abs(other - base)) <= 1e-2 * float(np.max(np.abs(base)))
        best, times = P.autotune_step(DecodeStep(f, plan, 32, "bfloat16"), qd, kp, vp, budgets=[148, 96], iters=2)
        assert np.max(np.abs(np_(best(qd, kp, vp)) - base)) <= 1e-2 * float(np.max(np.abs(base)))
        ups = upcast_spec(spec)
        assert_bf16_close(base, OA.naive_attention(ups.queries, oracle_forest(ups)))

    def test_repeat_launch_deterministic(self, cuda_ok, table):
        """Back-to-back launches over the same workspace give identical outputs."""
        spec = d128_forest(5, with_masks=True)
        f, q = build(spec, "bfloat16")
        plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 4, 2)
        outs = [np_(P.execute(f, q, plan, flags=FLAG_NO_TC)) for _ in range(4)]
        for o in outs[1:]:
            assert np.array_equal(o, outs[0])
        ups = upcast_spec(spec)
        assert_bf16_close(outs[0], OA.naive_attention(ups.queries, oracle_forest(ups)))


class TestSuffixPaths:
    """The suffix (unshared-node) groups run on the mma.sync kernel and the
    merge kernel combines the partials; CODEC_FLAG_FUSED_MERGE makes the
    suffix kernel fold each request's TC partials into its output itself,
    CODEC_FLAG_GEMV_SIMT swaps in the CUDA-core GEMV kernel. All three agree
    with the oracle, with and without ragged visibility."""

    @pytest.mark.parametrize("with_masks", [False, True])
    def test_paths_agree(self, cuda_ok, table, with_masks):
        spec = W.two_level(1500, 300, 40, h_q=32, h_kv=8, d=128, seed=11)
        if with_masks:
            spec = d128_forest(12, with_masks=True)
        f, q = build(spec, "bfloat16")
        plan = P.plan_device(f, spec.h_q // spec.h_kv, table, spec.h_kv, 148)
        kp, vp = f.device_pool("bfloat16")
        qd = q.queries.cuda()
        outs = {}
        for name, fl in (("fused", 4096), ("merge_kernel", 0), ("simt", 2048)):
            st = DecodeStep(f, plan, spec.h_q, "bfloat16", flags=fl, concurrent=False)
            if name == "fused" and not with_masks:
                assert st.info.n_merge_fused > 0
            outs[name] = np_(st(qd, kp, vp))
        ups = upcast_spec(spec)
        ref = OA.naive_attention(ups.queries, oracle_forest(ups))
        for name, o in outs.items():
            assert_bf16_close(o, ref)
        scale = float(np.max(np.abs(outs["merge_kernel"])))
        assert np.max(np.abs(outs["fused"] - outs["merge_kernel"])) <= 1e-4 * scale


def _full_config(name, seed=0):
    """A BASELINE.json config at full size: structure from workloads, bf16
    K/V/Q drawn on the device (seeded), the device plan and step."""
    import torch
    spec = W.make_config(name, tensors=False)
    h_q, h_kv, d = spec.h_q, spec.h_kv, spec.d
    f = P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, h_kv, d)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    sc = 1.0 / math.sqrt(d)
    T = f.total_tokens
    kp = (torch.randn((h_kv, T, d), generator=gen, device="cuda") * sc).to(torch.bfloat16)
    vp = (torch.randn((h_kv, T, d), generator=gen, device="cuda") * sc).to(torch.bfloat16)
    q = (torch.randn((f.bs, h_q, d), generator=gen, device="cuda") * sc).to(torch.bfloat16)
    table = P.load_default_profile()
    plan = P.plan_device(f, h_q // h_kv, table, h_kv, torch.cuda.get_device_properties(0).multi_processor_count)
    return f, kp, vp, q, DecodeStep(f, plan, h_q, "bfloat16", concurrent=False)


def _path_reference(f, kp, vp, q, r):
    """Single-softmax attention of request r over its root-to-leaf path
    (naive_attention, attention.py:164-187) in float64 on the device, from
    the same bf16 values: a plain torch reference for full-size checks."""
    import torch
    toks = torch.cat([torch.arange(f.token_offset[n], f.token_offset[n] + f.visible_count(n, r), device="cuda")
                      for n in f.paths[r]])
    g = q.shape[1] // f.h_kv
    k = kp[:, toks].double()                      # [h_kv, L, d]
    v = vp[:, toks].double()
    qq = q[r].double().view(f.h_kv, g, -1)        # [h_kv, g, d]
    s = torch.einsum("hgd,hld->hgl", qq, k) / math.sqrt(f.d)
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hgl,hld->hgd", p, v).reshape(q.shape[1], -1)


class TestFullConfigs:
    """cfg3 (tree-of-thought), cfg4 (imbalanced 64-tree forest, 17.5 GB of
    KV) and cfg5 (Llama-3-70B shape) at their BASELINE.json sizes through
    the device path; sampled requests against a float64 reference of the
    same bf16 inputs, the bf16 bar (max-abs 2e-3 and rel 1e-2)."""

    @pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
    def test_sampled_requests(self, cuda_ok, name):
        import torch
        f, kp, vp, q, step = _full_config(name, seed=7)
        out = step(q, kp, vp)
        torch.cuda.synchronize()
        assert bool(torch.isfinite(out).all())
        rng = np.random.default_rng(3)
        # spread over the forest, shortest paths first for cfg4 (prefixes up to 128K tokens)
        lens = np.array([f.request_len(r) for r in range(f.bs)])
        pool = np.argsort(lens)[: max(8, f.bs // 4)] if name == "cfg4" else np.arange(f.bs)
        for r in sorted(set(rng.choice(pool, size=min(6, len(pool)), replace=False).tolist()) | {f.bs - 1}):
            ref = _path_reference(f, kp, vp, q, r)
            got = out[r].double()
            err = float((got - ref).abs().max())
            rel = err / float(ref.abs().max())
            assert err <= 2e-3 and rel <= 1e-2, (name, r, err, rel)
        del kp, vp
        torch.cuda.empty_cache()


class TestGraph:
    def test_capture_replay_matches(self, cuda_ok, table):
        """DecodeStep.capture(): a CUDA-graph replay of the step gives the
        direct call's result bit for bit, also after new query values are
        written into the captured buffer."""
        import torch
        spec = W.two_level(3000, 200, 48, h_q=32, h_kv=8, d=128, seed=21)
        f, q = build(spec, "bfloat16")
        plan = P.plan_device(f, 4, table, 8, 148)
        kp, vp = f.device_pool("bfloat16")
        qd = q.queries.cuda().contiguous()
        step = DecodeStep(f, plan, 32, "bfloat16", concurrent=False)
        out = torch.empty((f.bs, 32, 128), dtype=torch.float32, device="cuda")
        replay = step.capture(qd, kp, vp, out)
        for trial in range(2):
            if trial:
                qd.copy_((torch.randn_like(qd, dtype=torch.float32) * 0.1).to(torch.bfloat16))
            replay()
            torch.cuda.synchronize()
            direct = step(qd, kp, vp)
            assert np.array_equal(np_(out), np_(direct))


class TestGrow:
    def test_grow_matches_rebuilt_step(self, cuda_ok, table):
        """DecodeStep.grow(): leaves built with spare capacity (visible_len
        below their length) grow one token per decode step in the device
        table; each grown step equals a step built from scratch on a forest
        whose visible counts include the new tokens -- also through a
        captured CUDA graph."""
        import torch
        bs, shared, cap, start = 24, 2048, 160, 100
        spec = W.two_level(shared, cap, bs, h_q=32, h_kv=8, d=128, seed=5, tensors=False)

        def forest(leaf_visible):  # node 1 = the shared root, node 2 + r = request r's leaf
            return P.forest_from_pool(spec.parent[1:], spec.length[1:], spec.paths, 8, 128,
                                      visible=[None] + [{r: leaf_visible} for r in range(bs)])

        f0 = forest(start)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(3)
        shape = (8, f0.total_tokens, 128)
        kp = (torch.randn(shape, generator=gen, device="cuda") / math.sqrt(128)).to(torch.bfloat16)
        vp = (torch.randn(shape, generator=gen, device="cuda") / math.sqrt(128)).to(torch.bfloat16)
        q = (torch.randn((bs, 32, 128), generator=gen, device="cuda") / math.sqrt(128)).to(torch.bfloat16)
        step = DecodeStep(f0, P.plan_device(f0, 4, table, 8, 148), 32, "bfloat16", concurrent=False)
        out = torch.empty((bs, 32, 128), dtype=torch.float32, device="cuda")
        replay = step.capture(q, kp, vp, out)
        for k in range(1, 4):
            step.grow(1)
            replay()
            torch.cuda.synchronize()
            f2 = forest(start + k)
            ref = DecodeStep(f2, P.plan_device(f2, 4, table, 8, 148), 32, "bfloat16", concurrent=False)(q, kp, vp)
            assert np.array_equal(np_(out), np_(ref)), k
            # and the grown step against the float64 oracle on the same bf16
            # values (root + each leaf's first start + k tokens)
            up = lambda t: t.double().cpu().numpy()
            kph, vph = up(kp), up(vp)
            z = np.zeros((0, 8, 128))
            nk = [z] + [kph[:, f2.token_offset[n]:f2.token_offset[n] + spec.length[n]].transpose(1, 0, 2)
                        for n in range(1, len(spec.parent))]
            nv = [z] + [vph[:, f2.token_offset[n]:f2.token_offset[n] + spec.length[n]].transpose(1, 0, 2)
                        for n in range(1, len(spec.parent))]
            vis = [None, None] + [{r: start + k} for r in range(bs)]
            fd = OA.ForestData(spec.parent, nk, nv, spec.paths, vis)
            assert_bf16_close(np_(out), OA.naive_attention(up(q), fd))
        with pytest.raises(ValueError, match="no room"):
            step.grow(cap)


class TestReduceTree:
    def test_partial_tree_matches_goldens(self, cuda_ok, table):
        """reduce_tree() over a PartialTree built like the reference's split
        phase (executor.py:145-206: rows with visible > start, per-row
        visible clipped to the slice) from codec_pac partials equals the
        reference's execute() / naive outputs (fp64, 1e-10)."""
        z = golden_npz()
        for doc in golden_json("forests.json")["forests"][:16]:
            spec = random_forest_spec(doc["seed"], with_masks=doc["masks"])
            f, q = build(spec)
            plan = P.plan_uniform_bk(P.tasks_from_forest(f), table, 4, doc["bk"])
            pt = P.PartialTree()
            qq = np.asarray(q.queries)
            for st in plan.subtasks:
                si = pt.slice_count.get(st.node, 0)
                pt.slice_count[st.node] = si + 1
                rows = tuple(r for r in f.node(st.node).query_set if f.visible_count(st.node, r) > st.start)
                if not rows:
                    continue
                vis = [min(f.visible_count(st.node, r), st.stop) - st.start for r in rows]
                node = f.node(st.node)
                pt.entries[(st.node, si)] = P.pac(qq[list(rows)], node.keys[st.start:st.stop],
                                                  node.values[st.start:st.stop], visible=vis)
                pt.rows[(st.node, si)] = rows
            out = np_(P.reduce_tree(pt, f, P.BlockPool(1)))
            assert rel_err(out, z[f"exec_u_{doc['seed']}"]) <= 1e-10
            assert rel_err(out, z[f"naive_{doc['seed']}"]) <= 1e-10


class TestMultiRequestKernel:
    @pytest.mark.parametrize("g", [1, 2, 4, 8])
    def test_lightly_shared_nodes(self, cuda_ok, table, g):
        """Nodes shared by 2..16 requests: those with <= 16 query-head rows
        on the multi-request mma.sync kernel, the others on the tensor
        cores; ragged visible counts per
        request inside a group (per-column masks), against the oracle and
        against the same plan with the kernel off (per-request suffix
        kernel)."""
        import torch
        rng = np.random.default_rng(40 + g)
        h_kv = 4
        parent, length, paths, vis = [0], [0], [], [None]
        for t in range(6):
            root = len(parent)
            parent.append(0)
            length.append(int(rng.integers(100, 3000)))
            vis.append(None)
            for _ in range(2 if t == 0 else int(rng.integers(2, 17))):  # root 0: 2 requests
                parent.append(root)
                length.append(int(rng.integers(5, 200)))
                vis.append(None)
                paths.append((root, len(parent) - 1))
        bs = len(paths)
        for r, (root, leaf) in enumerate(paths):  # ragged visibility in the shared roots
            if rng.random() < 0.4:
                vis[root] = vis[root] or {}
                vis[root][r] = int(rng.integers(1, length[root] + 1))
        spec = W.Spec(h_kv * g, h_kv, 128, parent, length, None, None, paths, None, vis)
        f = P.forest_from_pool(parent[1:], length[1:], paths, h_kv, 128, visible=vis[1:])
        gen = torch.Generator().manual_seed(g)
        T = f.total_tokens
        kp = (torch.randn((h_kv, T, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        vp = (torch.randn((h_kv, T, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        q = (torch.randn((bs, h_kv * g, 128), generator=gen) * 0.088).to(torch.bfloat16).cuda()
        # the multi-request kernel takes these slices when the transposed
        # tensor-core kernel is off (by default that one takes 2+ requests)
        plan = P.plan_device(f, g, table, h_kv, 148, tct=False)
        multi = DecodeStep(f, plan, h_kv * g, "bfloat16", flags=FLAG_NO_TCT)
        assert multi.info.n_multi_groups > 0  # root 0: 2 requests = 2 g <= 16 rows
        got = np_(multi(q, kp, vp))
        off = np_(DecodeStep(f, plan, h_kv * g, "bfloat16", flags=FLAG_NO_MULTI | FLAG_NO_TCT)(q, kp, vp))
        tct = DecodeStep(f, P.plan_device(f, g, table, h_kv, 148), h_kv * g, "bfloat16")
        assert tct.info.n_tct_groups > 0 and tct.info.n_multi_groups == 0
        z = np.zeros((0, h_kv, 128))
        node = lambda pool, n: pool[:, f.token_offset[n]:f.token_offset[n] + length[n]].permute(1, 0, 2).double().cpu().numpy()
        fd = OA.ForestData(parent, [z] + [node(kp, n) for n in range(1, len(parent))],
                           [z] + [node(vp, n) for n in range(1, len(parent))], paths, vis)
        ref = OA.naive_attention(q.double().cpu().numpy(), fd)
        assert_bf16_close(got, ref)
        assert_bf16_close(off, ref)
        assert_bf16_close(np_(tct(q, kp, vp)), ref)
        # the same inputs, the same step: bit-repeatable
        assert np.array_equal(np_(multi(q, kp, vp)), got)


class TestTransposedKernel:
    @pytest.mark.parametrize("g,counted,wide", [(g, c, w) for g in (2, 4, 8) for c in (0, 1048576)
                                                 for w in (False, True)] + [(1, 0, False), (16, 0, True)])
    def test_lightly_shared_roots(self, cuda_ok, table, g, counted, wide):
        """Roots read by 17..128 query-head rows (kern_tct.cu: tokens on the
        MMA's M, rows on N): several KV slices per root (TCT_SLICE), 16..64
        rows per CTA, ragged visible counts inside a group (per-column
        masks), and a band of large keys in the middle of some roots so a
        later tile passes the column references (the rescale of O^T in
        TMEM). Against the float64 oracle and the same plan with the kernel
        off (the M = 256 pair kernel), bit-repeatable."""
        import torch
        rng = np.random.default_rng(70 + g)
        h_kv = 4
        parent, length, paths, vis = [0], [0], [], [None]
        for t in range(6):
            root = len(parent)
            parent.append(0)
            length.append(int(rng.integers(300, 9000)))
            vis.append(None)
            n_req = int(rng.integers(max(2, 17 // g + 1), 128 // g + 1))
            for _ in range(n_req):
                parent.append(root)
                length.append(int(rng.integers(5, 200)))
                vis.append(None)
                paths.append((root, len(parent) - 1))
        bs = len(paths)
        for r, (root, leaf) in enumerate(paths):
            if rng.random() < 0.4:
                vis[root] = vis[root] or {}
                vis[root][r] = int(rng.integers(1, length[root] + 1))
        f = P.forest_from_pool(parent[1:], length[1:], paths, h_kv, 128, visible=vis[1:])
        gen = torch.Generator().manual_seed(g)
        T = f.total_tokens
        kp = torch.randn((h_kv, T, 128), generator=gen) * 0.088
        vp = torch.randn((h_kv, T, 128), generator=gen) * 0.088
        q = torch.randn((bs, h_kv * g, 128), generator=gen) * 0.5
        for n in range(1, len(parent), 3):  # large keys past the first tiles of every third node
            a = f.token_offset[n] + min(length[n] - 1, 700)
            kp[:, a:a + 40] *= 60.0
        kp, vp, q = (x.to(torch.bfloat16).cuda() for x in (kp, vp, q))
        plan = P.plan_device(f, g, table, h_kv, 148, tct_wide=wide)
        step = DecodeStep(f, plan, h_kv * g, "bfloat16", flags=counted | (FLAG_TCT_WIDE if wide else 0))
        assert step.info.n_tct_groups > 0 and (step.info.n_tct_wide > 0) == wide
        got = np_(step(q, kp, vp))
        off = np_(DecodeStep(f, P.plan_device(f, g, table, h_kv, 148, tct=False), h_kv * g, "bfloat16",
                             flags=FLAG_NO_TCT)(q, kp, vp))
        z = np.zeros((0, h_kv, 128))
        node = lambda pool, n: pool[:, f.token_offset[n]:f.token_offset[n] + length[n]].permute(1, 0, 2).double().cpu().numpy()
        fd = OA.ForestData(parent, [z] + [node(kp, n) for n in range(1, len(parent))],
                           [z] + [node(vp, n) for n in range(1, len(parent))], paths, vis)
        ref = OA.naive_attention(q.double().cpu().numpy(), fd)
        assert_bf16_close(got, ref)
        assert_bf16_close(off, ref)
        assert np.array_equal(np_(step(q, kp, vp)), got)
