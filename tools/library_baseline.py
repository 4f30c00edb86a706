"""The bench's cfg2 decode step beside FlashInfer's B200 decode kernels on the
same box, same KV bytes, same windows (a library reference point, not the
reference arm; FlashInfer is library code in this image).

    python tools/library_baseline.py [seconds] [page_size] [config] [tc_sm_budget]

(config: any two-level workload -- cfg2 (default, budget 96) or cfg5 (128).)

FlashInfer arm: the KV of the bench's own pools is copied into a paged cache
(HND, `page_size` tokens per page) in which the 32K-token system prompt's
pages are SHARED by all 256 requests' block tables (prefix caching as a
serving engine does it) and each request's 512 suffix tokens have their own
pages; `trtllm_batch_decode_with_kv_cache` (the trtllm-gen Blackwell decode
kernels FlashInfer ships as cubins) then runs one decode query per request
over its 33,280 tokens -- the FlashDecoding-style per-request schedule the
north star compares unique-KV bytes against (metrics.py:55-70). Both arms
are timed in >= `seconds` of back-to-back 20-step windows (median), the
bench's method -- ours as a CUDA-graph replay, FlashInfer's call directly
(its wrapper does not survive stream capture; at ms-scale device time the
host launch is hidden); outputs are compared with each other.
"""
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def windows(fn, secs, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    clk = bench.ClockSampler(0)
    ws, t0 = [], time.perf_counter()
    while time.perf_counter() - t0 < secs:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ws.append(e0.elapsed_time(e1) / n * 1e3)
    c = clk.stop() or {}
    return {"us": statistics.median(ws), "best_us": min(ws), "windows": len(ws), "sm_mhz": c.get("sm_mhz"),
            "power_w": c.get("power_w_median"), "reasons": c.get("reasons")}


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g.replay


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    ps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    dev = torch.device("cuda", 0)
    config = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
    budget = int(sys.argv[4]) if len(sys.argv) > 4 else 96
    ns = bench.prepare(config, dev, budgets=[budget])
    f, kp, vp, q = ns.forest, ns.kp, ns.vp, ns.q_dev
    bs, h_kv, d = f.bs, kp.shape[0], kp.shape[2]
    res = {"workload": ns.cfg["label"], "page_size": ps, "tc_sm_budget": budget}

    ours = ns.step.capture(q, kp, vp, ns.out)
    res["ours"] = windows(ours, secs)
    ours()
    torch.cuda.synchronize()
    out_ours = ns.out.clone()

    # paged cache: shared prefix pages, then each request's suffix pages
    root = f.paths[0][0]
    pre_len = f.nodes[root].len if hasattr(f.nodes[root], "len") else None
    n_pre = pre_len // ps
    toks = [torch.arange(f.token_offset[root], f.token_offset[root] + pre_len, device=dev).view(n_pre, ps)]
    tables = []
    nxt = n_pre
    for r in range(bs):
        leaf = f.paths[r][-1]
        L = f.visible_count(leaf, r)
        assert L % ps == 0 and len(f.paths[r]) == 2 and f.paths[r][0] == root
        toks.append(torch.arange(f.token_offset[leaf], f.token_offset[leaf] + L, device=dev).view(L // ps, ps))
        tables.append(list(range(n_pre)) + list(range(nxt, nxt + L // ps)))
        nxt += L // ps
    tok = torch.cat(toks)                                     # [pages, ps]
    kc = kp[:, tok].permute(1, 0, 2, 3).contiguous()          # [pages, h_kv, ps, d]
    vc = vp[:, tok].permute(1, 0, 2, 3).contiguous()
    bt = torch.tensor(tables, dtype=torch.int32, device=dev)
    seq = torch.tensor([pre_len + f.visible_count(f.paths[r][-1], r) for r in range(bs)], dtype=torch.int32,
                       device=dev)
    res["paged_cache_bytes"] = 2 * kc.numel() * kc.element_size()
    res["per_request_bytes"] = int(seq.sum()) * h_kv * d * 2 * 2
    import flashinfer
    from flashinfer.decode import trtllm_batch_decode_with_kv_cache
    res["flashinfer"] = flashinfer.__version__
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    o_fi = torch.empty((bs, q.shape[1], d), dtype=torch.bfloat16, device=dev)

    def fi():
        trtllm_batch_decode_with_kv_cache(q, (kc, vc), ws, bt, seq, int(seq.max()), bmm1_scale=d ** -0.5,
                                          bmm2_scale=1.0, out=o_fi, kv_layout="HND")
    try:
        fi()
        torch.cuda.synchronize()
        diff = (o_fi.float() - out_ours).abs().max().item()
        res["trtllm_gen_decode"] = dict(windows(fi, secs), max_abs_vs_ours=diff, launch="direct (its wrapper does not capture)")
    except Exception as e:  # noqa: BLE001
        res["trtllm_gen_decode"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    # FlashInfer's own shared-prefix method (cascade inference): level 0 =
    # all 256 queries against the prefix pages as one non-causal batch,
    # level 1 = each request against its suffix pages, then merge_state
    try:
        import time as _t
        t0 = _t.perf_counter()
        casc = flashinfer.MultiLevelCascadeAttentionWrapper(2, torch.zeros(256 << 20, dtype=torch.uint8, device=dev),
                                                            "HND")
        i32 = dict(dtype=torch.int32, device=dev)
        n_suf = (nxt - n_pre) // bs
        casc.plan([torch.tensor([0, bs], **i32), torch.arange(bs + 1, **i32)],
                  [torch.tensor([0, n_pre], **i32), torch.arange(bs + 1, **i32) * n_suf],
                  [torch.arange(n_pre, **i32), torch.arange(n_pre, nxt, **i32)],
                  [torch.tensor([ps], **i32), torch.full((bs,), ps, **i32)],
                  q.shape[1], h_kv, d, ps, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        o_c = {}

        def cf():
            o_c["o"] = casc.run(q, (kc, vc))
        cf()
        torch.cuda.synchronize()
        diff = (o_c["o"].float() - out_ours).abs().max().item()
        res["cascade"] = dict(windows(cf, secs), max_abs_vs_ours=diff, plan_and_jit_s=_t.perf_counter() - t0,
                              launch="direct")
    except Exception as e:  # noqa: BLE001
        res["cascade"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    # the same two-level cascade by hand on FlashInfer's Blackwell prefill
    # backends (the wrapper above picks its default): prefix level and
    # suffix level with LSE, merged by flashinfer.merge_state
    kc_n, vc_n = kc.permute(0, 2, 1, 3).contiguous(), vc.permute(0, 2, 1, 3).contiguous()  # NHD copies
    for be, lay in (("trtllm-gen", "HND"), ("cudnn", "NHD")):
        cache = (kc, vc) if lay == "HND" else (kc_n, vc_n)
        try:
            i32 = dict(dtype=torch.int32, device=dev)
            n_suf = (nxt - n_pre) // bs
            lv = []
            for qo, kvp, idx, lpl in (
                    (torch.tensor([0, bs], **i32), torch.tensor([0, n_pre], **i32), torch.arange(n_pre, **i32),
                     torch.tensor([ps], **i32)),
                    (torch.arange(bs + 1, **i32), torch.arange(bs + 1, **i32) * n_suf,
                     torch.arange(n_pre, nxt, **i32), torch.full((bs,), ps, **i32))):
                w = flashinfer.BatchPrefillWithPagedKVCacheWrapper(
                    torch.zeros(256 << 20, dtype=torch.uint8, device=dev), lay, backend=be)
                kw = {}
                if be == "cudnn":  # element offsets, explicit lengths and block tables
                    nb = qo.numel() - 1
                    qlen = qo[1:] - qo[:-1]
                    kvlen = (kvp[1:] - kvp[:-1]) * ps
                    kw = dict(seq_lens=kvlen, seq_lens_q=qlen, block_tables=idx.view(nb, -1),
                              max_token_per_sequence=int(qlen.max()), max_sequence_kv=int(kvlen.max()))
                    qo = qo * (q.shape[1] * d)
                w.plan(qo, kvp, idx, lpl, q.shape[1], h_kv, d, ps, causal=False, q_data_type=torch.bfloat16,
                       kv_data_type=torch.bfloat16, **kw)
                lv.append(w)
            o_m = {}

            def mc():
                o0, s0 = lv[0].run(q, cache, return_lse=True)
                o1, s1 = lv[1].run(q, cache, return_lse=True)
                o_m["o"] = flashinfer.merge_state(o0, s0, o1, s1)[0]
            mc()
            torch.cuda.synchronize()
            diff = (o_m["o"].float() - out_ours).abs().max().item()
            res["cascade_" + be] = dict(windows(mc, secs), max_abs_vs_ours=diff, launch="direct")
        except Exception as e:  # noqa: BLE001
            import traceback
            res["cascade_" + be] = {"error": f"{type(e).__name__}: {str(e)[:300]}",
                                    "where": traceback.format_exc().strip().splitlines()[-3][:300]}
    res["ours_again"] = windows(ours, secs)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
