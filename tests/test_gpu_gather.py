"""Fused multi-GPU output gather (parallel.PeerGather +
codec_decode_attention_gather) on ONE GPU: two ranks
are two processes sharing cuda:0 -- gloo for the handle exchange, CUDA IPC
for the peer buffers, the merge kernels' peer stores and the arrival
counters exactly as across NVLink. Every rank's gathered global output
must equal the unsharded step (same plan family) and the float64 path
reference within the bf16 bar, for the kv-head split and the tree
partition, over several steps (counters advance) and a CUDA-graph replay.
"""
import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, partition, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist

        import paper_2505_17694_b200 as P
        from paper_2505_17694_b200 import parallel as PL
        from paper_2505_17694_b200 import workloads as W
        from paper_2505_17694_b200.executor import FLAG_MERGE_ALL, DecodeStep

        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        h_q, h_kv, d = 32, 8, 128
        g = h_q // h_kv
        if partition == "heads":
            spec = W.two_level(2048, 96, 24, h_q=h_q, h_kv=h_kv, d=d, tensors=False)
            parent, length, paths = spec.parent[1:], spec.length[1:], spec.paths
        else:  # a small forest of independent trees of different sizes
            parent, length, paths = [], [], []
            for root_len, n_req in ((300, 3), (900, 7), (2000, 1), (128, 12), (1500, 5)):
                parent.append(0)
                length.append(root_len)
                root = len(parent)
                for i in range(n_req):
                    parent.append(root)
                    length.append(40 + 13 * i)
                    paths.append((root, len(parent)))
        full = P.forest_from_pool(parent, length, paths, h_kv, d)
        gen = torch.Generator(device=dev)
        gen.manual_seed(7)
        T = full.total_tokens
        kp = (torch.randn((h_kv, T, d), generator=gen, device=dev) / math.sqrt(d)).to(torch.bfloat16)
        vp = (torch.randn((h_kv, T, d), generator=gen, device=dev) / math.sqrt(d)).to(torch.bfloat16)
        qf = (torch.randn((full.bs, h_q, d), generator=gen, device=dev) / math.sqrt(d)).to(torch.bfloat16)
        table = P.load_default_profile()
        # the unsharded step (what the gathered output must reproduce)
        plan_full = P.plan_device(full, g, table, h_kv)
        ref = DecodeStep(full, plan_full, h_q, "bfloat16", device=dev)(qf, kp, vp)
        peers = PL.PeerGather(full.bs, h_q, d, dev, buffers=2)
        if partition == "heads":
            h0, h1 = PL.head_shard(h_kv, world, rank)
            forest, ql = full, qf[:, h0 * g:h1 * g].contiguous()
            kl, vl = kp[h0:h1].contiguous(), vp[h0:h1].contiguous()
            plan = P.plan_device(forest, g, table, h1 - h0)
            step = DecodeStep(forest, plan, h_q, "bfloat16", head_begin=h0, head_end=h1, device=dev,
                              flags=FLAG_MERGE_ALL)
            row_map, head0 = None, None
        else:
            part = PL.tree_partition(full, table, world, head_multiplicity=g)
            shard = PL.shard_trees(full, part, rank)
            forest = shard.forest(h_kv, d)
            kl, vl = shard.slice_pool(full, forest, kp, vp)
            ql = qf[list(shard.requests)].contiguous()
            plan = P.plan_device(forest, g, table, h_kv)
            step = DecodeStep(forest, plan, h_q, "bfloat16", device=dev, flags=FLAG_MERGE_ALL)
            row_map = torch.tensor(list(shard.requests), dtype=torch.int32, device=dev)
            head0 = 0
        errs = []
        for it in range(3):  # the arrival counters advance every step
            b = it % 2
            peers.output(b).zero_()
            torch.cuda.synchronize()
            dist.barrier()
            step.gather(ql, kl, vl, peers, head0=head0, row_map=row_map, buf=b)
            peers.wait()
            torch.cuda.synchronize()
            errs.append(float((peers.output(b) - ref).abs().max()))
        # graph replay of gather + wait
        peers.output(0).zero_()
        torch.cuda.synchronize()
        dist.barrier()
        replay = step.capture_gather(ql, kl, vl, peers, head0=head0, row_map=row_map, buf=0)
        dist.barrier()
        replay()
        torch.cuda.synchronize()
        errs.append(float((peers.output(0) - ref).abs().max()))
        # float64 reference of sampled requests over their paths
        got = peers.output(0)
        worst = 0.0
        for r in sorted({0, full.bs // 2, full.bs - 1}):
            toks = torch.cat([torch.arange(full.token_offset[n], full.token_offset[n] + full.visible_count(n, r),
                                           device=dev) for n in full.paths[r]])
            kk, vv = kp[:, toks].double(), vp[:, toks].double()
            qq = qf[r].double().view(h_kv, g, d)
            p = torch.softmax(torch.einsum("hgd,hld->hgl", qq, kk) / math.sqrt(d), dim=-1)
            o = torch.einsum("hgl,hld->hgd", p, vv).reshape(h_q, d)
            worst = max(worst, float((got[r].double() - o).abs().max()))
        dist.barrier()
        peers.close()
        q.put((rank, errs, worst, None))
        dist.destroy_process_group()
    except Exception as e:  # report, do not hang the parent
        import traceback
        q.put((rank, None, None, traceback.format_exc()))


@pytest.mark.parametrize("partition,world", [("heads", 2), ("trees", 2), ("heads", 4)])
def test_fused_gather_ranks_one_gpu(partition, world):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, partition, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, errs, worst, tb in res:
        assert tb is None, f"rank {rank}:\n{tb}"
        # the same plan family per shard: equal to the unsharded step up to
        # the split points of the shared nodes (fp32 merge order)
        assert max(errs) <= 2e-5, (rank, errs)
        assert worst <= 2e-3, (rank, worst)


def test_bench_two_ranks_one_gpu():
    """bench.py's multi-rank path end to end (torchrun, 2 ranks, fused
    gather) on one GPU: CODEC_BENCH_ONE_GPU=1 puts both ranks on cuda:0 with
    gloo for the control plane. Timing is meaningless here (two contexts
    time-slice the GPU); the line must verify and the gathered output must
    hold every rank's rows."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, CODEC_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(root / "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--config", "cfg1", "--no-cpu-baseline"]
    res = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and "fused peer-store" in line["config"]["parallelism"]
    v = line["verified"]
    assert v["ok"] and v["gather_ok"] and v["all_ranks_ok"], v


def test_bind_device():
    """codec_bind_device: binding this process's GPU succeeds (and is
    cached per thread); a device index the box does not have raises the
    library's CUDA error instead of silently launching elsewhere."""
    import torch

    from paper_2505_17694_b200 import _lib

    _lib.bind_device(torch.device("cuda", 0))
    assert _lib.lib().codec_bind_device(0) == 0
    n = torch.cuda.device_count()
    with pytest.raises(Exception) as ei:
        _lib.check(_lib.lib().codec_bind_device(n))
    assert "cudaSetDevice" in str(ei.value)
    _lib.check(_lib.lib().codec_bind_device(0))  # back on cuda:0 for the tests after this one
