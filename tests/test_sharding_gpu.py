"""The query-sharded prefill executed for real: 2 ranks, each a
separate process on cuda:0 (the box has one GPU; gloo carries the all-gather
through host memory, NCCL would do it over NVLink), run the bench's own path -
every rank holds only its zig-zag token shard of K/V and its query rows,
``sharding.LayerGather`` rebuilds the full cache (fused append + compress from
the gather buffers), ``two_stage_attention`` runs on the rank's chunks.  Each
rank's rows must be BITWISE equal to a 1-rank run of the whole layer
(selection, output, LSE): rows are independent given the cache
and every rank's cache must be bitwise the full cache (same kernel means)."""

import os
import socket
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, HQ, HKV, D = 16384, 32, 2, 128


def _inputs():
    g = torch.Generator(device="cuda").manual_seed(4242)
    q = torch.randn((L, HQ, D), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((L, HKV, D), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((L, HKV, D), generator=g, device="cuda").to(torch.bfloat16)
    return q, k, v


def _rank(rank, world, port, outdir):
    import torch.distributed as dist

    import paper_2506_07900_b200 as P
    from paper_2506_07900_b200 import sharding as S

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v = _inputs()
        chunks = S.zigzag_chunks(L, world, rank)
        k_loc = [k[lo:hi].clone() for lo, hi in chunks]
        v_loc = [v[lo:hi].clone() for lo, hi in chunks]
        cfg = P.SparseAttentionConfig(top_k=16)
        cache = P.BlockizedLayerCache(HKV, D, cfg, capacity=L)
        side = torch.cuda.Stream()
        S.LayerGather(k_loc, v_loc, world, stream=side).fill(cache)
        res = {"chunks": chunks, "fine": cache.fine_means.contiguous().cpu(),
               "coarse": cache.coarse_means.contiguous().cpu()}
        for i, (lo, hi) in enumerate(chunks):
            o, s, l = P.two_stage_attention(q[lo:hi], cache, cfg, lo, return_selection=True, return_lse=True)
            res[f"out{i}"], res[f"sel{i}"], res[f"lse{i}"] = o.cpu(), s.cpu(), l.cpu()
        torch.save(res, os.path.join(outdir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_bitwise_equal_one_rank():
    import paper_2506_07900_b200 as P

    world = 2
    with tempfile.TemporaryDirectory() as outdir:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_rank, args=(r, world, port, outdir)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
            assert p.exitcode == 0, p.exitcode
        ranks = [torch.load(os.path.join(outdir, f"rank{r}.pt")) for r in range(world)]
    torch.cuda.set_device(0)
    q, k, v = _inputs()
    cfg = P.SparseAttentionConfig(top_k=16)
    cache = P.BlockizedLayerCache(HKV, D, cfg, capacity=L)
    cache.append(k, v)
    out, sel, lse = P.two_stage_attention(q, cache, cfg, 0, return_selection=True, return_lse=True)
    fine, coarse = cache.fine_means.contiguous().cpu(), cache.coarse_means.contiguous().cpu()
    owned = []
    for res in ranks:
        assert torch.equal(res["fine"], fine) and torch.equal(res["coarse"], coarse)
        for i, (lo, hi) in enumerate(res["chunks"]):
            owned += list(range(lo, hi))
            assert torch.equal(res[f"sel{i}"], sel[lo:hi].cpu())
            assert torch.equal(res[f"out{i}"], out[lo:hi].cpu())
            assert torch.equal(res[f"lse{i}"], lse[lo:hi].cpu())
    assert sorted(owned) == list(range(L))
