"""Batched decode partitioned over sequences (SURVEY §8e, configs[3]) executed
under 2 ranks: each rank is a separate process on cuda:0 (one GPU here; on a
box every rank has its own B200), holds only its partition of the sequences'
caches and runs the bench's workflow on it - an eager decode step, a captured
graph of the step replayed with ``advance`` - with a barrier per step and no
collective on the data path.  Every rank's outputs, selections and device
lengths must be bitwise those of the same partition stepped in one process."""

import os
import socket
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SEQS, L0, STEPS = 4, [9000, 20000, 4097, 13000], 4


def _partition(world, rank):
    return [s for s in range(SEQS) if s % world == rank]


def _inputs(seq):
    g = torch.Generator(device="cuda").manual_seed(900 + seq)
    n = L0[seq]
    k = torch.randn((n, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((n, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn((STEPS + 1, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    kn = torch.randn((STEPS + 1, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    return k, v, q, kn


def _run_partition(seqs, barrier=lambda: None):
    import paper_2506_07900_b200 as P

    cfg = P.SparseAttentionConfig(top_k=16)
    caches, qs, kns = [], [], []
    for s in seqs:
        k, v, q, kn = _inputs(s)
        c = P.BlockizedLayerCache(2, 128, cfg, capacity=k.shape[0] + STEPS + 8)
        c.append(k, v)
        caches.append(c)
        qs.append(q)
        kns.append(kn)
    q = torch.stack(qs, 1)            # (STEPS + 1, S, 32, 128)
    kn = torch.stack(kns, 1)
    batch = P.DecodeBatch(caches, cfg)
    batch.reserve(STEPS + 8)
    bound = max(L0) + STEPS + 8
    res = {}
    o, s = batch.step(q[0], kn[0], kn[0], max_len=bound, return_selection=True)
    res["out0"], res["sel0"] = o.cpu(), s.cpu()
    qb, kb = q[1].clone(), kn[1].clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            go, gs = batch.step(qb, kb, kb, max_len=bound, return_selection=True, bookkeep=False)
    torch.cuda.current_stream().wait_stream(side)
    for t in range(1, STEPS + 1):
        qb.copy_(q[t])
        kb.copy_(kn[t])
        graph.replay()
        torch.cuda.synchronize()
        batch.advance(1)
        barrier()
        res[f"out{t}"], res[f"sel{t}"] = go.cpu(), gs.cpu()
    import ctypes

    from paper_2506_07900_b200 import _lib
    lib = _lib.load()
    lens = (ctypes.c_int64 * len(seqs))()
    _lib.check(lib.infllm2_decode_table_lengths(batch._table.data_ptr(), len(seqs), lens,
                                                torch.cuda.current_stream().cuda_stream), "lengths")
    res["dev_len"] = list(lens)
    res["host_len"] = [c.length for c in caches]
    return res


def _rank(rank, world, port, outdir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run_partition(_partition(world, rank), barrier=dist.barrier)
        torch.save(res, os.path.join(outdir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_decode_bitwise_equal_single_process():
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
        for r in range(world):
            got = torch.load(os.path.join(outdir, f"rank{r}.pt"))
            want = _run_partition(_partition(world, r))
            assert got["dev_len"] == got["host_len"] == want["host_len"]
            for t in range(STEPS + 1):
                assert torch.equal(got[f"sel{t}"], want[f"sel{t}"]), (r, t)
                assert torch.equal(got[f"out{t}"], want[f"out{t}"]), (r, t)
