"""World-size-2 CPU (gloo) tests of the query-sharded prefill plumbing.

The GPU box has one device, so the N>1 path's host logic is exercised here:
zig-zag ownership balances stage-1 work, every row is owned exactly once, and
the all-gather + reorder rebuilds the full K/V in natural row order on every
rank (the precondition for bitwise-identical kernel means and selections).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_07900_b200 import sharding as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _FakeCache:
    """Host stand-in for BlockizedLayerCache's append/truncate surface."""

    def __init__(self):
        self.rows = []

    def truncate(self, n):
        assert n == 0
        self.rows = []

    def append(self, k, v):
        self.rows.append((k.clone(), v.clone()))


def _worker(rank, world, port, seq, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        full_k = torch.randn((seq, 2, 8), generator=g)
        full_v = torch.randn((seq, 2, 8), generator=g)
        chunks = S.zigzag_chunks(seq, world, rank)
        k_local = [full_k[lo:hi] for lo, hi in chunks]
        v_local = [full_v[lo:hi] for lo, hi in chunks]
        cache = _FakeCache()
        S.fill_layer_cache(cache, k_local, v_local, world)
        k = torch.cat([kk for kk, _ in cache.rows])
        v = torch.cat([vv for _, vv in cache.rows])
        ok = torch.equal(k, full_k) and torch.equal(v, full_v) and len(cache.rows) == world + 1
        q_local = [torch.arange(lo, hi) for lo, hi in chunks]
        outs = S.sharded_prefill(q_local, cache, None, chunks, lambda q, c, cfg, lo: q - lo)
        ok = ok and all(torch.equal(o, torch.arange(0, hi - lo)) for o, (lo, hi) in zip(outs, chunks))
        out_q.put((rank, ok, chunks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_rebuilds_natural_order(world):
    seq = 64 * 2 * world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seq, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    owned = sorted(r for _, _, ch in res for lo, hi in ch for r in range(lo, hi))
    assert owned == list(range(seq))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_zigzag_balances_stage1_work(world):
    seq = 131072
    work = []
    for r in range(world):
        w = 0
        for lo, hi in S.zigzag_chunks(seq, world, r):
            t = np.arange(lo, hi)
            w += int(np.minimum(t // 16 + 1, seq // 16).sum())
        work.append(w)
    assert max(work) / min(work) < 1.001
