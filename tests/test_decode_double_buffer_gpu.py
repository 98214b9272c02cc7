"""The bench's end-to-end decode workflow (bench.py run_decode, e2e part): two
captured copies of a multi-layer decode step with their own input/output
buffers, replayed alternately while the next step's inputs are copied from
pinned host memory on a copy stream and each step's last-layer outputs are
copied back.  Every step's host-side outputs must equal eager stepping of the
same inputs bitwise, and host and device lengths must agree at the end."""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

HQ, HKV, D = 32, 2, 128
LAYERS, S, STEPS = 3, 4, 6
LENGTHS = [9000, 4097, 20000, 700]


def _build(cfg, seed, extra):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    layers = []
    for _ in range(LAYERS):
        caches = []
        for L in LENGTHS:
            c = P.BlockizedLayerCache(HKV, D, cfg, capacity=L + extra)
            c.append(torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16),
                     torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16))
            caches.append(c)
        layers.append(caches)
    return layers


def test_double_buffered_graph_steps_equal_eager():
    cfg = P.SparseAttentionConfig(top_k=16)
    extra = STEPS + 8
    bound = max(LENGTHS) + extra
    gen = torch.Generator(device="cuda").manual_seed(99)
    xs = [(torch.randn((LAYERS, S, HQ, D), generator=gen, device="cuda").to(torch.bfloat16),
           torch.randn((LAYERS, S, HKV, D), generator=gen, device="cuda").to(torch.bfloat16),
           torch.randn((LAYERS, S, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)) for _ in range(STEPS)]

    # reference: eager steps
    ref_layers = _build(cfg, 5, extra)
    ref_batches = [P.DecodeBatch(c, cfg) for c in ref_layers]
    want = []
    for q, k, v in xs:
        o = None
        for i, b in enumerate(ref_batches):
            o = b.step(q[i], k[i], v[i], max_len=bound)
        want.append(o.cpu())

    layers = _build(cfg, 5, extra)
    batches = [P.DecodeBatch(c, cfg) for c in layers]
    for b in batches:
        b.reserve(extra)
    bufs = [tuple(torch.empty_like(t) for t in xs[0]) for _ in range(2)]
    outs = [None, None]
    graphs = [torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for g in range(2):
            q, k, v = bufs[g]
            with torch.cuda.graph(graphs[g], stream=side):
                o = None
                for i, b in enumerate(batches):
                    o = b.step(q[i], k[i], v[i], max_len=bound, bookkeep=False)
            outs[g] = o
    torch.cuda.synchronize()
    host_in = [tuple(t.cpu().pin_memory() for t in x) for x in xs]
    host_out = [torch.empty((S, HQ, D), dtype=torch.bfloat16).pin_memory() for _ in range(STEPS)]
    copy = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]

    def h2d(step, g):
        with torch.cuda.stream(copy):
            for dst, src in zip(bufs[g], host_in[step]):
                dst.copy_(src, non_blocking=True)
            h2d_done[g].record(copy)

    copy.wait_stream(cur)
    h2d(0, 0)
    for i in range(STEPS):
        g = i & 1
        cur.wait_event(h2d_done[g])
        if i >= 2:
            cur.wait_event(d2h_done[g])
        graphs[g].replay()
        comp_done[g].record(cur)
        for b in batches:
            b.advance(1)
        if i + 1 < STEPS:
            if i >= 1:
                copy.wait_event(comp_done[1 - g])
            h2d(i + 1, 1 - g)
        with torch.cuda.stream(copy):
            copy.wait_event(comp_done[g])
            host_out[i].copy_(outs[g], non_blocking=True)
            d2h_done[g].record(copy)
    cur.wait_stream(copy)
    torch.cuda.synchronize()
    for i in range(STEPS):
        assert torch.equal(host_out[i], want[i]), i
    lib = _lib.load()
    for b in batches:
        buf = (ctypes.c_int64 * S)()
        _lib.check(lib.infllm2_decode_table_lengths(b._table.data_ptr(), S, buf, cur.cuda_stream), "lengths")
        assert list(buf) == [c.length for c in b.layers] == [L + STEPS for L in LENGTHS]
