"""Early means stream of the fused decode step (DESIGN §4 K4): when the stream's
previous decode step used ANOTHER layer's table, the kernel reads its lengths
and issues its first means tiles before griddepcontrol.wait.  Two layers
stepped alternately on one stream (early path, as a model's layers are) must
give bitwise the same selections, outputs, lengths and caches as the same
layers each stepped on its own stream (never early), eagerly and through a
captured graph."""

import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402


def _layers(cfg, kv):
    out = []
    for layer in kv:
        caches = []
        for k, v in layer:
            c = P.BlockizedLayerCache(2, 128, cfg, capacity=k.shape[0] + 64)
            c.append(k, v)
            caches.append(c)
        out.append(P.DecodeBatch(caches, cfg))
    return out


def test_alternating_layers_early_equals_isolated():
    cfg = P.SparseAttentionConfig(top_k=16)
    lengths = [9000, 30000, 4097, 64 * 300 - 1]
    g = torch.Generator(device="cuda").manual_seed(5)
    kv = [[(torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16),
            torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)) for L in lengths]
          for _ in range(2)]
    steps = 6
    q = torch.randn((steps, 2, 4, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    kn = torch.randn((steps, 2, 4, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    lib = _lib.load()

    # reference: each layer on its own stream -> the tracker never sees another table
    ref_layers = _layers(cfg, kv)
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    ref = []
    for s in range(steps):
        row = []
        for li in range(2):
            sts[li].wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(sts[li]):
                row.append(ref_layers[li].step(q[s, li], kn[s, li], kn[s, li], return_selection=True,
                                               return_lse=True))
            torch.cuda.current_stream().wait_stream(sts[li])
        ref.append(row)
    torch.cuda.synchronize()

    # early: both layers alternately on one stream
    lay = _layers(cfg, kv)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    n0 = lib.infllm2_decode_early_count()
    got = []
    with torch.cuda.stream(side):
        for s in range(steps):
            got.append([lay[li].step(q[s, li], kn[s, li], kn[s, li], return_selection=True, return_lse=True)
                        for li in range(2)])
    torch.cuda.synchronize()
    assert lib.infllm2_decode_early_count() - n0 >= 2 * steps - 1, "the early path did not run"
    for rr, gg in zip(ref, got):
        for (o1, s1, l1), (o2, s2, l2) in zip(rr, gg):
            assert torch.equal(s1, s2)
            assert torch.equal(o1, o2)
            assert torch.equal(l1, l2)
    for a, b in zip(ref_layers, lay):
        for ca, cb in zip(a.layers, b.layers):
            assert ca.length == cb.length
            assert torch.equal(ca.keys.contiguous(), cb.keys.contiguous())
            assert torch.equal(ca.values.contiguous(), cb.values.contiguous())
            assert torch.equal(ca.fine_means.contiguous(), cb.fine_means.contiguous())


def test_alternating_layers_graph_replay_early():
    """The bench's workflow: both layers captured in one graph, replayed with
    advance(); lengths on the device track the host and results equal eager
    isolated stepping."""
    cfg = P.SparseAttentionConfig(top_k=16)
    lengths = [20000, 5000]
    g = torch.Generator(device="cuda").manual_seed(9)
    kv = [[(torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16),
            torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)) for L in lengths]
          for _ in range(2)]
    q = torch.randn((2, 2, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    kn = torch.randn((2, 2, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    reps = 4
    bound = max(lengths) + reps + 8

    ref_layers = _layers(cfg, kv)
    for b in ref_layers:
        b.reserve(reps + 8)
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    ref = []
    for s in range(1 + reps):
        row = []
        for li in range(2):
            sts[li].wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(sts[li]):
                row.append(ref_layers[li].step(q[li], kn[li], kn[li], max_len=bound, return_selection=True))
            torch.cuda.current_stream().wait_stream(sts[li])
        ref.append(row)
    torch.cuda.synchronize()

    lay = _layers(cfg, kv)
    for b in lay:
        b.reserve(reps + 8)
    outs = [None, None]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        first = [lay[li].step(q[li], kn[li], kn[li], max_len=bound, return_selection=True) for li in range(2)]
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=side):
            for li in range(2):
                outs[li] = lay[li].step(q[li], kn[li], kn[li], max_len=bound, return_selection=True, bookkeep=False)
    for li in range(2):
        assert torch.equal(first[li][1], ref[0][li][1])
        assert torch.equal(first[li][0], ref[0][li][0])
    for r in range(reps):
        graph.replay()
        torch.cuda.synchronize()
        for b in lay:
            b.advance(1)
        for li in range(2):
            assert torch.equal(outs[li][1], ref[1 + r][li][1])
            assert torch.equal(outs[li][0], ref[1 + r][li][0])
    lib = _lib.load()
    import ctypes
    for a, b in zip(ref_layers, lay):
        n = len(b.layers)
        lens = (ctypes.c_int64 * n)()
        _lib.check(lib.infllm2_decode_table_lengths(b._table.data_ptr(), n, lens,
                                                    torch.cuda.current_stream().cuda_stream), "lengths")
        assert list(lens) == [c.length for c in b.layers]
        for ca, cb in zip(a.layers, b.layers):
            assert ca.length == cb.length
            assert torch.equal(ca.fine_means.contiguous(), cb.fine_means.contiguous())
