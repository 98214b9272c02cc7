"""Decode micro-batches on separate streams (DecodeBatch(concurrent=2), the
cluster sizing for co-resident launches) give bitwise the same selections,
outputs and caches as one batch stepping all sequences."""

import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402


def test_two_concurrent_micro_batches_equal_one_batch():
    cfg = P.SparseAttentionConfig(top_k=16)
    lengths = [9000, 30000, 4097, 20000]
    g = torch.Generator(device="cuda").manual_seed(77)
    kv = [(torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16),
           torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)) for L in lengths]

    def caches():
        out = []
        for k, v in kv:
            c = P.BlockizedLayerCache(2, 128, cfg, capacity=k.shape[0] + 16)
            c.append(k, v)
            out.append(c)
        return out

    steps = 3
    q = torch.randn((steps, 4, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    kn = torch.randn((steps, 4, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    one = P.DecodeBatch(caches(), cfg)
    ref = [one.step(q[s], kn[s], kn[s], return_selection=True) for s in range(steps)]
    c2 = caches()
    halves = [P.DecodeBatch(c2[:2], cfg, concurrent=2), P.DecodeBatch(c2[2:], cfg, concurrent=2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    got = []
    for s in range(steps):
        res = [None, None]
        cur = torch.cuda.current_stream()
        for m in range(2):
            streams[m].wait_stream(cur)
            with torch.cuda.stream(streams[m]):
                res[m] = halves[m].step(q[s, 2 * m:2 * m + 2], kn[s, 2 * m:2 * m + 2], kn[s, 2 * m:2 * m + 2],
                                        return_selection=True)
        for st in streams:
            cur.wait_stream(st)
        got.append((torch.cat([res[0][0], res[1][0]]), torch.cat([res[0][1], res[1][1]])))
    torch.cuda.synchronize()
    for (o1, s1), (o2, s2) in zip(ref, got):
        assert torch.equal(s1, s2)
        assert torch.equal(o1, o2)
    for a, b in zip(one.layers, c2):
        assert a.length == b.length
        assert torch.equal(a.keys.contiguous(), b.keys.contiguous())
        assert torch.equal(a.fine_means.contiguous(), b.fine_means.contiguous())
