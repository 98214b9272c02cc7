"""Batched decode (DecodeBatch / infllm2_decode_step) vs the single-sequence
path and the CPU oracle.

Each decode step appends one token per sequence and attends one query row
(the reference's decode: forward with n = 1, model.py:434-444).  Checks:
selections identical to two_stage_attention on an independently built cache
of the same content, outputs/LSE within float32 noise, kernel means bitwise
equal to a rebuild after every step (including single-row appends that cross a
coarse-stride multiple from old % 128 >= 32, the reference's F18 crash), and
selections identical to the oracle on the last step.
"""

import numpy as np
import pytest
import torch

from inputs import digest, make_qkv
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402


def _means(t):
    return t.contiguous().cpu().numpy()


@pytest.mark.parametrize("lengths,topk", [([3000, 5000, 777, 8190], 16), ([127, 1000, 4093], 8),
                                          ([64, 2111], 64)])
def test_decode_batch_matches_single_sequence_path(lengths, topk):
    cfg = P.SparseAttentionConfig(top_k=topk)
    steps = 4
    full = [make_qkv(31 + i, L + steps, steps, 32, 2, 128) for i, L in enumerate(lengths)]
    layers = []
    for (q, k, v), L in zip(full, lengths):
        layer = P.BlockizedLayerCache(2, 128, cfg)
        layer.append(torch.from_numpy(k[:L]).cuda(), torch.from_numpy(v[:L]).cuda())
        layers.append(layer)
    batch = P.DecodeBatch(layers, cfg)
    for st in range(steps):
        qs = torch.stack([torch.from_numpy(f[0][st]) for f in full]).cuda()
        ks = torch.stack([torch.from_numpy(f[1][L + st]) for f, L in zip(full, lengths)]).cuda()
        vs = torch.stack([torch.from_numpy(f[2][L + st]) for f, L in zip(full, lengths)]).cuda()
        out, sel, lse = batch.step(qs, ks, vs, return_selection=True, return_lse=True, out_dtype=torch.float32)
        for i, ((q, k, v), L) in enumerate(zip(full, lengths)):
            n_now = L + st + 1
            assert layers[i].length == n_now
            ref = P.BlockizedLayerCache(2, 128, cfg)
            ref.append(torch.from_numpy(k[:n_now]).cuda(), torch.from_numpy(v[:n_now]).cuda())
            assert digest(_means(layers[i].fine_means)) == digest(_means(ref.fine_means))
            assert digest(_means(layers[i].coarse_means)) == digest(_means(ref.coarse_means))
            o2, s2, l2 = P.two_stage_attention(qs[i:i + 1], ref, cfg, n_now - 1, return_selection=True,
                                               return_lse=True, out_dtype=torch.float32, split_p=True)
            assert torch.equal(sel[i], s2[0]), (i, st, sel[i].tolist(), s2[0].tolist())
            assert (out[i] - o2[0]).abs().max().item() < 1e-4
            assert (lse[i] - l2[0]).abs().max().item() < 1e-4
    # last step vs the oracle (float64 dots)
    geom = O.Geometry(top_k=topk)
    for i, ((q, k, v), L) in enumerate(zip(full, lengths)):
        n_now = L + steps
        fine = O.window_means(k[:n_now], 32, 16)
        ref = O.two_stage_attention(q[steps - 1:steps], k[:n_now], v[:n_now], fine, geom, n_now - 1)
        assert np.array_equal(sel[i].cpu().numpy(), ref.selection[0]), i
        assert np.abs(out[i].cpu().numpy() - ref.out[0]).max() < 1e-4


def test_decode_table_rebuilds_after_external_append_and_growth():
    cfg = P.SparseAttentionConfig(top_k=8)
    q, k, v = make_qkv(5, 400, 4, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg)        # small capacity: grows during the test
    layer.append(torch.from_numpy(k[:60]).cuda(), torch.from_numpy(v[:60]).cuda())
    batch = P.DecodeBatch([layer], cfg)
    n = 60
    for t in range(6):
        if t == 3:   # external prefill append between decode steps
            layer.append(torch.from_numpy(k[n:n + 100]).cuda(), torch.from_numpy(v[n:n + 100]).cuda())
            n += 100
        batch.step(torch.from_numpy(q[t % 4:t % 4 + 1]).cuda(), torch.from_numpy(k[n:n + 1]).cuda(),
                   torch.from_numpy(v[n:n + 1]).cuda())
        n += 1
        assert layer.length == n
    ref = P.BlockizedLayerCache(2, 128, cfg)
    ref.append(torch.from_numpy(k[:n]).cuda(), torch.from_numpy(v[:n]).cuda())
    assert digest(_means(layer.fine_means)) == digest(_means(ref.fine_means))
    assert torch.equal(layer.keys.contiguous(), ref.keys.contiguous())


@pytest.mark.parametrize("lengths", [[3000, 5000, 777, 8190, 64, 1, 130, 20000], [16383, 16385]])
def test_fused_decode_matches_five_launch_path(lengths, monkeypatch):
    """The single-launch decode (decode_fused.cu) against the five-launch path
    (decode.cu) over several steps: identical selections and kernel means,
    outputs within float32 noise."""
    cfg = P.SparseAttentionConfig(top_k=16)
    steps = 5
    full = [make_qkv(71 + i, L + steps, steps, 32, 2, 128) for i, L in enumerate(lengths)]

    def run(legacy):
        if legacy:
            monkeypatch.setenv("INFLLM2_DECODE_LEGACY", "1")
        else:
            monkeypatch.delenv("INFLLM2_DECODE_LEGACY", raising=False)
        layers = []
        for (q, k, v), L in zip(full, lengths):
            layer = P.BlockizedLayerCache(2, 128, cfg)
            layer.append(torch.from_numpy(k[:L]).cuda(), torch.from_numpy(v[:L]).cuda())
            layers.append(layer)
        batch = P.DecodeBatch(layers, cfg)
        res = []
        for st in range(steps):
            qs = torch.stack([torch.from_numpy(f[0][st]) for f in full]).cuda()
            ks = torch.stack([torch.from_numpy(f[1][L + st]) for f, L in zip(full, lengths)]).cuda()
            vs = torch.stack([torch.from_numpy(f[2][L + st]) for f, L in zip(full, lengths)]).cuda()
            res.append(batch.step(qs, ks, vs, return_selection=True, return_lse=True, out_dtype=torch.float32))
        torch.cuda.synchronize()
        return res, layers

    got, lay_f = run(False)
    ref, lay_l = run(True)
    for (o1, s1, l1), (o2, s2, l2) in zip(got, ref):
        assert torch.equal(s1, s2)
        assert (o1 - o2).abs().max().item() < 1e-4
        assert (l1 - l2).abs().max().item() < 1e-4
    for a, b in zip(lay_f, lay_l):
        assert a.length == b.length
        assert torch.equal(a.keys.contiguous(), b.keys.contiguous())
        assert torch.equal(a.values.contiguous(), b.values.contiguous())
        assert digest(_means(a.fine_means)) == digest(_means(b.fine_means))
        assert digest(_means(a.coarse_means)) == digest(_means(b.coarse_means))


def test_decode_batch_small_model_shape():
    """MiniCPM4-0.5B geometry (G = 8, D = 64): the batched five-launch decode
    path equals the prefill path on an independently built cache (selections
    identical; outputs within float32 noise of the split-P prefill)."""
    cfg = P.SparseAttentionConfig(top_k=16)
    lengths = [1500, 3001]
    full = [make_qkv(91 + i, L + 3, 3, 16, 2, 64) for i, L in enumerate(lengths)]
    layers = []
    for (q, k, v), L in zip(full, lengths):
        layer = P.BlockizedLayerCache(2, 64, cfg)
        layer.append(torch.from_numpy(k[:L]).cuda(), torch.from_numpy(v[:L]).cuda())
        layers.append(layer)
    batch = P.DecodeBatch(layers, cfg)
    for st in range(3):
        qs = torch.stack([torch.from_numpy(f[0][st]) for f in full]).cuda()
        ks = torch.stack([torch.from_numpy(f[1][L + st]) for f, L in zip(full, lengths)]).cuda()
        vs = torch.stack([torch.from_numpy(f[2][L + st]) for f, L in zip(full, lengths)]).cuda()
        out, sel = batch.step(qs, ks, vs, return_selection=True, out_dtype=torch.float32)
        for i, ((q, k, v), L) in enumerate(zip(full, lengths)):
            n_now = L + st + 1
            ref = P.BlockizedLayerCache(2, 64, cfg)
            ref.append(torch.from_numpy(k[:n_now]).cuda(), torch.from_numpy(v[:n_now]).cuda())
            o2, s2 = P.two_stage_attention(qs[i:i + 1], ref, cfg, n_now - 1, return_selection=True,
                                           out_dtype=torch.float32, split_p=True)
            assert torch.equal(sel[i], s2[0])
            assert (out[i] - o2[0]).abs().max().item() < 1e-4
