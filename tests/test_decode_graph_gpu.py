"""configs[3] decode at full size, through the workflow bench.py times.

8 sequences x 128K cached tokens in one DecodeBatch (the per-GPU share of
BASELINE configs[3]), stepped the way the bench does: one eager step, a CUDA
graph captured with ``bookkeep=False``, replays followed by ``advance()``, then
eager steps again.  After every phase the host lengths must equal the
device-resident lengths the kernels bump (infllm2_decode_table_lengths).
Every step's selection must equal the float64 CUDA-core verifier's on the same
cache (``exact=True``, single-row path), and the last step's selection for two
sampled (sequence, group) pairs must equal the CPU oracle (the reference's
algorithm, float64 dots; reference decode = append then attend n = 1,
/root/reference/pkg/src/deskinfer/model.py:434-444).

Also: forced_consume_budget with top_k <= the forced count (budget 0 while free
blocks remain) selects the forced blocks only, as select_topk does
(sparse.py:265-277).
"""

import ctypes

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: F401

from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

HQ, HKV, D = 32, 2, 128


def _device_lengths(batch):
    lib = _lib.load()
    n = len(batch.layers)
    buf = (ctypes.c_int64 * n)()
    _lib.check(lib.infllm2_decode_table_lengths(batch._table.data_ptr(), n, buf,
                                                torch.cuda.current_stream().cuda_stream), "lengths")
    return list(buf)


def _assert_lengths(batch, phase):
    host = [l.length for l in batch.layers]
    dev = _device_lengths(batch)
    assert host == dev, (phase, host, dev)


def _verify_step(batch, cfg, q, sel, out, lse):
    """Selections of one step vs the float64 verifier on the same caches."""
    for i, layer in enumerate(batch.layers):
        o2, s2, l2 = P.two_stage_attention(q[i:i + 1], layer, cfg, layer.length - 1, exact=True,
                                           return_selection=True, return_lse=True, out_dtype=torch.float32)
        assert torch.equal(sel[i], s2[0]), (i, sel[i].tolist(), s2[0].tolist())
        assert (out[i].float() - o2[0]).abs().max().item() < 2 * OUT_ABS
        assert (lse[i] - l2[0]).abs().max().item() < LSE_TC


def test_decode_128k_graph_replay_workflow():
    torch.cuda.set_device(0)
    S, L, top_k = 8, 131072, 16
    cfg = P.SparseAttentionConfig(top_k=top_k)
    phases = dict(eager=1, replay=5, eager2=5)
    extra = sum(phases.values()) + 2
    gen = torch.Generator(device="cuda").manual_seed(2506)
    layers = []
    for s in range(S):
        c = P.BlockizedLayerCache(HKV, D, cfg, capacity=L + extra, device="cuda:0")
        k = torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
        v = torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
        c.append(k, v)
        layers.append(c)
    batch = P.DecodeBatch(layers, cfg)
    batch.reserve(extra)
    bound = L + extra
    nsteps = sum(phases.values())
    qs = torch.randn((nsteps, S, HQ, D), generator=gen, device="cuda").to(torch.bfloat16)
    ks = torch.randn((nsteps, S, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    vs = torch.randn((nsteps, S, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    steps_done = 0

    # phase 1: eager
    out, sel, lse = batch.step(qs[0], ks[0], vs[0], max_len=bound, return_selection=True, return_lse=True)
    steps_done += 1
    _assert_lengths(batch, "eager")
    _verify_step(batch, cfg, qs[0], sel, out, lse)

    # phase 2: capture (executes nothing) + replays with fresh inputs copied in
    q_buf, k_buf, v_buf = qs[1].clone(), ks[1].clone(), vs[1].clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            g_out, g_sel, g_lse = batch.step(q_buf, k_buf, v_buf, max_len=bound, bookkeep=False,
                                             return_selection=True, return_lse=True)
    torch.cuda.synchronize()
    _assert_lengths(batch, "after capture")        # the capture must not advance anything
    for r in range(phases["replay"]):
        i = steps_done
        q_buf.copy_(qs[i])
        k_buf.copy_(ks[i])
        v_buf.copy_(vs[i])
        graph.replay()
        batch.advance(1)
        torch.cuda.synchronize()
        steps_done += 1
        _assert_lengths(batch, f"replay {r}")
        _verify_step(batch, cfg, qs[i], g_sel, g_out, g_lse)

    # phase 3: eager again (host bookkeeping continues from the replays)
    for r in range(phases["eager2"]):
        i = steps_done
        out, sel, lse = batch.step(qs[i], ks[i], vs[i], max_len=bound, return_selection=True, return_lse=True)
        steps_done += 1
        _assert_lengths(batch, f"eager2 {r}")
        _verify_step(batch, cfg, qs[i], sel, out, lse)
    assert all(l.length == L + nsteps for l in layers)

    # the appended rows are the inputs, and the means equal a rebuild
    for s in (0, S - 1):
        keys = layers[s].keys
        assert torch.equal(keys[L:].contiguous(), ks[:, s].contiguous())
        fine, coarse = layers[s].rebuild_kernels()
        assert torch.equal(layers[s].fine_means.contiguous(), fine.contiguous())
        assert torch.equal(layers[s].coarse_means.contiguous(), coarse.contiguous())

    # last step vs the CPU oracle on two (sequence, group) pairs
    geom = O.Geometry(top_k=top_k)
    last = nsteps - 1
    for s in (1, 6):
        k = layers[s].keys.float().cpu().numpy()
        v = layers[s].values.float().cpu().numpy()
        q = qs[last, s:s + 1].float().cpu().numpy()
        fine = O.window_means(k, 32, 16)
        pos = layers[s].length - 1
        ref = O.two_stage_attention(q, k, v, fine, geom, pos)
        assert np.array_equal(sel[s].cpu().numpy(), ref.selection[0]), (s, sel[s].tolist(), ref.selection[0])
        err = np.abs(out[s].float().cpu().numpy() - ref.out[0])
        assert (err <= OUT_ABS + OUT_REL * np.abs(ref.out[0])).all(), err.max()


@pytest.mark.parametrize("top_k", [1, 2, 3])
def test_decode_consume_budget_zero(top_k):
    """forced_consume_budget with top_k <= |forced|: budget 0 while free blocks
    remain -> the selection is the forced blocks only (sparse.py:265-277)."""
    cfg = P.SparseAttentionConfig(top_k=top_k, forced_consume_budget=True)
    lengths = [5000, 777, 130]
    gen = torch.Generator(device="cuda").manual_seed(7)
    layers, ref_layers = [], []
    for L in lengths:
        k = torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
        v = torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
        a = P.BlockizedLayerCache(HKV, D, cfg)
        a.append(k, v)
        b = P.BlockizedLayerCache(HKV, D, cfg)
        b.append(k, v)
        layers.append(a)
        ref_layers.append(b)
    batch = P.DecodeBatch(layers, cfg)
    for st in range(3):
        q = torch.randn((len(lengths), HQ, D), generator=gen, device="cuda").to(torch.bfloat16)
        kn = torch.randn((len(lengths), HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
        vn = torch.randn((len(lengths), HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
        out, sel = batch.step(q, kn, vn, return_selection=True, out_dtype=torch.float32)
        for i, ref in enumerate(ref_layers):
            ref.append(kn[i:i + 1], vn[i:i + 1])
            o2, s2 = P.two_stage_attention(q[i:i + 1], ref, cfg, ref.length - 1, return_selection=True,
                                           out_dtype=torch.float32, exact=True)
            assert torch.equal(sel[i], s2[0]), (top_k, i, sel[i].tolist(), s2[0].tolist())
            pos = ref.length - 1
            forced = P.force_blocks(pos // 64 + 1, pos // 64, 1, 2)
            got = sel[i, 0][sel[i, 0] >= 0].cpu().numpy()
            if top_k <= len(forced):
                assert np.array_equal(got, forced), (got, forced)
            assert (out[i] - o2[0]).abs().max().item() < OUT_ABS
