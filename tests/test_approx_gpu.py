"""Opt-in approx-LSE selection mode on the GPU:
``two_stage_attention(..., lse="approx")`` → ``infllm2_select_approx``.

* vs the fixtures composed from the reference's own functions
  (tests/golden/make_golden_approx.py): selections identical per (row, group)
  on the float64 CUDA-core path and the tensor-core path, outputs within the
  usual bars;
* tensor-core vs float64 verifier at larger caches (8B and 0.5B shapes) and at
  the full 128K size;
* with no coarse kernel (L < s_c) the mode is the exact one.
"""

import json
import os

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: F401

from golden_util import GOLDEN
from cases import build_inputs
from inputs import digest, make_qkv
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402

NAMES = sorted(os.path.basename(p)[:-4] for p in os.listdir(GOLDEN) if p.startswith("approx_") and p.endswith(".npz"))


def _load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    q, k, v = build_inputs(meta["seed"], meta["length"], meta["n_q"], meta["hq"], meta["hkv"], meta["d"],
                           meta["scale"], meta["kind"])
    assert digest(q, k, v) == meta["input_sha"]
    return meta, z, q, k, v


def _check_near_ties(s_tc, s_f64, q, k, v, geom, start, max_frac=2e-4):
    """Tensor-core (float32 accumulation) vs float64 selections: identical
    except for rare (row, group) pairs whose float64 oracle shows a near-tie
    at the top-k boundary (relative margin < 1e-5)."""
    bad = torch.nonzero((s_tc != s_f64).any(-1)).cpu().numpy()
    assert len(bad) <= max(1, int(max_frac * s_tc.shape[0] * s_tc.shape[1])), len(bad)
    if len(bad) == 0:
        return
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    coarse = O.window_means(k, geom.kernel_size, geom.coarse_stride)
    rows = np.unique(bad[:, 0])
    ref = O.two_stage_attention(q, k, v, fine, geom, start, rows=rows, lse_mode="approx", coarse_means=coarse,
                                keep_scores=True)
    top = {(i, g): float(np.max(sc)) for i, g, sc in ref.scores}
    for r, g in bad:
        assert ref.margins[r, g] < 1e-5 * top[(int(r), int(g))], (int(r), int(g), ref.margins[r, g])


def _run(meta, z, q, k, v, exact):
    cfg = P.SparseAttentionConfig(**meta["geometry"])
    layer = P.BlockizedLayerCache(meta["hkv"], meta["d"], cfg, capacity=meta["length"])
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    rows = z["rows"]
    qd = torch.from_numpy(q[rows]).cuda()
    sels, outs = [], []
    for run in np.split(np.arange(rows.size), np.flatnonzero(np.diff(rows) != 1) + 1):
        o, s = P.two_stage_attention(qd[run[0]:run[-1] + 1], layer, cfg, meta["start"] + int(rows[run[0]]),
                                     return_selection=True, out_dtype=torch.float32, exact=exact, lse="approx")
        sels.append(s)
        outs.append(o)
    return torch.cat(sels).cpu().numpy(), torch.cat(outs).cpu().numpy()


@pytest.mark.parametrize("exact", [True, False], ids=["simt", "default"])
@pytest.mark.parametrize("name", NAMES)
def test_approx_vs_reference_composition(name, exact):
    meta, z, q, k, v = _load(name)
    sel, out = _run(meta, z, q, k, v, exact)
    bad = np.argwhere((sel != z["selection"]).any(axis=-1))
    assert bad.size == 0, f"{len(bad)} (row, group) selections differ, first {bad[:4].tolist()}"
    pos_of = {int(r): j for j, r in enumerate(z["rows"])}
    got = out[[pos_of[int(r)] for r in z["out_rows"]]]
    want = z["out"]
    if exact:
        assert np.max(np.abs(got - want)) <= 1e-5
    else:
        assert np.all(np.abs(got - want) <= OUT_ABS + OUT_REL * np.abs(want))


@pytest.mark.parametrize("shape", [(32, 2, 128), (16, 2, 64)], ids=["8B", "0.5B"])
@pytest.mark.parametrize("length,topk", [(8192, 16), (6000, 64)])
def test_approx_tensor_core_vs_verifier_and_oracle(length, topk, shape):
    hq, hkv, d = shape
    cfg = P.SparseAttentionConfig(top_k=topk)
    q, k, v = make_qkv(4321 + length, length, length, hq, hkv, d)
    layer = P.BlockizedLayerCache(hkv, d, cfg, capacity=length)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    o, s = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, out_dtype=torch.float32, lse="approx")
    o2, s2 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, out_dtype=torch.float32, lse="approx",
                                   exact=True)
    geom = O.Geometry(top_k=topk)
    _check_near_ties(s, s2, q, k, v, geom, 0)
    same = (s == s2).all(-1).repeat_interleave(hq // hkv, dim=1)
    ok = (o - o2).abs() <= OUT_ABS + OUT_REL * o2.abs()
    assert bool(ok[same].all())
    # sampled rows vs the oracle (float64 dots)
    rows = np.unique(np.concatenate([[0, 127, 128, length - 1], np.random.default_rng(length).integers(0, length, 24)]))
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    coarse = O.window_means(k, geom.kernel_size, geom.coarse_stride)
    ref = O.two_stage_attention(q, k, v, fine, geom, 0, rows=rows, lse_mode="approx", coarse_means=coarse)
    sn = s.cpu().numpy()
    mism = [(int(r), g) for r in rows for g in range(hkv) if not np.array_equal(sn[r, g], ref.selection[r, g])]
    assert not mism, mism[:5]
    # and it is a different selection rule from the exact one
    e = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True)[1]
    assert bool((e != s).any())


def test_approx_full_size_128k():
    L = 131072
    cfg = P.SparseAttentionConfig(top_k=16)
    g = torch.Generator(device="cuda").manual_seed(5)
    k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(k, v)
    kn, vn = k.float().cpu().numpy(), v.float().cpu().numpy()
    for start, n in ((0, 40), (L - 64, 64)):
        q = torch.randn((n, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
        o, s = P.two_stage_attention(q, layer, cfg, start, return_selection=True, out_dtype=torch.float32,
                                     lse="approx")
        o2, s2 = P.two_stage_attention(q, layer, cfg, start, return_selection=True, out_dtype=torch.float32,
                                       lse="approx", exact=True)
        _check_near_ties(s, s2, q.float().cpu().numpy(), kn, vn, O.Geometry(top_k=16), start, max_frac=0.02)
        same = (s == s2).all(-1).repeat_interleave(16, dim=1)
        err = (o - o2).abs()
        assert bool((err <= OUT_ABS + OUT_REL * o2.abs())[same].all())


def test_approx_is_exact_without_coarse_kernels_and_validates():
    cfg = P.SparseAttentionConfig(top_k=16)
    q, k, v = make_qkv(77, 100, 100, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    a = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, lse="approx")[1]
    e = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True)[1]
    assert torch.equal(a, e)
    with pytest.raises(P.ValidationError):
        P.two_stage_attention(qd, layer, cfg, 0, lse="bogus")


def test_approx_after_batched_decode_steps():
    """Decode steps maintain the float32 coarse means only; the approx mode
    re-derives their bf16 split, so a decoded cache selects like a cache built
    from the same rows in one append (the length 2045 -> 2051 crosses a coarse
    window)."""
    cfg = P.SparseAttentionConfig(top_k=8)
    L0, steps = 2045, 6
    q, k, v = make_qkv(99, L0 + steps, 64, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(torch.from_numpy(k[:L0]).cuda(), torch.from_numpy(v[:L0]).cuda())
    batch = P.DecodeBatch([layer], cfg)
    for st in range(steps):
        batch.step(torch.from_numpy(q[st:st + 1]).cuda(), torch.from_numpy(k[L0 + st:L0 + st + 1]).cuda(),
                   torch.from_numpy(v[L0 + st:L0 + st + 1]).cuda())
    ref = P.BlockizedLayerCache(2, 128, cfg)
    ref.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    L = L0 + steps
    a = P.two_stage_attention(qd, layer, cfg, L - 64, return_selection=True, lse="approx")[1]
    b = P.two_stage_attention(qd, ref, cfg, L - 64, return_selection=True, lse="approx")[1]
    assert torch.equal(a, b)
    assert torch.equal(layer._coarse_hi[:, :L // 128], ref._coarse_hi[:, :L // 128])
