"""Dense causal GQA attention on the tensor cores (infllm2_dense_attend, SURVEY
§8 a21): the below-threshold path of the operator and the dense backend.

* vs the float64 restatement of the reference's masked grouped attention
  (model.dense_attention, model.py:194-253) on the cache's bf16 K/V, for full
  prefills and for chunks that start mid-cache, ragged row counts included;
* in the dense regime ``two_stage_attention`` (which then routes here) equals
  the sparse kernels' result and the reference's selection (all blocks).
"""

import ctypes

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: F401

from inputs import make_qkv

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402
from paper_2506_07900_b200 import model as M  # noqa: E402
from paper_2506_07900_b200.sparse import _ptr, _stream  # noqa: E402


def _dense(q, layer, cfg, start, lse=False):
    lib = _lib.load()
    geom = cfg.geometry()
    n, hq, d = q.shape
    out = torch.empty((n, hq, d), dtype=torch.float32, device="cuda")
    l = torch.empty((n, hq), dtype=torch.float32, device="cuda") if lse else None
    kc, vc, cap, *_ = layer._device_args()
    _lib.check(lib.infllm2_dense_attend(ctypes.byref(geom), _ptr(q), q.stride(0), n, start, hq, layer.n_kv_heads, d,
                                        _ptr(kc), _ptr(vc), cap, layer.length, _ptr(out), _ptr(l),
                                        _lib.FLAG_OUT_F32, _stream(q.device)), "dense")
    return out, l


@pytest.mark.parametrize("length,start,n", [(1000, 0, 1000), (3000, 2800, 200), (4096, 0, 4096), (777, 700, 77),
                                            (130, 0, 130)])
def test_dense_kernel_vs_float64(length, start, n):
    cfg = P.SparseAttentionConfig(top_k=16)
    q, k, v = make_qkv(55 + length, length, n, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    out, l = _dense(qd, layer, cfg, start, lse=True)
    keys = layer.keys.float().reshape(length, -1)
    vals = layer.values.float().reshape(length, -1)
    ref = M.dense_attention(qd.float().reshape(n, -1), keys, vals, n_q_heads=32, n_kv_heads=2,
                            causal_offset=start).reshape(n, 32, 128)
    err = (out - ref).abs()
    assert bool((err <= OUT_ABS + OUT_REL * ref.abs()).all()), float(err.max())
    early = torch.arange(n, device="cuda") + start < 256      # hi + lo weights there
    if bool(early.any()):
        assert float(err[early].max()) <= 1e-4
    # LSE vs float64 logsumexp of the same scores
    qf = qd.double()
    kf = layer.keys.double()
    for r in (0, n // 2, n - 1):
        pos = start + r
        s = torch.einsum("hd,khd->hk", qf[r].reshape(2, 16, 128).reshape(32, 128),
                         kf[:pos + 1].repeat_interleave(16, dim=1)) / np.sqrt(128)
        assert (l[r] - torch.logsumexp(s, dim=-1)).abs().max().item() <= LSE_TC


def test_two_stage_dense_regime_routes_to_dense_kernel():
    cfg = P.SparseAttentionConfig(top_k=64)
    q, k, v = make_qkv(4141, 4096, 4096, 32, 2, 128)           # 64 blocks - 3 forced <= 64: dense regime
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    geom = cfg.geometry()
    assert _lib.load().infllm2_dense_regime(ctypes.byref(geom), 4096, 0, 4096) == 1
    assert _lib.load().infllm2_dense_regime(ctypes.byref(P.SparseAttentionConfig(top_k=16).geometry()), 4096, 0,
                                            4096) == 0
    o, s, l = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True,
                                    out_dtype=torch.float32)
    o2, s2, l2 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True,
                                       out_dtype=torch.float32, exact=True)
    assert torch.equal(s, s2)
    assert bool(((o - o2).abs() <= OUT_ABS + OUT_REL * o2.abs()).all())
    assert (l - l2).abs().max().item() <= LSE_TC


def test_dense_validation():
    cfg = P.SparseAttentionConfig(top_k=16)
    layer = P.BlockizedLayerCache(2, 64, cfg)                  # D = 64: not the dense kernel's shape
    q, k, v = make_qkv(1, 100, 10, 16, 2, 64)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda().to(torch.bfloat16)
    with pytest.raises(Exception):
        _dense(qd, layer, cfg, 0)
