"""K1 (infllm2_append_compress: fused append + fine/coarse kernel-mean re-sync)
edge cases, each checked BITWISE against a from-scratch rebuild
(build_kernels, sparse.py:76-91; the reference's own invariant incremental ==
rebuild, test_sparse.py:276-290) after every operation:
random single-row and multi-row appends and truncates (crossing window and
coarse-stride boundaries, including the F18 case), float32 sources (rounded to
bf16 on the way in), both production head geometries, coarse strides 16/64/128
and the reference's tiny test geometry (the scalar path)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402


def _check(layer, keys):
    assert torch.equal(layer.keys.contiguous(), keys.to(torch.bfloat16))
    f, c = layer.rebuild_kernels()
    assert torch.equal(layer.fine_means.contiguous(), f.contiguous())
    assert torch.equal(layer.coarse_means.contiguous(), c.contiguous())
    n_f, n_c = layer._nk_valid, layer._nc_valid
    # the bf16 split the tensor-core scorer reads
    hi = layer._fine_hi[:, :n_f].transpose(0, 1)
    assert torch.equal(hi, f.to(torch.bfloat16))
    assert torch.equal(layer._fine_lo[:, :n_f].transpose(0, 1), (f - hi.float()).to(torch.bfloat16))
    chi = layer._coarse_hi[:, :n_c].transpose(0, 1)
    assert torch.equal(chi, c.to(torch.bfloat16))


@pytest.mark.parametrize("hkv,d,cfg_kw", [(2, 128, {}), (2, 64, {}), (2, 128, dict(coarse_stride=16)),
                                          (2, 128, dict(coarse_stride=64)), (4, 256, {}),
                                          (2, 4, dict(block_size=8, kernel_size=4, kernel_stride=2,
                                                      coarse_stride=4, top_k=2))])
def test_append_truncate_sequence_bitwise(hkv, d, cfg_kw):
    cfg = P.SparseAttentionConfig(**cfg_kw)
    rng = np.random.default_rng(hkv * 1000 + d + len(cfg_kw))
    g = torch.Generator(device="cuda").manual_seed(d)
    layer = P.BlockizedLayerCache(hkv, d, cfg)          # small capacity: grows (realloc) during the test
    keys = torch.empty((0, hkv, d), device="cuda")
    for step in range(60):
        r = rng.random()
        if r < 0.15 and keys.shape[0] > 4:
            n = int(rng.integers(0, keys.shape[0]))
            layer.truncate(n)
            keys = keys[:n]
        else:
            n = int(rng.choice([1, 1, 2, 15, 16, 17, 31, 33, 127, 129, 300]))
            k = torch.randn((n, hkv, d), generator=g, device="cuda")
            if rng.random() < 0.5:
                k = k.to(torch.bfloat16)       # bf16 source; else float32 (rounded on the way in)
            v = torch.randn((n, hkv, d), generator=g, device="cuda").to(k.dtype)
            layer.append(k, v)
            keys = torch.cat([keys, k.to(torch.bfloat16).float()])
            assert torch.equal(layer.values[-n:].contiguous(), v.to(torch.bfloat16))
        assert layer.length == keys.shape[0]
        _check(layer, keys)


def test_large_prefill_then_single_row_appends_cross_coarse_boundaries():
    """A 20 000-row prefill append, then single rows across several s_c = 128
    boundaries from old % 128 >= 32 (the reference's F18 crash)."""
    cfg = P.SparseAttentionConfig()
    g = torch.Generator(device="cuda").manual_seed(5)
    k = torch.randn((20000, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=20300)
    layer.append(k, k)
    keys = k.float()
    _check(layer, keys)
    for _ in range(300):
        r = torch.randn((1, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
        layer.append(r, r)
        keys = torch.cat([keys, r.float()])
    _check(layer, keys)
