"""Tree-draft verification: ``model.forward_tree`` and
``tree.tree_attention``.

The reference verifies trees only densely (``forward_tree``, specdec.py:565-625),
so parity is anchored three ways:
* dense backend vs the reference's logits (tests/golden/model_tree.npz, made
  by make_golden_tree.py) — bf16 K/V are the only systematic difference, as in
  test_model_seam_gpu.py;
* sparse backend == dense backend in the degradation regime (every block
  selected);
* the operator in a genuinely sparse regime (8B shape, 3000-row prefix) vs the
  oracle composition: the reference's per-row two-stage algorithm at position
  base-1, dense float64 attention over ancestor rows, log-sum-exp merge.
"""

import ast
import os
import types

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: F401

from golden_util import GOLDEN
from inputs import make_qkv
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import model as M  # noqa: E402


def _bundle():
    z = np.load(os.path.join(GOLDEN, "model_seam.npz"))
    cfg = ast.literal_eval(bytes(z["config"]).decode())
    params = {k[len("param:"):]: z[k] for k in z.files if k.startswith("param:")}
    c = types.SimpleNamespace(rope_base=10000.0, tied_lm_head=True, **cfg)
    return types.SimpleNamespace(config=c, params=params, lm_head=params["embedding"]), z["tokens"]


def _tree_case(backend, sc):
    bundle, tokens = _bundle()
    t = np.load(os.path.join(GOLDEN, "model_tree.npz"))
    cache = M.make_cache(bundle, backend, sc)
    M.forward(bundle, tokens[:int(t["prefix_len"])], cache, backend=backend, sparse_config=sc)
    mask = P.PackedMask.from_parents(t["parents"])
    res = M.forward_tree(bundle, cache, t["tokens"], t["depths"], mask, backend=backend, sparse_config=sc)
    assert cache.length == int(t["prefix_len"])          # the cache is read, never modified
    return res.logits.cpu().numpy(), t["logits"]


def test_forward_tree_dense_vs_reference():
    got, want = _tree_case("dense", None)
    scale = np.abs(want).max()
    err = np.abs(got - want)
    assert err.mean() <= 5e-3 * scale
    assert err.max() <= 5e-2 * scale
    assert (got.argmax(-1) == want.argmax(-1)).mean() >= 0.9


def test_forward_tree_sparse_equals_dense_when_every_block_is_selected():
    sc = P.SparseAttentionConfig(top_k=64)              # 300-row prefix: 5 blocks, all selected
    sparse, _ = _tree_case("sparse", sc)
    dense, _ = _tree_case("dense", None)
    assert np.abs(sparse - dense).max() <= 1e-4 * max(1.0, np.abs(dense).max())


def _oracle_tree(q, k, v, fine, geom, kt, vt, vis):
    """Per node: the reference's two-stage row at position base-1 (oracle),
    dense float64 attention over the visible tree rows, log-sum-exp merge."""
    n, hq, d = q.shape
    base, hkv = k.shape[0], k.shape[1]
    g = hq // hkv
    out = np.zeros((n, hq, d), np.float64)
    sel = []
    for i in range(n):
        r = O.two_stage_attention(q[i:i + 1], k, v, fine, geom, base - 1)
        sel.append(r.selection[0])
        for h in range(hq):
            kk = kt[vis[i], h // g].astype(np.float64)
            vv = vt[vis[i], h // g].astype(np.float64)
            s = (kk @ q[i, h].astype(np.float64)) / np.sqrt(d)
            lt = O.logsumexp_f64(s)
            ot = np.exp(s - lt) @ vv
            lp = r.lse[0, h]
            m = max(lp, lt)
            wp, wt = np.exp(lp - m), np.exp(lt - m)
            out[i, h] = (r.out[0, h] * wp + ot * wt) / (wp + wt)
    return out, np.stack(sel)


@pytest.mark.parametrize("exact", [True, False], ids=["simt", "default"])
def test_tree_attention_sparse_regime_vs_oracle(exact):
    base, n, hq, hkv, d = 3000, 10, 32, 2, 128
    cfg = P.SparseAttentionConfig(top_k=8)
    geom = O.Geometry(top_k=8)
    _, k, v = make_qkv(565, base, 1, hq, hkv, d)
    q, kt, vt = make_qkv(566, n, n, hq, hkv, d)
    parents = [-1, 0, 0, 1, 2, 2, 4, -1, 7, 8]
    mask = P.PackedMask.from_parents(parents)
    layer = P.BlockizedLayerCache(hkv, d, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    out, sel = P.tree_attention(torch.from_numpy(q).cuda(), layer, cfg, torch.from_numpy(kt).cuda(),
                                torch.from_numpy(vt).cuda(), mask, exact=exact, return_selection=True)
    assert layer.length == base
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    ref_out, ref_sel = _oracle_tree(q, k, v, fine, geom, kt, vt, mask.to_dense())
    assert np.array_equal(sel.cpu().numpy(), ref_sel)
    got = out.cpu().numpy()
    if exact:
        assert np.max(np.abs(got - ref_out)) <= 1e-5
    else:
        assert np.all(np.abs(got - ref_out) <= OUT_ABS + OUT_REL * np.abs(ref_out))


def test_tree_validation():
    bundle, tokens = _bundle()
    cfg = P.SparseAttentionConfig(top_k=4)
    cache = M.make_cache(bundle, "sparse", cfg)
    mask = P.PackedMask.from_parents([-1, 0])
    with pytest.raises(P.ValidationError):
        M.forward_tree(bundle, cache, np.array([1, 2]), np.array([1, 2]), mask)      # empty prefix
    M.forward(bundle, tokens[:40], cache, backend="sparse", sparse_config=cfg)
    with pytest.raises(P.ValidationError):
        M.forward_tree(bundle, cache, np.array([1, 2, 3]), np.array([1, 2, 3]), mask)  # 3 tokens, 2-node mask
    with pytest.raises(P.ValidationError):
        P.PackedMask.from_parents([-1, 2, 0])                                         # parent after child
    with pytest.raises(P.ValidationError):
        M.forward_tree(bundle, cache, np.array([1, 2]), np.array([1, 2]), mask, backend="flash")
    bad = P.PackedMask(words=np.zeros((2, 1), np.uint64), n_nodes=2)
    with pytest.raises(P.ValidationError):
        bad.validate()


@pytest.mark.parametrize("n,base,top_k,seed", [(10, 3000, 8, 1), (40, 5000, 16, 2), (100, 4097, 16, 3),
                                                (130, 9000, 8, 4)])
def test_tree_kernel_packed_mask_vs_oracle(n, base, top_k, seed):
    """infllm2_forward_tree (tcgen05 stage 1 at the broadcast position, packed
    uint64 mask consumed in stage 2) vs the oracle composition and vs the
    float64 verifier path: selections identical, outputs within the
    tensor-core bar; > 64 nodes span several mask words and tree tiles."""
    hq, hkv, d = 32, 2, 128
    rng = np.random.default_rng(seed)
    parents = [-1] + [int(rng.integers(-1, i)) for i in range(1, n)]
    mask = P.PackedMask.from_parents(parents)
    cfg = P.SparseAttentionConfig(top_k=top_k)
    geom = O.Geometry(top_k=top_k)
    _, k, v = make_qkv(600 + seed, base, 1, hq, hkv, d)
    q, kt, vt = make_qkv(700 + seed, n, n, hq, hkv, d)
    layer = P.BlockizedLayerCache(hkv, d, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd, ktd, vtd = (torch.from_numpy(x).cuda() for x in (q, kt, vt))
    out, sel = P.tree_attention(qd, layer, cfg, ktd, vtd, mask, return_selection=True)
    assert layer.length == base
    out_x, sel_x = P.tree_attention(qd, layer, cfg, ktd, vtd, mask, exact=True, return_selection=True)
    assert torch.equal(sel, sel_x)
    assert bool(((out - out_x).abs() <= OUT_ABS + OUT_REL * out_x.abs()).all())
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    pick = sorted({0, n - 1, n // 2, min(n - 1, 65)})
    ref_out, ref_sel = _oracle_tree(q[pick], k, v, fine, geom, kt, vt, mask.to_dense()[pick])
    assert np.array_equal(sel.cpu().numpy()[pick], ref_sel)
    got = out.cpu().numpy()[pick]
    assert np.all(np.abs(got - ref_out) <= OUT_ABS + OUT_REL * np.abs(ref_out))
    # split_p: the tight bar
    out_s = P.tree_attention(qd, layer, cfg, ktd, vtd, mask, split_p=True).cpu().numpy()[pick]
    assert np.max(np.abs(out_s - ref_out)) <= 5e-5
