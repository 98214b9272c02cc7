"""Model seam (forward(..., backend=...) / make_cache, model.py:386-462,
specdec.py:632-641) and the per-stage functions (sparse.py:163-384) on the GPU.

* logits of a 300-token prefill + three decode steps vs the UNMODIFIED
  reference's (tests/golden/model_seam.npz, made by make_golden_model.py) for
  both backends; the only systematic difference is the bf16 K/V cache, so the
  bar is relative to the logit scale;
* the reference's degradation property (test_sparse.py:418-437): with a top-k
  covering every block, the sparse backend equals the dense one;
* each stage function vs the oracle's restatement.
"""

import ast
import types

import numpy as np
import pytest
import torch

import os

from golden_util import GOLDEN
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import model as M  # noqa: E402
from paper_2506_07900_b200 import stages as S  # noqa: E402


def _bundle():
    z = np.load(os.path.join(GOLDEN, "model_seam.npz"))
    cfg = ast.literal_eval(bytes(z["config"]).decode())
    sparse = ast.literal_eval(bytes(z["sparse"]).decode())
    params = {k[len("param:"):]: z[k] for k in z.files if k.startswith("param:")}
    c = types.SimpleNamespace(rope_base=10000.0, tied_lm_head=True, **cfg)
    bundle = types.SimpleNamespace(config=c, params=params, lm_head=params["embedding"])
    return bundle, sparse, z


def _run(bundle, backend, sc, tokens):
    cache = M.make_cache(bundle, backend, sc)
    steps = [M.forward(bundle, tokens[:300], cache, backend=backend, sparse_config=sc).logits]
    for t in range(300, len(tokens)):
        steps.append(M.forward(bundle, tokens[t:t + 1], cache, backend=backend, sparse_config=sc).logits)
    assert cache.length == len(tokens)
    return torch.cat(steps).cpu().numpy()


@pytest.mark.parametrize("backend", ["dense", "sparse"])
def test_forward_logits_vs_reference(backend):
    bundle, sparse, z = _bundle()
    sc = P.SparseAttentionConfig(**sparse) if backend == "sparse" else None
    got = _run(bundle, backend, sc, z["tokens"])
    want = z[f"logits_{backend}"]
    scale = np.abs(want).max()
    err = np.abs(got - want)
    row = err.max(axis=1)
    # The bf16 K/V cache (relative 2^-9 per element, amplified by the scale-0.2
    # weights) is the only systematic difference: measured mean 1.4e-3*scale,
    # p95 row 1.2e-2*scale.  With the sparse backend, bf16 keys also move the
    # kernel means, so a near-tie selection can flip and that row
    # attends other blocks: allow at most 1% of rows beyond 5e-2*scale.
    assert err.mean() <= 5e-3 * scale
    assert np.percentile(row, 95) <= 2e-2 * scale
    assert (row > 5e-2 * scale).mean() <= 0.01
    # the next-token choice is the observable that matters to a caller
    assert (got.argmax(-1) == want.argmax(-1)).mean() >= 0.95


def test_sparse_equals_dense_when_every_block_is_selected():
    bundle, _, z = _bundle()
    sc = P.SparseAttentionConfig(top_k=64)          # 303 tokens -> <= 5 blocks: dense regime
    dense = _run(bundle, "dense", None, z["tokens"])
    sparse = _run(bundle, "sparse", sc, z["tokens"])
    assert np.abs(sparse - dense).max() <= 1e-4 * max(1.0, np.abs(dense).max())


def test_forward_validation():
    bundle, _, z = _bundle()
    with pytest.raises(P.ValidationError):
        M.forward(bundle, np.array([], dtype=np.int64))
    with pytest.raises(P.ValidationError):
        M.forward(bundle, np.array([999]))
    with pytest.raises(P.ValidationError):
        M.forward(bundle, z["tokens"][:4], backend="flash")
    with pytest.raises(P.ValidationError):
        M.make_cache(bundle, "flash")


def test_stage_functions_vs_oracle():
    rng = np.random.default_rng(11)
    d, g, nk, L = 128, 16, 300, 4800
    q = rng.standard_normal((g, d)).astype(np.float32)
    means = rng.standard_normal((nk, d)).astype(np.float32)
    per_head = torch.stack([S.kernel_scores(q[h], means) for h in range(g)])
    assert per_head.dtype == torch.float64
    gs = S.group_scores(per_head)
    ref_gs = O.group_kernel_scores(q, means, "sgemv")
    assert np.allclose(gs.cpu().numpy(), ref_gs, rtol=1e-5, atol=1e-12)
    geom = O.Geometry(top_k=8)
    pos = L - 1
    blocks = [(b * 64, min((b + 1) * 64, pos + 1)) for b in range(pos // 64 + 1)]
    rb = S.block_scores(ref_gs, blocks, 32, 16).cpu().numpy()
    assert np.array_equal(rb, O.block_scores(ref_gs, pos, geom))
    forced = O.force_blocks(len(blocks), pos // 64, 1, 2)
    for consume in (False, True):
        got = S.select_topk(rb, 8, forced, forced_consume_budget=consume).cpu().numpy()
        assert np.array_equal(got, O.select_topk(rb, 8, forced, consume))
    # reference known-answer cases (test_sparse.py:199-213)
    assert S.select_topk(np.array([0.5, 0.9, 0.9, 0.9, 0.1]), 2, np.array([], dtype=np.int64)).tolist() == [1, 2]
    assert S.select_topk(np.ones(6), 3, np.array([], dtype=np.int64)).tolist() == [0, 1, 2]
    assert S.select_topk(np.array([0.1, 0.2, 0.3, 0.4]), 2, np.array([0])).tolist() == [0, 2, 3]
    assert S.select_topk(np.array([0.1, 0.2, 0.3, 0.4]), 2, np.array([0]),
                         forced_consume_budget=True).tolist() == [0, 3]
    with pytest.raises(P.ValidationError):
        S.select_topk(np.ones(3), 0, np.array([], dtype=np.int64))
    coarse = rng.standard_normal((nk // 8, d)).astype(np.float32)
    assert abs(S.exact_lse(q[0], means) - O.exact_lse(q[0], means)) < 1e-5
    assert abs(S.approx_lse(q[0], coarse, 16, 128) - O.approx_lse(q[0], coarse, 16, 128)) < 1e-5
    with pytest.raises(P.ValidationError):
        S.approx_lse(q[0], coarse, 16, 100)
    keys = rng.standard_normal((L, 2, d)).astype(np.float32)
    values = rng.standard_normal((L, 2, d)).astype(np.float32)
    sel = O.select_topk(rb, 8, forced)
    out, rows = S.sparse_attend(q, keys, values, sel, blocks, pos, 1, g)
    ref_rows = O.selected_rows(sel, pos, 64)
    ref_out, _ = O.sparse_attend(q, keys[:, 1], values[:, 1], ref_rows, "sgemv")
    assert rows == ref_rows.size
    assert np.abs(out.cpu().numpy() - ref_out).max() < 1e-5
    with pytest.raises(P.ValidationError):
        S.sparse_attend(q, keys, values, np.array([], dtype=np.int64), blocks, pos, 1, g)
    with pytest.raises(P.NumericError):
        S.kernel_scores(np.full(d, np.nan, dtype=np.float32), means)
