"""GPU parity: libinfllm2 (through its C ABI) vs the reference's golden fixtures and the oracle.

Bars:
* kernel means: bitwise (sha256) equal to the reference's float32 means;
* block selection: identical ascending ids per (row, KV group), ties included;
* outputs: float32 out within 1e-5 (CUDA-core path) / OUT_ABS + OUT_REL*|ref|
  (tensor-core path, bf16 P; tests/bars.py) of the reference; LSE within 1e-5 / LSE_TC.
"""

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: F401
from envelope import record
from golden_util import case_inputs, case_names, load
from inputs import digest, make_qkv
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402


def _cfg(meta):
    return P.SparseAttentionConfig(**meta["geometry"])


def _layer(meta, k, v, cfg):
    layer = P.BlockizedLayerCache(meta["hkv"], meta["d"], cfg, capacity=meta["length"])
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    return layer


def _means_np(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().cpu().numpy()


@pytest.mark.parametrize("name", case_names())
def test_kernel_means_bitwise_vs_reference(name):
    meta, _ = load(name)
    q, k, v = case_inputs(meta)
    layer = _layer(meta, k, v, _cfg(meta))
    torch.cuda.synchronize()
    assert digest(_means_np(layer.fine_means)) == meta["fine_sha"]
    assert digest(_means_np(layer.coarse_means)) == meta["coarse_sha"]
    f, c = layer.rebuild_kernels()
    assert digest(_means_np(f)) == meta["fine_sha"]
    assert digest(_means_np(c)) == meta["coarse_sha"]


@pytest.mark.parametrize("name", ["inc_small", "inc_b8"])
def test_incremental_append_truncate_bitwise(name):
    meta, z = load(name)
    cfg = P.SparseAttentionConfig(**meta["geometry"])
    layer = P.BlockizedLayerCache(meta["hkv"], meta["d"], cfg)
    for step, (op, arg) in enumerate(z["ops"]):
        if op == 0:
            kk = make_qkv(meta["seed"] + step, int(arg), 1, 1, meta["hkv"], meta["d"])[1]
            t = torch.from_numpy(kk).cuda()
            layer.append(t, t)
        else:
            layer.truncate(int(arg))
        assert layer.length == meta["lengths"][step]
        assert digest(_means_np(layer.fine_means)) == meta["fine_sha"][step], step
        assert digest(_means_np(layer.coarse_means)) == meta["coarse_sha"][step], step


def _run_case(name, exact, split_p=False):
    meta, z = load(name)
    q, k, v = case_inputs(meta)
    cfg = _cfg(meta)
    layer = _layer(meta, k, v, cfg)
    rows = z["rows"]
    qd = torch.from_numpy(q[rows]).cuda()
    # rows may be a sample: run each contiguous run of rows as one call
    sels, outs, lses = [], [], []
    runs = np.split(np.arange(rows.size), np.flatnonzero(np.diff(rows) != 1) + 1)
    for run in runs:
        o, s, l = P.two_stage_attention(qd[run[0]:run[-1] + 1], layer, cfg, meta["start"] + int(rows[run[0]]),
                                        return_selection=True, return_lse=True,
                                        out_dtype=torch.float32, exact=exact, split_p=split_p)
        sels.append(s)
        outs.append(o)
        lses.append(l)
    sel = torch.cat(sels).cpu().numpy()
    out = torch.cat(outs).cpu().numpy()
    lse = torch.cat(lses).cpu().numpy()
    return meta, z, q, k, v, cfg, sel, out, lse


@pytest.mark.parametrize("exact", [True, False], ids=["simt", "default"])
@pytest.mark.parametrize("name", case_names())
def test_selection_and_outputs_vs_reference(name, exact):
    meta, z, q, k, v, cfg, sel, out, lse = _run_case(name, exact)
    bad = np.argwhere((sel != z["selection"]).any(axis=-1))
    assert bad.size == 0, f"{len(bad)} (row, group) selections differ, first {bad[:4].tolist()}"
    pos_of = {int(r): j for j, r in enumerate(z["rows"])}
    idx = [pos_of[int(r)] for r in z["out_rows"]]
    got = out[idx]
    want = z["out"]
    record(f"parity_{name}_{'simt' if exact else 'tc'}", out_max_abs=np.abs(got - want).max())
    if exact:
        assert np.max(np.abs(got - want)) <= 1e-5
    else:
        assert np.all(np.abs(got - want) <= OUT_ABS + OUT_REL * np.abs(want))
    # LSE vs the oracle restatement over the same (reference) selection
    geom = O.Geometry(**meta["geometry"])
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    sub = z["out_rows"][:8]
    ref = O.two_stage_attention(q, k, v, fine, geom, meta["start"], rows=sub)
    tol = 1e-5 if exact else LSE_TC
    record(f"parity_{name}_lse", lse_max_abs=np.max(np.abs(lse[[pos_of[int(r)] for r in sub]] - ref.lse[sub])))
    assert np.max(np.abs(lse[[pos_of[int(r)] for r in sub]] - ref.lse[sub])) <= tol


@pytest.mark.parametrize("name", case_names())
def test_split_p_outputs_tight(name):
    """Tensor-core stage 2 with the softmax weights as bf16 hi + lo
    (split_p=True): outputs within 2e-5 + 1e-4|ref| of the reference."""
    meta, z, q, k, v, cfg, sel, out, lse = _run_case(name, False, split_p=True)
    assert np.array_equal(sel, z["selection"])
    pos_of = {int(r): j for j, r in enumerate(z["rows"])}
    got = out[[pos_of[int(r)] for r in z["out_rows"]]]
    want = z["out"]
    assert np.all(np.abs(got - want) <= 2e-5 + 1e-4 * np.abs(want))


def test_touch_stats_and_traces_match_reference_counts():
    meta, z = load("b8_2k_prefill")
    q, k, v = case_inputs(meta)
    cfg = _cfg(meta)
    layer = _layer(meta, k, v, cfg)
    stats = P.TouchStats()
    traces = []
    P.two_stage_attention(torch.from_numpy(q).cuda(), layer, cfg, 0, stats=stats, traces=traces)
    assert stats.stage1 == meta["stage1_rows"]
    assert stats.stage2 == meta["stage2_rows"]
    assert stats.dense_rows == meta["dense_rows"]
    assert len(traces) == 2 * 2048
    t = traces[2 * 1500 + 1]
    assert t["query_pos"] == 1500 and t["group"] == 1
    assert t["selected"] == [int(b) for b in z["selection"][1500, 1] if b >= 0]
    np.testing.assert_allclose(t["scores_topk"], z["scores_topk"][1500, 1, :len(t["selected"])], rtol=1e-5)


@pytest.mark.parametrize("shape", [(32, 2, 128), (16, 2, 64)], ids=["8B", "0.5B"])
@pytest.mark.parametrize("length,topk", [(8192, 16), (6000, 64), (4096, 8), (5000, 32)])
def test_random_vs_oracle_sampled_rows(length, topk, shape):
    """Larger caches than the fixtures: GPU vs oracle (f64 dots) on sampled rows,
    for the MiniCPM4-8B attention shape and the 0.5B one (G = 8, D = 64)."""
    hq, hkv, d = shape
    geom = O.Geometry(top_k=topk)
    cfg = P.SparseAttentionConfig(top_k=topk)
    q, k, v = make_qkv(1234 + length, length, length, hq, hkv, d)
    layer = P.BlockizedLayerCache(hkv, d, cfg, capacity=length)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    o, s, l = P.two_stage_attention(torch.from_numpy(q).cuda(), layer, cfg, 0, return_selection=True,
                                    return_lse=True, out_dtype=torch.float32)
    s, o, l = s.cpu().numpy(), o.cpu().numpy(), l.cpu().numpy()
    rng = np.random.default_rng(length)
    rows = np.unique(np.concatenate([[0, 63, 64, length - 1], rng.integers(0, length, 40)]))
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    ref = O.two_stage_attention(q, k, v, fine, geom, 0, rows=rows)
    mism = [(int(r), g, float(ref.margins[r, g])) for r in rows for g in range(2)
            if not np.array_equal(s[r, g], ref.selection[r, g])]
    assert not mism, f"selection mismatches (row, group, oracle margin): {mism[:5]}"
    assert np.all(np.abs(o[rows] - ref.out[rows]) <= OUT_ABS + OUT_REL * np.abs(ref.out[rows]))
    assert np.max(np.abs(l[rows] - ref.lse[rows])) <= LSE_TC


def test_decode_steps_match_prefill_rows():
    """Appending one row at a time (decode) == the same rows in one prefill call
    when the cache length is the same at call time."""
    cfg = P.SparseAttentionConfig(top_k=16)
    q, k, v = make_qkv(77, 3000, 3000, 32, 2, 128)
    kd, vd, qd = (torch.from_numpy(x).cuda() for x in (k, v, q))
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(kd[:2900], vd[:2900])
    for t in range(2900, 3000):
        layer.append(kd[t:t + 1], vd[t:t + 1])
        o, s = P.two_stage_attention(qd[t:t + 1], layer, cfg, t, return_selection=True,
                                     out_dtype=torch.float32)
        ref_layer = P.BlockizedLayerCache(2, 128, cfg)
        if t % 25 == 0:
            ref_layer.append(kd[:t + 1], vd[:t + 1])
            o2, s2 = P.two_stage_attention(qd[t:t + 1], ref_layer, cfg, t, return_selection=True,
                                           out_dtype=torch.float32)
            assert torch.equal(s, s2)
            assert torch.equal(o, o2)


def test_validation_errors():
    cfg = P.SparseAttentionConfig()
    layer = P.BlockizedLayerCache(2, 128, cfg)
    k = torch.zeros(100, 2, 128, device="cuda")
    layer.append(k, k)
    with pytest.raises(P.ValidationError):
        P.two_stage_attention(torch.zeros(1, 32, 128, device="cuda"), layer, cfg, 100)
    with pytest.raises(P.ValidationError):
        P.two_stage_attention(torch.zeros(1, 31, 128, device="cuda"), layer, cfg, 10)
    with pytest.raises(P.ValidationError):
        layer.truncate(101)
    with pytest.raises(P.ValidationError):
        layer.append(torch.zeros(3, 3, 128, device="cuda"), torch.zeros(3, 3, 128, device="cuda"))


def test_dense_degradation_vs_dense_oracle():
    """Budget covers every block -> equals dense attention (test_acceptance.py:68-106)."""
    rng = np.random.default_rng(101)
    worst = 0.0
    for trial in range(30):
        m = int(rng.choice([8, 16, 32, 64]))
        cfg = P.SparseAttentionConfig(block_size=m, kernel_size=m // 2, kernel_stride=m // 4,
                                      coarse_stride=m // 2, top_k=int(rng.integers(1, 5)),
                                      n_init_blocks=int(rng.integers(0, 3)),
                                      n_local_blocks=int(rng.integers(0, 3)))
        n_blocks = int(rng.integers(1, cfg.max_selected + 1))
        length = max(n_blocks * m - int(rng.integers(0, m)), 1)
        q, k, v = make_qkv(trial, length, 1, 4, 2, 8)
        layer = P.BlockizedLayerCache(2, 8, cfg)
        layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        out = P.two_stage_attention(torch.from_numpy(q).cuda(), layer, cfg, length - 1,
                                    out_dtype=torch.float32).cpu().numpy()
        dense, _ = O.dense_attention(q, k, v, length - 1)
        worst = max(worst, float(np.abs(out - dense).max()))
    assert worst < 1e-5


class _RefLikeLayer:
    """Stand-in for deskinfer's LayerCache surface (keys/values/length/heads)."""

    def __init__(self, k, v):
        self.keys, self.values = k, v
        self.length = k.shape[0]
        self.n_kv_heads, self.head_dim = k.shape[1], k.shape[2]


@pytest.mark.parametrize("name", ["small_prefill", "b8_3k_chunk"])
def test_numpy_compat_adapter_matches_reference(name):
    """compat.two_stage_attention_numpy (the reference-signature switch in
    INTEGRATION.md) reproduces the reference's outputs and traces."""
    from paper_2506_07900_b200.compat import two_stage_attention_numpy
    meta, z = load(name)
    q, k, v = case_inputs(meta)
    cfg = _cfg(meta)
    layer = _RefLikeLayer(k, v)
    rows = z["out_rows"]
    traces = []
    for r in rows[:6]:
        out = two_stage_attention_numpy(q[r:r + 1], layer, cfg, meta["start"] + int(r), traces=traces)
        j = int(np.flatnonzero(z["out_rows"] == r)[0])
        assert out.dtype == np.float32
        assert np.all(np.abs(out[0] - z["out"][j]) <= OUT_ABS + OUT_REL * np.abs(z["out"][j]))
    pos_of = {int(r): j for j, r in enumerate(z["rows"])}
    for t in traces:
        j = pos_of[t["query_pos"] - meta["start"]]
        assert t["selected"] == [int(b) for b in z["selection"][j, t["group"]] if b >= 0]


def test_small_model_shape_chunks_and_verifier():
    """MiniCPM4-0.5B attention geometry (G = 8, D = 64) on the tensor-core path:
    a chunk starting off the 32-position unit grid equals the same rows of the
    whole prefill (selections bitwise, F12), and the tensor-core selections equal
    the float64 verifier's."""
    cfg = P.SparseAttentionConfig(top_k=16)
    q, k, v = make_qkv(505, 3000, 3000, 16, 2, 64)
    layer = P.BlockizedLayerCache(2, 64, cfg, capacity=3000)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    o, s = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, out_dtype=torch.float32)
    o2, s2 = P.two_stage_attention(qd[1001:1778], layer, cfg, 1001, return_selection=True, out_dtype=torch.float32)
    assert torch.equal(s[1001:1778], s2)
    assert (o[1001:1778] - o2).abs().max().item() < 1e-6
    o3, s3 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, out_dtype=torch.float32, exact=True)
    assert torch.equal(s, s3)
    assert bool(((o - o3).abs() <= OUT_ABS + OUT_REL * o3.abs()).all())     # bf16 softmax weights (DESIGN §4 K3p)


def test_check_finite_raises_numeric_error():
    """check_finite=True mirrors the reference's NumericError (sparse.py:176-177)."""
    cfg = P.SparseAttentionConfig(top_k=8)
    q, k, v = make_qkv(9, 512, 4, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    P.two_stage_attention(qd, layer, cfg, 508, check_finite=True)      # finite: fine
    qd[1, 3, 7] = float("nan")
    with pytest.raises(P.NumericError):
        P.two_stage_attention(qd, layer, cfg, 508, check_finite=True)


@pytest.mark.parametrize("topk", [16, 64])
def test_full_size_128k_tensor_core_vs_float64_verifier(topk):
    """At BASELINE's full size (131072-token cache, 8B shape): the tensor-core
    stage 1 + stage 2 against the float64 CUDA-core verifier (exact=True) on row
    chunks at the start, middle and end of the sequence - selections bitwise,
    outputs within the tensor-core bar."""
    L = 131072
    cfg = P.SparseAttentionConfig(top_k=topk)
    g = torch.Generator(device="cuda").manual_seed(topk)
    k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(k, v)
    for start, n in ((0, 48), (65500, 80), (L - 96, 96)):
        q = torch.randn((n, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
        o, s, l = P.two_stage_attention(q, layer, cfg, start, return_selection=True, return_lse=True,
                                        out_dtype=torch.float32)
        o2, s2, l2 = P.two_stage_attention(q, layer, cfg, start, return_selection=True, return_lse=True,
                                           out_dtype=torch.float32, exact=True)
        assert torch.equal(s, s2), (start, int((s != s2).any(-1).sum()))
        # bf16 softmax weights (hi + lo below position 256, where few keys would
        # expose the 2^-9 per-weight rounding)
        err = (o - o2).abs()
        assert bool((err <= OUT_ABS + OUT_REL * o2.abs()).all())
        assert (l - l2).abs().max().item() <= LSE_TC
        o3 = P.two_stage_attention(q, layer, cfg, start, out_dtype=torch.float32, split_p=True)
        assert (o3 - o2).abs().max().item() <= 5e-5


def test_dense_regime_shortcut_equals_scored_selection():
    """Below the sparsity threshold the selection is written without scoring
    (every candidate block); it must equal the scored selection (requesting
    the traces forces the scorer)."""
    cfg = P.SparseAttentionConfig(top_k=64)
    q, k, v = make_qkv(4040, 4096, 4096, 32, 2, 128)          # 64 blocks - 3 forced <= 64: dense
    layer = P.BlockizedLayerCache(2, 128, cfg)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    o1, s1 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, out_dtype=torch.float32)
    traces = []
    o2, s2 = P.two_stage_attention(qd[-96:], layer, cfg, 4096 - 96, return_selection=True, out_dtype=torch.float32,
                                   traces=traces)
    assert torch.equal(s1[-96:], s2)
    assert torch.equal(o1[-96:], o2)
    nb = torch.arange(64, device="cuda")
    assert torch.equal(s1[-1, 0, :64], nb.int())
