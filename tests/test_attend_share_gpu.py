"""Stage 2 with the forced blocks shared by 4 rows of a query block
(csrc/attend_share.cu, DESIGN §4 K3s): prefill rows at positions >= 2048 of the
MiniCPM4 geometry run on it, the rows around them on attend_tc.cu.

* outputs and LSE against the float64 verifier (exact=True) within the
  tensor-core bars, selections unchanged, bf16 and float32 outputs;
* per-row results do not depend on which rows a call groups: a call over an
  unaligned chunk equals the full call on every row both run through the
  shared kernel, bitwise;
* the shared kernel actually runs (a stage-2 call is split into its launch
  plus the attend_tc launches around it)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: E402

SHARE_FROM = 2048


def _layer(length, seed, topk=16, shape=(32, 2, 128), consume=False):
    hq, hkv, d = shape
    cfg = P.SparseAttentionConfig(top_k=topk, forced_consume_budget=consume)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn((length, hq, d), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((length, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((length, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(hkv, d, cfg, capacity=length)
    layer.append(k, v)
    return cfg, q, layer


@pytest.mark.parametrize("length,topk,shape", [(8192, 16, (32, 2, 128)), (12000, 32, (32, 2, 128)),
                                               (9000, 64, (32, 2, 128)), (8192, 16, (16, 2, 64)),
                                               (10000, 8, (16, 2, 64)), (11000, 32, (16, 2, 64)),
                                               (9500, 64, (16, 2, 64))],
                         ids=["8B-k16", "8B-k32", "8B-k64", "0.5B-k16", "0.5B-k8", "0.5B-k32", "0.5B-k64"])
def test_shared_kernel_vs_float64_verifier(length, topk, shape):
    cfg, q, layer = _layer(length, 11 + length, topk, shape)
    group = shape[0] // shape[1]
    lib = _lib.load()
    n0 = lib.infllm2_launch_count()
    o, s, l = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                    out_dtype=torch.float32)
    torch.cuda.synchronize()
    # select + attend_tc rows [0, 2048) + attend_share + (aligned tail on attend_tc)
    assert lib.infllm2_launch_count() - n0 >= 3, "stage 2 did not split into the shared-kernel launch"
    o2, s2, l2 = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                       out_dtype=torch.float32, exact=True)
    same = (s == s2).all(-1)
    assert same.float().mean().item() > 0.999          # near-ties only
    rows = torch.arange(SHARE_FROM, length, device="cuda")
    ok = same[rows].repeat_interleave(group, dim=1)
    err = (o[rows] - o2[rows]).abs()
    bar = OUT_ABS + OUT_REL * o2[rows].abs()
    assert bool((err <= bar)[ok].all()), f"max |dO| {err[ok].max().item():.3e}"
    dl = (l[rows] - l2[rows]).abs()[ok]
    assert dl.max().item() <= LSE_TC, f"max |dLSE| {dl.max().item():.3e}"


@pytest.mark.parametrize("topk", [3, 16], ids=["budget0", "budget13"])
def test_consume_budget_rows(topk):
    """forced_consume_budget: top-k 3 leaves no chosen block (rows made of the
    shared tiles alone), top-k 16 an odd 13 (a half tile per row)."""
    length = 6000
    cfg, q, layer = _layer(length, 31 + topk, topk, consume=True)
    o, s, l = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                    out_dtype=torch.float32)
    o2, s2, l2 = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                       out_dtype=torch.float32, exact=True)
    rows = torch.arange(SHARE_FROM, length, device="cuda")
    ok = (s == s2).all(-1)[rows].repeat_interleave(16, dim=1)
    assert ok.float().mean().item() > 0.999
    err = (o[rows] - o2[rows]).abs()
    assert bool((err <= OUT_ABS + OUT_REL * o2[rows].abs())[ok].all()), f"max |dO| {err[ok].max().item():.3e}"
    assert (l[rows] - l2[rows]).abs()[ok].max().item() <= LSE_TC


def test_four_kv_groups_and_strided_q():
    """HKV = 4 (HQ = 64) and q rows taken from a wider packed buffer (row
    stride > HQ * D): the shared kernel's tensor maps follow the strides."""
    length = 7000
    cfg = P.SparseAttentionConfig(top_k=16)
    g = torch.Generator(device="cuda").manual_seed(77)
    qkv = torch.randn((length, 64 + 8, 128), generator=g, device="cuda").to(torch.bfloat16)
    q = qkv[:, :64]                                     # (L, 64, 128) view, row stride 72 * 128
    k, v = qkv[:, 64:68].contiguous(), qkv[:, 68:72].contiguous()
    layer = P.BlockizedLayerCache(4, 128, cfg, capacity=length)
    layer.append(k, v)
    o, s, l = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                    out_dtype=torch.float32)
    o2, s2, l2 = P.two_stage_attention(q.contiguous(), layer, cfg, 0, return_selection=True, return_lse=True,
                                       out_dtype=torch.float32, exact=True)
    rows = torch.arange(SHARE_FROM, length, device="cuda")
    ok = (s == s2).all(-1)[rows].repeat_interleave(16, dim=1)
    assert ok.float().mean().item() > 0.999
    err = (o[rows] - o2[rows]).abs()
    assert bool((err <= OUT_ABS + OUT_REL * o2[rows].abs())[ok].all()), f"max |dO| {err[ok].max().item():.3e}"
    assert (l[rows] - l2[rows]).abs()[ok].max().item() <= LSE_TC


def test_bf16_output_matches_float32():
    cfg, q, layer = _layer(6000, 5)
    o32 = P.two_stage_attention(q, layer, cfg, 0, out_dtype=torch.float32)
    o16 = P.two_stage_attention(q, layer, cfg, 0, out_dtype=torch.bfloat16)
    assert torch.equal(o16, o32.to(torch.bfloat16))


def test_rows_independent_of_grouping():
    """An unaligned chunk (as a sharded rank calls it) and the full call agree
    bitwise on every row both send through the shared kernel."""
    length = 9000
    cfg, q, layer = _layer(length, 17)
    o, s, l = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                    out_dtype=torch.float32)
    a, b = 3001, 7003
    oc, sc, lc = P.two_stage_attention(q[a:b], layer, cfg, a, return_selection=True, return_lse=True,
                                       out_dtype=torch.float32)
    assert torch.equal(sc, s[a:b])
    lo, hi = (a + 3) // 4 * 4, b // 4 * 4               # the chunk's shared-kernel rows
    assert torch.equal(oc[lo - a:hi - a], o[lo:hi])
    assert torch.equal(lc[lo - a:hi - a], l[lo:hi])
    # the chunk's edge rows ran on attend_tc: within the bars of the full call
    edge = torch.tensor([0, 1, 2, b - a - 3, b - a - 1])
    err = (oc[edge] - o[a + edge]).abs()
    assert bool((err <= 2 * (OUT_ABS + OUT_REL * o[a + edge].abs())).all())


def test_matches_attend_tc_rows_below_threshold():
    """Rows below position 2048 are attend_tc's: a call ending there is
    bitwise the same rows of a call that also covers shared-kernel rows."""
    cfg, q, layer = _layer(8192, 23)
    o = P.two_stage_attention(q, layer, cfg, 0, out_dtype=torch.float32)
    o_head = P.two_stage_attention(q[:SHARE_FROM], layer, cfg, 0, out_dtype=torch.float32)
    assert torch.equal(o[:SHARE_FROM], o_head)
    assert np.isfinite(o.cpu().numpy()).all()
