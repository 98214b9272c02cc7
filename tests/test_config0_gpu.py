"""BASELINE configs[0] on the B200: one 8B-shaped layer, 8K prefill, k = 16,
EVERY row against the unmodified reference (tests/golden/config0_8k_full.npz,
made by make_golden_config0.py).

* block selection: identical ascending ids for all 8192 x 2 (row, group) pairs;
* outputs (float32 out, tensor-core stage 2 with bf16 softmax weights) of the
  271 stored rows within the tensor-core bar, split_p within the tight bar;
* LSE vs the oracle (float64 dots over the same selection) within 1e-5 ... see
  the bars below; kernel means bitwise.
"""

import json
import os

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL, SPLIT_ABS, SPLIT_REL  # noqa: F401
from envelope import record
from golden_util import GOLDEN
from inputs import digest, make_qkv
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402



def test_config0_8k_every_row_vs_reference():
    z = np.load(os.path.join(GOLDEN, "config0_8k_full.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    L = meta["length"]
    q, k, v = make_qkv(meta["seed"], L, L, 32, 2, 128)
    assert digest(q, k, v) == meta["input_sha"]
    cfg = P.SparseAttentionConfig(**meta["geometry"])
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    assert digest(layer.fine_means.contiguous().cpu().numpy()) == meta["fine_sha"]
    assert digest(layer.coarse_means.contiguous().cpu().numpy()) == meta["coarse_sha"]
    qd = torch.from_numpy(q).cuda()
    out, sel, lse = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True,
                                          out_dtype=torch.float32)
    sel = sel.cpu().numpy()
    bad = np.argwhere((sel != z["selection"].astype(np.int32)).any(-1))
    assert bad.size == 0, f"{len(bad)} of {L * 2} (row, group) selections differ, first {bad[:4].tolist()}"
    rows = torch.as_tensor(z["out_rows"], device="cuda").long()
    want = z["out"]
    got = out[rows].cpu().numpy()
    err = np.abs(got - want)
    record("config0_out", max_abs=err.max(), max_rel=(err / (np.abs(want) + 1e-3)).max())
    assert (err <= OUT_ABS + OUT_REL * np.abs(want)).all(), err.max()
    o2 = P.two_stage_attention(qd, layer, cfg, 0, out_dtype=torch.float32, split_p=True)
    err2 = np.abs(o2[rows].cpu().numpy() - want)
    record("config0_out_split_p", max_abs=err2.max())
    assert (err2 <= SPLIT_ABS + SPLIT_REL * np.abs(want)).all(), err2.max()
    # LSE vs the oracle on 64 rows (the reference returns no LSE; the oracle's
    # is logsumexp of the same float64 stage-2 scores)
    fine = O.window_means(k, 32, 16)
    sub = z["out_rows"][::4].astype(np.int64)
    ref = O.two_stage_attention(q, k, v, fine, O.Geometry(**meta["geometry"]), 0, rows=sub)
    assert np.array_equal(ref.selection[sub], z["selection"][sub].astype(np.int64))
    lerr = np.abs(lse[torch.as_tensor(sub, device="cuda")].cpu().numpy() - ref.lse[sub])
    record("config0_lse", max_abs=lerr.max())
    assert lerr.max() <= LSE_TC, lerr.max()
