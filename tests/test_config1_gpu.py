"""BASELINE configs[1]: one 8B-shaped layer, 32K prefill followed by 256 decode
steps on the B200, against the unmodified reference
(tests/golden/config1_32k_decode.npz, made by make_golden_config1.py).

* prefill (tensor-core stage 1 + 2 over all 32 768 rows): block indices of 96
  sampled rows identical to the reference's, outputs within the tensor-core bar;
* 256 batched decode steps (``DecodeBatch``: append + incremental kernel
  re-sync + fused cluster kernel): every step's block indices identical to the
  reference's, outputs of every 16th step within float32 noise;
* kernel means after the last step bitwise equal to the reference's.
"""

import json
import os

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL  # noqa: F401

from golden_util import GOLDEN
from inputs import digest, make_qkv

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402


def test_config1_32k_prefill_then_256_decode_steps():
    z = np.load(os.path.join(GOLDEN, "config1_32k_decode.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    L0, steps = meta["L0"], meta["steps"]
    q, k, v = make_qkv(meta["seed"], L0 + steps, L0 + steps, 32, 2, 128)
    assert digest(q, k, v) == meta["input_sha"]
    cfg = P.SparseAttentionConfig(**meta["geometry"])
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L0 + steps)
    layer.append(torch.from_numpy(k[:L0]).cuda(), torch.from_numpy(v[:L0]).cuda())

    # ---- 32K prefill, all rows in one call
    out, sel = P.two_stage_attention(torch.from_numpy(q[:L0]).cuda(), layer, cfg, 0, return_selection=True,
                                     out_dtype=torch.float32)
    rows = z["prefill_rows"]
    got = sel[torch.as_tensor(rows, device="cuda").long()].cpu().numpy()
    bad = np.argwhere((got != z["prefill_sel"]).any(-1))
    assert bad.size == 0, f"prefill: {len(bad)} (row, group) selections differ, first {bad[:4].tolist()}"
    o = out[torch.as_tensor(z["prefill_out_rows"], device="cuda").long()].cpu().numpy()
    want = z["prefill_out"]
    assert (np.abs(o - want) <= OUT_ABS + OUT_REL * np.abs(want)).all()

    # ---- 256 decode steps
    batch = P.DecodeBatch([layer], cfg)
    outs = []
    for st in range(steps):
        pos = L0 + st
        o1, s1 = batch.step(torch.from_numpy(q[pos:pos + 1]).cuda(), torch.from_numpy(k[pos:pos + 1]).cuda(),
                            torch.from_numpy(v[pos:pos + 1]).cuda(), return_selection=True, out_dtype=torch.float32)
        assert np.array_equal(s1[0].cpu().numpy(), z["decode_sel"][st]), (st, s1[0].tolist())
        if st % 16 == 15:
            outs.append(o1[0].cpu().numpy())
    assert layer.length == L0 + steps
    assert np.max(np.abs(np.stack(outs) - z["decode_out"])) <= 2e-4
    fine = layer.fine_means.contiguous().cpu().numpy()
    coarse = layer.coarse_means.contiguous().cpu().numpy()
    assert digest(fine) == meta["fine_sha_end"] and digest(coarse) == meta["coarse_sha_end"]
