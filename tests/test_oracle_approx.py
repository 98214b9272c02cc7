"""Pin the oracle's opt-in approx-LSE selection mode to
fixtures composed from the reference's own functions
(tests/golden/make_golden_approx.py: approx_lse, group_scores, block_scores,
force_blocks, select_topk, sparse_attend of the unmodified reference).

* selections identical per (row, group) with the reference's float32 dots
  (``dot="sgemv"``), outputs within 1e-6;
* the mode reduces to the exact one when the cache holds no coarse kernel
  (L < s_c) and differs from it otherwise (a third of selections).
"""

import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN
from inputs import digest
from cases import build_inputs
from oracle import infllm2_oracle as O

NAMES = sorted(os.path.basename(p)[:-4] for p in os.listdir(GOLDEN) if p.startswith("approx_") and p.endswith(".npz"))


def _load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    q, k, v = build_inputs(meta["seed"], meta["length"], meta["n_q"], meta["hq"], meta["hkv"], meta["d"],
                           meta["scale"], meta["kind"])
    assert digest(q, k, v) == meta["input_sha"], "input generator drifted from the fixture"
    return meta, z, q, k, v


def _run(meta, q, k, v, rows, mode, dot="sgemv"):
    geom = O.Geometry(**meta["geometry"])
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    coarse = O.window_means(k, geom.kernel_size, geom.coarse_stride)
    assert digest(fine) == meta["fine_sha"] and digest(coarse) == meta["coarse_sha"]
    return O.two_stage_attention(q, k, v, fine, geom, meta["start"], rows=rows, dot=dot, lse_mode=mode,
                                 coarse_means=coarse)


def test_fixtures_present():
    assert len(NAMES) >= 7


@pytest.mark.parametrize("name", NAMES)
def test_approx_selection_and_outputs(name):
    meta, z, q, k, v = _load(name)
    rows = z["rows"]
    res = _run(meta, q, k, v, rows, "approx")
    got = res.selection[rows]
    bad = np.argwhere((got != z["selection"]).any(axis=-1))
    assert bad.size == 0, f"{len(bad)} (row, group) selections differ, first {bad[:5].tolist()}"
    assert np.max(np.abs(res.out[z["out_rows"]] - z["out"])) <= 1e-6


def test_approx_equals_exact_without_coarse_kernels():
    meta, z, q, k, v = _load("approx_b8_short")          # L = 100 < s_c = 128
    rows = z["rows"]
    a = _run(meta, q, k, v, rows, "approx")
    e = _run(meta, q, k, v, rows, "exact")
    assert np.array_equal(a.selection, e.selection)


def test_approx_differs_from_exact_at_length():
    meta, z, q, k, v = _load("approx_b8_2k")
    rows = z["rows"]
    a = _run(meta, q, k, v, rows, "approx")
    e = _run(meta, q, k, v, rows, "exact")
    differ = (a.selection[rows] != e.selection[rows]).any(axis=-1).mean()
    assert 0.02 < differ < 0.9        # a different selection rule, not a different algorithm


def test_approx_mode_validation():
    meta, z, q, k, v = _load("approx_small")
    geom = O.Geometry(**meta["geometry"])
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    with pytest.raises(O.OracleValidationError):
        O.two_stage_attention(q, k, v, fine, geom, 0, lse_mode="approx")
    with pytest.raises(O.OracleValidationError):
        O.two_stage_attention(q, k, v, fine, geom, 0, lse_mode="bogus")
