"""The oracle on BASELINE configs[0]'s reference fixture (8K prefill, every row
run by the unmodified reference: tests/golden/config0_8k_full.npz): sampled
rows select exactly what the reference selected, with the reference's float32
sgemv dots (bit-identical mode) and with float64 dots (machine-independent),
and the kernel means are bitwise the reference's."""

import json
import os

import numpy as np

from golden_util import GOLDEN
from inputs import digest, make_qkv
from oracle import infllm2_oracle as O


def _load():
    z = np.load(os.path.join(GOLDEN, "config0_8k_full.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    q, k, v = make_qkv(meta["seed"], meta["length"], meta["length"], 32, 2, 128)
    assert digest(q, k, v) == meta["input_sha"]
    return meta, z, q, k, v


def test_oracle_matches_config0_fixture():
    meta, z, q, k, v = _load()
    geom = O.Geometry(**meta["geometry"])
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    assert digest(fine) == meta["fine_sha"]
    assert digest(O.window_means(k, geom.kernel_size, geom.coarse_stride)) == meta["coarse_sha"]
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([[0, 1, 63, 64, 65, 4095, 4096, 8191], rng.integers(0, 8192, 120)]))
    for dot in ("sgemv", "f64"):
        res = O.two_stage_attention(q, k, v, fine, geom, 0, rows=rows, dot=dot)
        assert np.array_equal(res.selection[rows], z["selection"][rows].astype(np.int64)), dot
    # outputs of the stored rows that were sampled, sgemv mode: float32-exact
    pos_of = {int(r): j for j, r in enumerate(z["out_rows"])}
    common = [r for r in rows if int(r) in pos_of]
    res = O.two_stage_attention(q, k, v, fine, geom, 0, rows=np.asarray(common), dot="sgemv")
    want = z["out"][[pos_of[int(r)] for r in common]]
    assert np.max(np.abs(res.out[common] - want)) <= 1e-6
