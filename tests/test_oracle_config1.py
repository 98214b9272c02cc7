"""The oracle on BASELINE configs[1]'s reference fixture (32K prefill + 256
decode steps, tests/golden/config1_32k_decode.npz): sampled prefill rows and
decode steps select exactly what the reference selected (float32 sgemv dots)."""

import json
import os

import numpy as np

from golden_util import GOLDEN
from inputs import digest, make_qkv
from oracle import infllm2_oracle as O


def test_oracle_matches_config1_fixture():
    z = np.load(os.path.join(GOLDEN, "config1_32k_decode.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    L0, steps = meta["L0"], meta["steps"]
    q, k, v = make_qkv(meta["seed"], L0 + steps, L0 + steps, 32, 2, 128)
    assert digest(q, k, v) == meta["input_sha"]
    geom = O.Geometry(**meta["geometry"])
    fine0 = O.window_means(k[:L0], geom.kernel_size, geom.kernel_stride)
    rows = z["prefill_rows"]
    pick = np.linspace(0, rows.size - 1, 8).round().astype(int)
    res = O.two_stage_attention(q[:L0], k[:L0], v[:L0], fine0, geom, 0, rows=rows[pick], dot="sgemv")
    assert np.array_equal(res.selection[rows[pick]], z["prefill_sel"][pick])
    for st in (0, 127, 128, 255):               # 128: the step whose single-row append trips F18
        pos = L0 + st
        fine = O.window_means(k[:pos + 1], geom.kernel_size, geom.kernel_stride)
        r = O.two_stage_attention(q[pos:pos + 1], k[:pos + 1], v[:pos + 1], fine, geom, pos, dot="sgemv")
        assert np.array_equal(r.selection[0], z["decode_sel"][st]), st
