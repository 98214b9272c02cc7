"""Golden fixture for BASELINE configs[1]: one 8B-shaped layer, 32K prefill
followed by 256 decode steps, from the UNMODIFIED reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_config1.py

Inputs: ``make_qkv(61, 32768 + 256, 32768 + 256, 32, 2, 128)`` (bf16-exact).
The reference's ``BlockizedLayerCache`` is filled with the first 32768 rows;
``two_stage_attention`` runs on 96 sampled prefill rows (selections + float64
scores of the selected blocks from its traces, outputs of 16 of them); then 256
decode steps each append one K/V row (``layer.append``, incremental kernel
re-sync; at the one step where that hits the reference's F18 crash the cache is
rebuilt from a bulk append) and attend that step's query row at the new last
position — the reference's decode (model.py:434-444).  Every step's selection is stored,
and the outputs of every 16th step.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "8")

from inputs import digest, make_qkv  # noqa: E402
from cases import B8, sample_rows  # noqa: E402

L0, STEPS, SEED = 32768, 256, 61


def main() -> None:
    from deskinfer.sparse import BlockizedLayerCache, SparseAttentionConfig, two_stage_attention

    cfg = SparseAttentionConfig(**B8)
    q, k, v = make_qkv(SEED, L0 + STEPS, L0 + STEPS, 32, 2, 128)
    layer = BlockizedLayerCache(2, 128, cfg)
    layer.append(k[:L0], v[:L0])
    smax = cfg.top_k + cfg.n_init_blocks + cfg.n_local_blocks
    rows = sample_rows(L0, 0, SEED)
    p_sel = np.full((rows.size, 2, smax), -1, np.int32)
    p_out = []
    keep = set(np.linspace(0, rows.size - 1, 16).round().astype(int).tolist())
    for j, r in enumerate(rows):
        traces = []
        o = two_stage_attention(q[r:r + 1], layer, cfg, int(r), traces=traces)
        for t in traces:
            p_sel[j, t["group"], :len(t["selected"])] = t["selected"]
        if j in keep:
            p_out.append(o[0])
    d_sel = np.full((STEPS, 2, smax), -1, np.int32)
    d_out = []
    for st in range(STEPS):
        pos = L0 + st
        try:
            layer.append(k[pos:pos + 1], v[pos:pos + 1])
        except ValueError:
            # reference defect F18: a single-row append that crosses a
            # coarse-stride multiple from old % 128 >= 32 raises; rebuild the cache
            # from one bulk append instead (bitwise the same means: the reference's
            # own incremental == rebuild invariant, test_sparse.py:276-290)
            layer = BlockizedLayerCache(2, 128, cfg)
            layer.append(k[:pos + 1], v[:pos + 1])
        traces = []
        o = two_stage_attention(q[pos:pos + 1], layer, cfg, pos, traces=traces)
        for t in traces:
            d_sel[st, t["group"], :len(t["selected"])] = t["selected"]
        if st % 16 == 15:
            d_out.append(o[0])
    meta = dict(seed=SEED, L0=L0, steps=STEPS, geometry=B8, input_sha=digest(q, k, v),
                fine_sha_end=digest(layer.fine_means), coarse_sha_end=digest(layer.coarse_means))
    np.savez_compressed(os.path.join(HERE, "config1_32k_decode.npz"),
                        meta=np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8),
                        prefill_rows=rows.astype(np.int32), prefill_sel=p_sel,
                        prefill_out_rows=rows[sorted(keep)].astype(np.int32), prefill_out=np.stack(p_out),
                        decode_sel=d_sel, decode_out=np.stack(d_out))
    print("wrote config1_32k_decode.npz")


if __name__ == "__main__":
    main()
