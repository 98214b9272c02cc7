"""Golden fixture for BASELINE configs[0]: one 8B-shaped layer (32 q / 2 KV heads,
d 128), 8K prefill, m 64, p 32, s 16, k 16, init 1, local 2 — EVERY query row,
from the UNMODIFIED reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_config0.py

Inputs: ``make_qkv(1_000, 8192, 8192, 32, 2, 128)`` (bf16-exact float32).  The
reference's ``BlockizedLayerCache`` holds all 8192 rows; ``two_stage_attention``
runs on every row (rows are independent given the cache: chunked calls are
bitwise equal to one call), fanned over worker processes.  Stored:

* ``selection`` (8192, 2, 19) int16 — every (row, group)'s selected ids from the
  traces (sparse.py:458-467), -1 padded;
* ``margin_score`` (8192, 2) float64 — the reference's score of the lowest
  selected non-forced block (tie diagnostics);
* ``out_rows`` / ``out`` — outputs of every 32nd row plus the first/last rows
  and the block-boundary neighbours (the full 8192 x 32 x 128 float32 output
  would be 128 MiB);
* ``row_digest`` — sha256 of each 256-row chunk's float32 output, so a run of
  the reference elsewhere can be compared exactly;
* ``fine_sha`` / ``coarse_sha`` of the reference's kernel means.
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ["OPENBLAS_NUM_THREADS"] = "1"

from inputs import digest, make_qkv  # noqa: E402
from cases import B8  # noqa: E402

SEED, L = 1_000, 8192
_STATE = {}


def _init():
    from deskinfer.sparse import BlockizedLayerCache, SparseAttentionConfig
    cfg = SparseAttentionConfig(**B8)
    q, k, v = make_qkv(SEED, L, L, 32, 2, 128)
    layer = BlockizedLayerCache(2, 128, cfg)
    layer.append(k, v)
    _STATE.update(cfg=cfg, q=q, layer=layer)


def _rows(chunk):
    from deskinfer.sparse import two_stage_attention
    if not _STATE:
        _init()
    cfg, q, layer = _STATE["cfg"], _STATE["q"], _STATE["layer"]
    lo, hi = chunk
    smax = cfg.top_k + cfg.n_init_blocks + cfg.n_local_blocks
    sel = np.full((hi - lo, 2, smax), -1, np.int16)
    margin = np.full((hi - lo, 2), np.nan, np.float64)
    outs = np.zeros((hi - lo, 32, 128), np.float32)
    for r in range(lo, hi):
        traces = []
        o = two_stage_attention(q[r:r + 1], layer, cfg, r, traces=traces)
        outs[r - lo] = o[0]
        for t in traces:
            ids = t["selected"]
            sel[r - lo, t["group"], :len(ids)] = ids
            free = [s for b, s in zip(ids, t["scores_topk"]) if b not in t["forced"]]
            if free:
                margin[r - lo, t["group"]] = min(free)
    return lo, sel, margin, outs


def out_row_set() -> np.ndarray:
    picks = set(range(0, L, 32)) | {L - 1}
    for b in range(1, L // 64):
        for dlt in (-1, 0, 1):
            if b % 16 == 0:
                picks.add(b * 64 + dlt)
    return np.asarray(sorted(picks), dtype=np.int64)


def main() -> None:
    from deskinfer.sparse import BlockizedLayerCache, SparseAttentionConfig
    chunks = [(lo, min(lo + 256, L)) for lo in range(0, L, 256)]
    sel = np.full((L, 2, 19), -1, np.int16)
    margin = np.full((L, 2), np.nan, np.float64)
    keep = out_row_set()
    out = np.zeros((keep.size, 32, 128), np.float32)
    pos_of = {int(r): j for j, r in enumerate(keep)}
    digests = [""] * len(chunks)
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for lo, s, mg, o in ex.map(_rows, chunks):
            hi = lo + s.shape[0]
            sel[lo:hi] = s
            margin[lo:hi] = mg
            digests[lo // 256] = digest(o)
            for r in range(lo, hi):
                if r in pos_of:
                    out[pos_of[r]] = o[r - lo]
            print("rows", lo, hi, flush=True)
    cfg = SparseAttentionConfig(**B8)
    q, k, v = make_qkv(SEED, L, L, 32, 2, 128)
    layer = BlockizedLayerCache(2, 128, cfg)
    layer.append(k, v)
    meta = dict(seed=SEED, length=L, geometry=B8, hq=32, hkv=2, d=128, input_sha=digest(q, k, v),
                fine_sha=digest(layer.fine_means), coarse_sha=digest(layer.coarse_means))
    np.savez_compressed(os.path.join(HERE, "config0_8k_full.npz"),
                        meta=np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8),
                        selection=sel, margin_score=margin, out_rows=keep.astype(np.int32), out=out,
                        row_digest=np.array(digests))
    print("wrote config0_8k_full.npz")


if __name__ == "__main__":
    main()
