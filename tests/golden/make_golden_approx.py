"""Golden fixtures for the opt-in approx-LSE selection mode.

Usage (build container only; /root/reference must exist):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_approx.py

The reference has no driver for this mode, so each row is composed from the
UNMODIFIED reference's own functions (imported read-only from
``/root/reference/pkg/src``): the cache and its fine/coarse means
(``BlockizedLayerCache``), ``approx_lse`` (sparse.py:292-312) for the
normaliser, ``group_scores`` / ``block_scores`` / ``force_blocks`` /
``select_topk`` / ``sparse_attend`` (sparse.py:183-384) for the rest.  The only
line that is not a reference call is the mode's definition itself (DESIGN.md §4
K2p): head h's weights are exp(z_hj - approx_lse(q_h, coarse[:nc_t])) with
nc_t = min(t // s_c + 1, L // s_c), and the exact ``kernel_scores`` when the
cache holds no coarse kernel.

Writes ``approx_<case>.npz`` with the selection of every stored row (-1 padded)
and the outputs of up to 24 of them; inputs come from ``tests/golden/inputs.py`` (sha256 recorded).
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

from inputs import digest  # noqa: E402
from cases import B8, SMALL, build_inputs, sample_rows  # noqa: E402

# name: (geometry, seed, L, n_q, start, hq, hkv, d, rows)
APPROX_CASES = {
    "approx_small":    (SMALL, 31, 50, 50, 0, 4, 2, 4, None),
    "approx_small_g16": (dict(SMALL, top_k=4), 32, 120, 120, 0, 32, 2, 16, None),
    "approx_b8_short": (B8, 33, 100, 100, 0, 32, 2, 128, None),            # L < s_c: exact fallback
    "approx_b8_2k":    (B8, 34, 2048, 2048, 0, 32, 2, 128, "sample96"),
    "approx_b8_4k_k64": (dict(B8, top_k=64), 35, 4096, 4096, 0, 32, 2, 128, "sample96"),
    "approx_b8_chunk": (B8, 36, 3000, 200, 2800, 32, 2, 128, None),
    "approx_g8_d64":   (B8, 37, 2048, 2048, 0, 16, 2, 64, "sample96"),
}


def run(name):
    from deskinfer.sparse import (BlockizedLayerCache, SparseAttentionConfig, approx_lse, block_scores,
                                  force_blocks, group_scores, kernel_scores, select_topk, sparse_attend)

    geom, seed, length, n_q, start, hq, hkv, d, rows = APPROX_CASES[name]
    cfg = SparseAttentionConfig(**geom)
    q, k, v = build_inputs(seed, length, n_q, hq, hkv, d, 1.0, "iid")
    layer = BlockizedLayerCache(hkv, d, cfg)
    layer.append(k, v)
    fine, coarse = layer.fine_means, layer.coarse_means
    keys, values = layer.keys, layer.values
    gsz = hq // hkv
    row_ids = np.arange(n_q) if rows is None else sample_rows(n_q, start, seed)
    smax = cfg.top_k + cfg.n_init_blocks + cfg.n_local_blocks
    sel = np.full((row_ids.size, hkv, smax), -1, np.int32)
    out = np.zeros((row_ids.size, hq, d), np.float32)
    scale = 1.0 / np.sqrt(d)
    for j, r in enumerate(row_ids):
        pos = start + int(r)
        n_cand = pos // cfg.block_size + 1
        blocks = [(b * cfg.block_size, min((b + 1) * cfg.block_size, pos + 1)) for b in range(n_cand)]
        n_kernels = min(pos // cfg.kernel_stride + 1, fine.shape[0])
        nc_t = min(pos // cfg.coarse_stride + 1, coarse.shape[0])
        forced = force_blocks(n_cand, pos // cfg.block_size, cfg.n_init_blocks, cfg.n_local_blocks)
        for g in range(hkv):
            qh = q[r, g * gsz:(g + 1) * gsz, :]
            if n_kernels > 0:
                mu = fine[:n_kernels, g, :]
                if nc_t > 0:
                    per_head = np.stack([
                        np.exp((mu @ qh[h]) * scale
                               - approx_lse(qh[h], coarse[:nc_t, g, :], cfg.kernel_stride, cfg.coarse_stride))
                        for h in range(gsz)])
                else:
                    per_head = np.stack([kernel_scores(qh[h], mu) for h in range(gsz)])
                bs = block_scores(group_scores(per_head), blocks, cfg.kernel_size, cfg.kernel_stride)
            else:
                bs = np.zeros(n_cand, np.float64)
            chosen = select_topk(bs, cfg.top_k, forced, forced_consume_budget=cfg.forced_consume_budget)
            sel[j, g, :chosen.size] = chosen
            o, _ = sparse_attend(qh, keys, values, chosen, blocks, pos, g, gsz)
            out[j, g * gsz:(g + 1) * gsz] = o
    meta = dict(name=name, geometry=geom, seed=seed, length=length, n_q=n_q, start=start, hq=hq, hkv=hkv, d=d,
                scale=1.0, kind="iid", input_sha=digest(q, k, v), fine_sha=digest(fine),
                coarse_sha=digest(coarse))
    keep = np.unique(np.linspace(0, row_ids.size - 1, min(24, row_ids.size)).round().astype(np.int64))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        meta=np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8),
                        rows=row_ids.astype(np.int32), selection=sel,
                        out_rows=row_ids[keep].astype(np.int32), out=out[keep])
    return name, row_ids.size


if __name__ == "__main__":
    names = sys.argv[1:] or list(APPROX_CASES)
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for res in ex.map(run, names):
            print(*res, flush=True)
