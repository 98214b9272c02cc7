"""Golden case table and input construction (no reference import; safe on the GPU box)."""

from __future__ import annotations

import numpy as np

from inputs import make_qkv, round_bf16

SMALL = dict(block_size=8, kernel_size=4, kernel_stride=2, coarse_stride=4,
             top_k=2, n_init_blocks=1, n_local_blocks=1)
B8 = dict(block_size=64, kernel_size=32, kernel_stride=16, coarse_stride=128,
          top_k=16, n_init_blocks=1, n_local_blocks=2)

# name: (geometry, seed, L, n_q, start, hq, hkv, d, rows, out_rows, scale, kind)
#   rows=None -> every query row; kind: "iid" | "uniform" | "needle"
CASES = {
    "small_prefill":      (SMALL, 1, 50, 50, 0, 4, 2, 4, None, None, 1.0, "iid"),
    "small_prefill_b":    (dict(SMALL, top_k=3, n_local_blocks=2), 2, 77, 77, 0, 4, 2, 4, None, None, 1.0, "iid"),
    "small_consume":      (dict(SMALL, top_k=3, n_local_blocks=2, forced_consume_budget=True), 3, 61, 61, 0, 4, 2, 4, None, None, 1.0, "iid"),
    "small_noforce":      (dict(SMALL, n_init_blocks=0, n_local_blocks=0, top_k=3), 4, 45, 45, 0, 4, 2, 8, None, None, 1.0, "iid"),
    "small_chunk":        (SMALL, 5, 64, 20, 44, 4, 2, 4, None, None, 1.0, "iid"),
    "small_uniform_ties": (SMALL, 6, 48, 48, 0, 4, 2, 4, None, None, 1.0, "uniform"),
    "small_stride_eq":    (dict(SMALL, kernel_size=2, kernel_stride=2, coarse_stride=2), 7, 40, 40, 0, 4, 1, 4, None, None, 1.0, "iid"),
    "small_g16":          (dict(SMALL, top_k=4), 8, 120, 120, 0, 32, 2, 16, None, None, 1.0, "iid"),
    "b8_2k_prefill":      (B8, 11, 2048, 2048, 0, 32, 2, 128, None, 48, 1.0, "iid"),
    "b8_1300_ragged":     (B8, 12, 1300, 1300, 0, 32, 2, 128, None, 32, 1.0, "iid"),
    "b8_8k_sampled":      (B8, 13, 8192, 8192, 0, 32, 2, 128, "sample96", 24, 1.0, "iid"),
    "b8_4k_decode":       (B8, 14, 4096, 1, 4095, 32, 2, 128, None, None, 1.0, "iid"),
    "b8_3k_chunk":        (B8, 15, 3000, 200, 2800, 32, 2, 128, None, 24, 1.0, "iid"),
    "b8_k8_default":      (dict(B8, top_k=8), 16, 2048, 2048, 0, 32, 2, 128, "sample96", 16, 1.0, "iid"),
    "b8_k64_dense":       (dict(B8, top_k=64), 17, 4096, 4096, 0, 32, 2, 128, "sample96", 16, 1.0, "iid"),
    "b8_consume":         (dict(B8, forced_consume_budget=True), 18, 2048, 2048, 0, 32, 2, 128, "sample96", 16, 1.0, "iid"),
    "b8_needle":          (B8, 19, 4096, 4096, 0, 32, 2, 128, "sample96", 16, 1.0, "needle"),
    "b8_uniform_ties":    (B8, 20, 2048, 2048, 0, 32, 2, 128, "sample96", 8, 1.0, "uniform"),
    "g8_d64_2k":          (B8, 21, 2048, 2048, 0, 16, 2, 64, "sample96", 16, 1.0, "iid"),
}


def sample_rows(n: int, start: int, seed: int, count: int = 96) -> np.ndarray:
    """Seeded rows plus the first/last rows and block-boundary neighbours."""
    rng = np.random.default_rng(seed + 99)
    picks = {0, n - 1, min(n - 1, 63), min(n - 1, 64), min(n - 1, 65)}
    for b in (1, 7, 31, n // 128):
        for delta in (-1, 0, 1):
            r = b * 64 + delta
            if 0 <= r < n:
                picks.add(r)
    while len(picks) < min(count, n):
        picks.add(int(rng.integers(0, n)))
    return np.asarray(sorted(picks), dtype=np.int64)


def build_inputs(seed, length, n_q, hq, hkv, d, scale, kind):
    q, k, v = make_qkv(seed, length, n_q, hq, hkv, d, scale)
    if kind == "uniform":
        k = np.ones_like(k)
    elif kind == "needle":
        rng = np.random.default_rng(seed + 7)
        direction = rng.standard_normal((hkv, d)).astype(np.float32)
        direction /= np.linalg.norm(direction, axis=1, keepdims=True)
        direction = round_bf16(4.0 * direction)
        nb = -(-length // 64)
        for blk in (nb // 3, (2 * nb) // 3):
            k[blk * 64:(blk + 1) * 64] = direction[None]
        g_size = hq // hkv
        for h in range(hq):
            q[:, h, :] = direction[h // g_size][None]
    return q, k, v
