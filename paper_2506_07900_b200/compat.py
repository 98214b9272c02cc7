"""Reference-signature adapter: NumPy in, NumPy out.

`deskinfer.sparse.two_stage_attention(q, layer, config, start_position, *,
stats=None, traces=None)` (sparse.py:387-395) takes float32 numpy arrays and the
reference's own `BlockizedLayerCache`.  `two_stage_attention_numpy` has exactly
that signature and semantics, runs the GPU path, and returns a float32 numpy
array, so a maintainer can route the reference's `model.forward`
(model.py:442-444) to the B200 kernels with one assignment.

The reference cache's keys/values are uploaded once per (layer object, length)
and appended incrementally afterwards; they are stored as bf16 on the GPU, so
results equal the reference's exactly only for bf16-representable inputs (the
parity fixtures are bf16-exact by construction).
"""

from __future__ import annotations

import weakref

import numpy as np
import torch

from . import sparse as _gpu

_MIRRORS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _config(cfg) -> _gpu.SparseAttentionConfig:
    if isinstance(cfg, _gpu.SparseAttentionConfig):
        return cfg
    return _gpu.SparseAttentionConfig(
        block_size=cfg.block_size, kernel_size=cfg.kernel_size, kernel_stride=cfg.kernel_stride,
        coarse_stride=cfg.coarse_stride, top_k=cfg.top_k, n_init_blocks=cfg.n_init_blocks,
        n_local_blocks=cfg.n_local_blocks, forced_consume_budget=bool(cfg.forced_consume_budget))


def mirror_cache(layer, config, device="cuda") -> _gpu.BlockizedLayerCache:
    """GPU mirror of a reference LayerCache, kept in sync by length."""
    cfg = _config(config)
    entry = _MIRRORS.get(layer)
    if entry is None or entry.config != cfg or entry.length > layer.length:
        entry = _gpu.BlockizedLayerCache(layer.n_kv_heads, layer.head_dim, cfg,
                                         capacity=max(layer.length, 64), device=device)
        _MIRRORS[layer] = entry
    if entry.length < layer.length:
        k = torch.from_numpy(np.ascontiguousarray(layer.keys[entry.length:], dtype=np.float32))
        v = torch.from_numpy(np.ascontiguousarray(layer.values[entry.length:], dtype=np.float32))
        entry.append(k.to(entry.device), v.to(entry.device))
    return entry


def two_stage_attention_numpy(q, layer, config, start_position, *, stats=None, traces=None) -> np.ndarray:
    """Drop-in for deskinfer.sparse.two_stage_attention (sparse.py:387-468)."""
    cache = mirror_cache(layer, config)
    qt = torch.from_numpy(np.ascontiguousarray(q, dtype=np.float32)).to(cache.device)
    out = _gpu.two_stage_attention(qt, cache, _config(config), int(start_position), stats=stats,
                                   traces=traces, out_dtype=torch.float32)
    return out.cpu().numpy()
