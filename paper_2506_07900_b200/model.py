"""Model seam: the reference's ``forward(..., backend=...)`` and ``make_cache``
on the GPU, feeding post-RoPE q/k/v into the InfLLM v2 operator.

Restates ``deskinfer.model.forward`` (model.py:386-462) for any bundle with
the reference's layout (``bundle.config``: hidden_dim, n_layers, n_q_heads,
n_kv_heads, head_dim, vocab_size, max_seq_len, rope_base, ffn_dim,
tied_lm_head; ``bundle.params``: float32 arrays named as in
``param_shapes``; ``bundle.lm_head``), and ``specdec.make_cache``
(specdec.py:632-641).  Projections, RMSNorm, RoPE and the MLP run in float32
on the GPU (torch/cuBLAS, TF32 off); the cache appends happen BEFORE
attending (F4, model.py:434-444); q is rounded to bf16 on both backends (the
operator's input precision, the cache holds bf16 K/V); ``backend="sparse"`` calls
``two_stage_attention`` when a cache is given, otherwise the dense causal
GQA path (F16).  Returns a ``ForwardResult`` of CUDA tensors.
"""

from __future__ import annotations

import dataclasses
import weakref
from typing import Optional

import numpy as np
import torch

from .errors import NumericError, ValidationError
from .sparse import BlockizedLayerCache, KVCache, SparseAttentionConfig, blockized_cache, two_stage_attention


@dataclasses.dataclass
class ForwardResult:
    logits: torch.Tensor    # (n, vocab) float32
    hiddens: torch.Tensor   # (n, d) float32, last layer output before the final norm


_PARAMS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _device_params(bundle, device: torch.device) -> dict:
    """float32 copies of the bundle's tensors on `device`, cached per bundle."""
    try:
        cached = _PARAMS.get(bundle)
    except TypeError:            # bundle not weak-referenceable: no cache
        cached = None
    if cached is not None and cached["_device"] == device:
        return cached
    p = {name: torch.as_tensor(np.asarray(a, dtype=np.float32), device=device) for name, a in bundle.params.items()}
    p["_lm_head"] = torch.as_tensor(np.asarray(bundle.lm_head, dtype=np.float32), device=device)
    p["_device"] = device
    try:
        _PARAMS[bundle] = p
    except TypeError:
        pass
    return p


def rms_norm(x: torch.Tensor, weight: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """model.py:145-149: float64 statistics, result in x's dtype."""
    x64 = x.double()
    denom = torch.sqrt((x64 * x64).mean(dim=-1, keepdim=True) + eps)
    return ((x64 / denom) * weight.double()).to(x.dtype)


def rope_angles(cfg, positions: np.ndarray, device) -> tuple[torch.Tensor, torch.Tensor]:
    """model.py:152-159: float64 angles, float32 tables (n, head_dim)."""
    half = cfg.head_dim // 2
    inv_freq = cfg.rope_base ** (-np.arange(0, half, dtype=np.float64) / half)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    cos = np.concatenate([np.cos(ang), np.cos(ang)], axis=-1).astype(np.float32)
    sin = np.concatenate([np.sin(ang), np.sin(ang)], axis=-1).astype(np.float32)
    return torch.as_tensor(cos, device=device), torch.as_tensor(sin, device=device)


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """model.py:162-169 on (n, heads, head_dim)."""
    half = x.shape[-1] // 2
    rot = torch.cat([-x[..., half:], x[..., :half]], dim=-1)
    return x * cos[:, None, :] + rot * sin[:, None, :]


def dense_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, n_q_heads: int, n_kv_heads: int,
                    causal_offset: int = 0) -> torch.Tensor:
    """Causal GQA (model.py:229-253, 194-226): float32 dots, float64 softmax
    and weighted sum; q (n, HQ*D), k/v (m, HKV*D) -> (n, HQ*D) float32."""
    n, m = q.shape[0], k.shape[0]
    if causal_offset < 0 or causal_offset + n > m:
        raise ValidationError(f"causal_offset {causal_offset} with {n} queries exceeds {m} keys")
    if not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(k).all()) and bool(torch.isfinite(v).all())):
        raise NumericError("non-finite values in attention inputs")
    d = q.shape[1] // n_q_heads
    g = n_q_heads // n_kv_heads
    q3 = q.float().reshape(n, n_q_heads, d)
    k3 = k.float().reshape(m, n_kv_heads, d)
    v3 = v.double().reshape(m, n_kv_heads, d)
    allowed = torch.arange(m, device=q.device)[None, :] <= (causal_offset + torch.arange(n, device=q.device))[:, None]
    scale = float(np.float32(1.0 / np.sqrt(d)))
    out = torch.empty((n, n_q_heads, d), dtype=torch.float32, device=q.device)
    for h in range(n_q_heads):
        s = ((q3[:, h, :] @ k3[:, h // g, :].T) * scale).double()
        s = s.masked_fill(~allowed, float("-inf"))
        out[:, h, :] = (torch.softmax(s, dim=-1) @ v3[:, h // g, :]).float()
    return out.reshape(n, n_q_heads * d)


def masked_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, allowed: torch.Tensor, *,
                     n_q_heads: int, n_kv_heads: int) -> torch.Tensor:
    """GQA with an explicit (n, m) visibility mask (model.py:194-226): float32
    dots, float64 softmax and weighted sum; q (n, HQ*D), k/v (m, HKV*D)."""
    n, m = q.shape[0], k.shape[0]
    if not bool(allowed.any(dim=1).all()):
        raise ValidationError("every query must see at least one key")
    if not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(k).all()) and bool(torch.isfinite(v).all())):
        raise NumericError("non-finite values in attention inputs")
    d = q.shape[1] // n_q_heads
    g = n_q_heads // n_kv_heads
    q3 = q.float().reshape(n, n_q_heads, d)
    k3 = k.float().reshape(m, n_kv_heads, d)
    v3 = v.double().reshape(m, n_kv_heads, d)
    scale = float(np.float32(1.0 / np.sqrt(d)))
    out = torch.empty((n, n_q_heads, d), dtype=torch.float32, device=q.device)
    for h in range(n_q_heads):
        s = ((q3[:, h, :] @ k3[:, h // g, :].T) * scale).double()
        s = s.masked_fill(~allowed, float("-inf"))
        out[:, h, :] = (torch.softmax(s, dim=-1) @ v3[:, h // g, :]).float()
    return out.reshape(n, n_q_heads * d)


def forward_tree(bundle, cache: KVCache, tokens, depths, mask, *, backend: str = "dense",
                 sparse_config: Optional[SparseAttentionConfig] = None) -> ForwardResult:
    """Score every node of a draft tree in one pass without touching the cache
    (specdec.py:565-625): node i at position ``cache.length + depths[i] - 1``
    sees every cached row plus its ancestor-or-self tree rows (``mask``, a
    ``tree.PackedMask``).  ``backend="sparse"`` attends the prefix through the
    two-stage operator (``tree.tree_attention``).  Like
    ``forward``, q and the node K/V enter attention in bf16 (the cache dtype)."""
    from .tree import tree_attention

    cfg = bundle.config
    toks = np.asarray(tokens, dtype=np.int64).reshape(-1)
    dep = np.asarray(depths, dtype=np.int64).reshape(-1)
    n = toks.size
    if n == 0:
        raise ValidationError("empty tree batch")
    if dep.shape != (n,) or mask.n_nodes != n:
        raise ValidationError("tokens, depths, and mask disagree on node count")
    if toks.min() < 0 or toks.max() >= cfg.vocab_size:
        raise ValidationError("token id out of range")
    if backend not in ("dense", "sparse"):
        raise ValidationError(f"unknown attention backend {backend!r}")
    base = cache.length
    if base == 0:
        raise ValidationError("tree scoring needs a non-empty prefix cache")
    if backend == "sparse" and sparse_config is None:
        sparse_config = SparseAttentionConfig()
    dev = cache.layers[0].device
    p = _device_params(bundle, dev)
    cos, sin = rope_angles(cfg, base + dep - 1, dev)
    vis = torch.as_tensor(mask.to_dense(), device=dev)
    allowed = torch.cat([torch.ones((n, base), dtype=torch.bool, device=dev), vis], dim=1)
    x = p["embedding"][torch.as_tensor(toks, device=dev)]
    for i in range(cfg.n_layers):
        lp = f"layers.{i}."
        h = rms_norm(x, p[lp + "attn_norm.weight"])
        q = (h @ p[lp + "attn.wq"]).reshape(n, cfg.n_q_heads, cfg.head_dim)
        k = (h @ p[lp + "attn.wk"]).reshape(n, cfg.n_kv_heads, cfg.head_dim)
        v = (h @ p[lp + "attn.wv"]).reshape(n, cfg.n_kv_heads, cfg.head_dim)
        q = apply_rope(q, cos, sin).to(torch.bfloat16).float()
        k = apply_rope(k, cos, sin).to(torch.bfloat16).float()
        v = v.to(torch.bfloat16).float()
        layer = cache.layers[i]
        if backend == "sparse":
            attn = tree_attention(q, layer, sparse_config, k, v, mask).reshape(n, -1)
        else:
            keys = torch.cat([layer.keys.float(), k]).reshape(base + n, -1)
            values = torch.cat([layer.values.float(), v]).reshape(base + n, -1)
            attn = masked_attention(q.reshape(n, -1), keys, values, allowed, n_q_heads=cfg.n_q_heads,
                                    n_kv_heads=cfg.n_kv_heads)
        x = x + attn @ p[lp + "attn.wo"]
        h = rms_norm(x, p[lp + "mlp_norm.weight"])
        x = x + (_silu(h @ p[lp + "mlp.w_gate"]) * (h @ p[lp + "mlp.w_up"])) @ p[lp + "mlp.w_down"]
    logits = rms_norm(x, p["final_norm.weight"]) @ p["_lm_head"].T
    return ForwardResult(logits=logits, hiddens=x)


def _silu(x: torch.Tensor) -> torch.Tensor:
    return x / (1.0 + torch.exp(-x))


def make_cache(bundle, backend: str = "dense", sparse_config: Optional[SparseAttentionConfig] = None, *,
               capacity: int = 0, device=None) -> KVCache:
    """specdec.py:632-641: a cache of GPU layer caches.  Both backends use
    BlockizedLayerCache layers (the dense path simply ignores the means)."""
    if backend not in ("dense", "sparse"):
        raise ValidationError(f"unknown attention backend {backend!r}")
    return blockized_cache(bundle.config, sparse_config or SparseAttentionConfig(), capacity=capacity,
                           device=device)


def forward(bundle, tokens, cache: Optional[KVCache] = None, *, backend: str = "dense",
            sparse_config: Optional[SparseAttentionConfig] = None, device=None) -> ForwardResult:
    """Run ``tokens`` through the model, appending to ``cache`` if given (model.py:386-462)."""
    cfg = bundle.config
    toks = np.asarray(tokens, dtype=np.int64).reshape(-1)
    if toks.size == 0:
        raise ValidationError("empty token sequence")
    if toks.min() < 0 or toks.max() >= cfg.vocab_size:
        raise ValidationError("token id out of range")
    start = cache.length if cache is not None else 0
    n = toks.size
    if start + n > cfg.max_seq_len:
        raise ValidationError(f"sequence length {start + n} exceeds max_seq_len {cfg.max_seq_len}")
    if backend not in ("dense", "sparse"):
        raise ValidationError(f"unknown attention backend {backend!r}")
    if backend == "sparse" and sparse_config is None:
        sparse_config = SparseAttentionConfig()
    if cache is not None and cache.layers:
        dev = cache.layers[0].device
    else:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    p = _device_params(bundle, dev)
    cos, sin = rope_angles(cfg, np.arange(start, start + n), dev)
    x = p["embedding"][torch.as_tensor(toks, device=dev)]
    for i in range(cfg.n_layers):
        lp = f"layers.{i}."
        h = rms_norm(x, p[lp + "attn_norm.weight"])
        q = (h @ p[lp + "attn.wq"]).reshape(n, cfg.n_q_heads, cfg.head_dim)
        k = (h @ p[lp + "attn.wk"]).reshape(n, cfg.n_kv_heads, cfg.head_dim)
        v = (h @ p[lp + "attn.wv"]).reshape(n, cfg.n_kv_heads, cfg.head_dim)
        # q enters attention in bf16 on both backends (the operator's input
        # precision), so the dense and sparse paths see identical inputs
        q = apply_rope(q, cos, sin).to(torch.bfloat16).float()
        k = apply_rope(k, cos, sin)
        if cache is not None:
            layer = cache.layers[i]
            layer.append(k, v)                       # append BEFORE attending (F4)
            keys, values = layer.keys, layer.values
        else:
            layer = None
            keys, values = k, v
        if backend == "sparse" and layer is not None:
            attn = two_stage_attention(q, layer, sparse_config, start, out_dtype=torch.float32)
            attn = attn.reshape(n, cfg.n_q_heads * cfg.head_dim)
        else:
            attn = dense_attention(q.reshape(n, -1), keys.reshape(keys.shape[0], -1),
                                   values.reshape(values.shape[0], -1), n_q_heads=cfg.n_q_heads,
                                   n_kv_heads=cfg.n_kv_heads, causal_offset=start if cache is not None else 0)
        x = x + attn @ p[lp + "attn.wo"]
        h = rms_norm(x, p[lp + "mlp_norm.weight"])
        x = x + (_silu(h @ p[lp + "mlp.w_gate"]) * (h @ p[lp + "mlp.w_up"])) @ p[lp + "mlp.w_down"]
    logits = rms_norm(x, p["final_norm.weight"]) @ p["_lm_head"].T
    return ForwardResult(logits=logits, hiddens=x)
