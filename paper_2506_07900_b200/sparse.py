"""Drop-in GPU mirror of the reference's sparse-attention surface.

Same names, argument meaning and exception types as
``/root/reference/pkg/src/deskinfer/sparse.py`` (cited as ``sparse.py``), but
tensors are CUDA ``torch.Tensor``s and all numeric work runs in
``libinfllm2.so`` (hand-written sm_100a CUDA, see ``csrc/``):

* ``SparseAttentionConfig``            sparse.py:31-51
* ``BlockizedLayerCache``              sparse.py:94-144 (+ LayerCache model.py:298-352)
* ``blockized_cache`` / ``KVCache``    sparse.py:147-156, model.py:355-369
* ``build_kernels``                    sparse.py:76-91
* ``two_stage_attention``              sparse.py:387-468
* host integer helpers ``partition_blocks`` / ``kernel_range_for_block`` /
  ``force_blocks`` / ``TouchStats``    sparse.py:58-67,191-198,218-227,319-344

PyTorch is used for device memory and streams only; the product path never
falls back to a CPU or PyTorch computation.
"""

from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import NumericError, ValidationError

__all__ = [
    "SparseAttentionConfig", "BlockizedLayerCache", "KVCache", "blockized_cache", "build_kernels",
    "two_stage_attention", "partition_blocks", "kernel_range_for_block", "force_blocks",
    "TouchStats", "ValidationError", "NumericError",
]


# --------------------------------------------------------------------------
# configuration (sparse.py:31-51)


@dataclasses.dataclass
class SparseAttentionConfig:
    block_size: int = 64        # m: tokens per KV block
    kernel_size: int = 32       # p: keys averaged into one kernel
    kernel_stride: int = 16     # s: distance between kernel starts
    coarse_stride: int = 128    # s_c: stride of the coarse LSE kernels
    top_k: int = 8              # k: scored blocks kept per query/group
    n_init_blocks: int = 1      # always-attended leading blocks
    n_local_blocks: int = 2     # always-attended trailing blocks (incl. own)
    forced_consume_budget: bool = False  # forced blocks count against top_k

    def __post_init__(self) -> None:
        if min(self.block_size, self.kernel_size, self.kernel_stride,
               self.coarse_stride, self.top_k) <= 0:
            raise ValidationError("block/kernel/stride/top_k sizes must be positive")
        if self.kernel_stride > self.kernel_size:
            raise ValidationError("kernel_stride must not exceed kernel_size")
        if self.coarse_stride < self.kernel_stride or self.coarse_stride % self.kernel_stride:
            raise ValidationError("coarse_stride must be a multiple of kernel_stride")
        if self.n_init_blocks < 0 or self.n_local_blocks < 0:
            raise ValidationError("forced block counts must be non-negative")

    def geometry(self) -> _lib.Geometry:
        return _lib.Geometry(self.block_size, self.kernel_size, self.kernel_stride,
                             self.coarse_stride, self.top_k, self.n_init_blocks,
                             self.n_local_blocks, int(bool(self.forced_consume_budget)))

    @property
    def max_selected(self) -> int:
        return self.top_k + self.n_init_blocks + self.n_local_blocks


# --------------------------------------------------------------------------
# host-side integer helpers (no numeric work)


def partition_blocks(length: int, block_size: int) -> list[tuple[int, int]]:
    """Blocks ``(j*m, min((j+1)*m, L))`` (sparse.py:58-67)."""
    if block_size <= 0:
        raise ValidationError("block_size must be positive")
    if length < 0:
        raise ValidationError("length must be non-negative")
    return [(s, min(s + block_size, length)) for s in range(0, length, block_size)]


def kernel_range_for_block(block: tuple[int, int], kernel_size: int, stride: int,
                           n_kernels: int) -> tuple[int, int]:
    """Kernel index range intersecting ``block`` (sparse.py:191-198)."""
    start, end = block
    lo = 0 if start < kernel_size else (start - kernel_size) // stride + 1
    hi = min(n_kernels, -(-end // stride))
    return min(lo, n_kernels), hi


def force_blocks(n_blocks: int, query_block: int, n_init: int, n_local: int) -> np.ndarray:
    """Leading and local-window block ids (sparse.py:218-227)."""
    if not 0 <= query_block < max(n_blocks, 1):
        raise ValidationError(f"query block {query_block} outside 0..{n_blocks - 1}")
    forced = set(range(min(n_init, n_blocks)))
    if n_local > 0:
        forced.update(range(max(0, query_block - n_local + 1), query_block + 1))
    return np.asarray(sorted(forced), dtype=np.int64)


@dataclasses.dataclass
class TouchStats:
    """Row-touch counters per (query, group) (sparse.py:319-344)."""

    stage1: int = 0
    stage2: int = 0
    dense_rows: int = 0
    samples: int = 0

    def add(self, stage1: int, stage2: int, dense_rows: int) -> None:
        self.stage1 += stage1
        self.stage2 += stage2
        self.dense_rows += dense_rows
        self.samples += 1

    @property
    def sparse_rows(self) -> int:
        return self.stage1 + self.stage2

    @property
    def ratio(self) -> float:
        return self.sparse_rows / self.dense_rows if self.dense_rows else 0.0


# --------------------------------------------------------------------------
# device plumbing


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


_WS: dict = {}
_WS_PER_DEVICE = 4          # scratch buffers kept per device (most recently used streams)
_WS_CAPTURED: list = []     # buffers a captured CUDA graph may reference: never released


def _workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    """Scratch reused across calls, one buffer per (device, stream): calls on
    different streams never share scratch.  A buffer used while a CUDA graph is
    being captured is kept alive for the life of the process (the graph holds
    its address), so growing the cache later cannot hand that memory to
    anything else."""
    stream = torch.cuda.current_stream(device)
    key = (device.type, device.index, stream.cuda_stream)
    ws = _WS.get(key)
    capturing = torch.cuda.is_current_stream_capturing()
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = ws
    else:
        _WS.pop(key)
        _WS[key] = ws            # most recently used last
    # bound the cache when callers churn through streams: a dropped buffer was
    # allocated on (and is only reused by) its own stream, so freeing is ordered
    same_dev = [k for k in _WS if k[:2] == key[:2]]
    for k in same_dev[:-_WS_PER_DEVICE]:
        del _WS[k]
    if capturing and not any(w is ws for w in _WS_CAPTURED):
        _WS_CAPTURED.append(ws)
    return ws


def _as_device_rows(x, n_kv_heads: int, head_dim: int, device: torch.device, what: str) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x))
    if x.dim() != 3 or x.shape[1] != n_kv_heads or x.shape[2] != head_dim:
        raise ValidationError(f"{what} shape {tuple(x.shape)} != (n, {n_kv_heads}, {head_dim})")
    if x.dtype not in (torch.bfloat16, torch.float32):
        x = x.to(torch.float32)
    return x.to(device).contiguous()


# --------------------------------------------------------------------------
# the blockized cache (sparse.py:94-144, model.py:298-352)


class BlockizedLayerCache:
    """Per-layer K/V cache on the GPU with kernel means kept in sync.

    Storage is head-major bf16 ``[HKV][cap][D]`` (one KV group's 64-row block
    is one contiguous 16 KB run); fine means are float32 ``[HKV][cap/s][D]``
    plus a bf16 hi/lo split for the tensor-core scorer; coarse means float32.
    Capacity grows by doubling like ``LayerCache.append`` (model.py:324-331);
    pass ``capacity`` to preallocate.  Appends/truncates recompute only the
    windows whose rows changed (sparse.py:111-133) and are bitwise equal to a
    rebuild.
    """

    def __init__(self, n_kv_heads: int, head_dim: int, config: SparseAttentionConfig, *,
                 capacity: int = 0, device=None):
        self.n_kv_heads = int(n_kv_heads)
        self.head_dim = int(head_dim)
        self.config = config
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.length = 0
        self._cap = 0
        self._nk_valid = 0
        self._nc_valid = 0
        self._nc_split = 0      # coarse rows whose bf16 hi/lo split is current (decode steps write f32 only)
        self._k = self._v = None
        self._fine = self._fine_hi = self._fine_lo = self._coarse = None
        self._coarse_hi = self._coarse_lo = None
        _lib.load()
        self._reserve(max(int(capacity), 0))

    # -- storage
    def _means_cap(self, stride: int) -> int:
        return self._cap // stride + 1

    def _reserve(self, need: int) -> None:
        if need <= self._cap and self._k is not None:
            return
        cap = max(need, 2 * self._cap, 64)
        h, d, dev = self.n_kv_heads, self.head_dim, self.device
        s, sc = self.config.kernel_stride, self.config.coarse_stride
        # zero-filled: rows past the length are read (P = 0) by the decode
        # stage-2 tiles, so they must be finite
        k = torch.zeros((h, cap, d), dtype=torch.bfloat16, device=dev)
        v = torch.zeros_like(k)
        fine = torch.empty((h, cap // s + 1, d), dtype=torch.float32, device=dev)
        hi = torch.empty((h, cap // s + 1, d), dtype=torch.bfloat16, device=dev)
        lo = torch.empty_like(hi)
        coarse = torch.empty((h, cap // sc + 1, d), dtype=torch.float32, device=dev)
        chi = torch.empty((h, cap // sc + 1, d), dtype=torch.bfloat16, device=dev)   # approx-LSE mode
        clo = torch.empty_like(chi)
        if self._k is not None and self.length:
            k[:, :self.length].copy_(self._k[:, :self.length])
            v[:, :self.length].copy_(self._v[:, :self.length])
            fine[:, :self._nk_valid].copy_(self._fine[:, :self._nk_valid])
            hi[:, :self._nk_valid].copy_(self._fine_hi[:, :self._nk_valid])
            lo[:, :self._nk_valid].copy_(self._fine_lo[:, :self._nk_valid])
            coarse[:, :self._nc_valid].copy_(self._coarse[:, :self._nc_valid])
            chi[:, :self._nc_valid].copy_(self._coarse_hi[:, :self._nc_valid])
            clo[:, :self._nc_valid].copy_(self._coarse_lo[:, :self._nc_valid])
        self._k, self._v = k, v
        self._fine, self._fine_hi, self._fine_lo, self._coarse = fine, hi, lo, coarse
        self._coarse_hi, self._coarse_lo = chi, clo
        self._cap = cap

    @property
    def capacity(self) -> int:
        return self._cap

    @property
    def keys(self) -> torch.Tensor:
        """(length, HKV, D) bf16 view."""
        return self._k[:, :self.length].transpose(0, 1)

    @property
    def values(self) -> torch.Tensor:
        return self._v[:, :self.length].transpose(0, 1)

    @property
    def fine_means(self) -> torch.Tensor:
        """(length // s, HKV, D) float32 view."""
        return self._fine[:, :self._nk_valid].transpose(0, 1)

    @property
    def coarse_means(self) -> torch.Tensor:
        return self._coarse[:, :self._nc_valid].transpose(0, 1)

    @property
    def n_blocks(self) -> int:
        return -(-self.length // self.config.block_size)

    # -- mutation (model.py:322-346)
    def append(self, k, v) -> None:
        k = _as_device_rows(k, self.n_kv_heads, self.head_dim, self.device, "k")
        v = _as_device_rows(v, self.n_kv_heads, self.head_dim, self.device, "v")
        if k.shape != v.shape:
            raise ValidationError("k/v shape mismatch")
        if k.dtype != v.dtype:
            v = v.to(k.dtype)
        n = k.shape[0]
        if n == 0:
            return
        self._reserve(self.length + n)
        # one streaming pass: the new rows enter the cache and the dirty fine and
        # coarse windows are recomputed from the same staged rows
        self._sync(self.length, self.length + n, k, v)

    def truncate(self, new_length: int) -> None:
        if not 0 <= new_length <= self.length:
            raise ValidationError(f"cannot truncate cache of length {self.length} to {new_length}")
        old = self.length
        self.length = int(new_length)
        if self.length != old:
            self.notify_truncate(old)

    def notify_append(self, old_length: int) -> None:
        """Re-sync after rows [old_length, length) were written externally."""
        self._sync(old_length, self.length)

    def notify_truncate(self, old_length: int) -> None:
        self._sync(old_length, self.length)

    def _sync(self, l_old: int, l_new: int, k_new=None, v_new=None) -> None:
        """infllm2_append_compress: append k_new/v_new (if given) at l_old and
        recompute the dirty fine + coarse windows (sparse.py:111-133)."""
        lib = _lib.load()
        cfg = self.config
        st = _stream(self.device)
        split_full = self._nc_split >= self._nc_valid
        n_new = 0 if k_new is None else k_new.shape[0]
        f32 = 1 if (k_new is not None and k_new.dtype == torch.float32) else 0
        _lib.check(lib.infllm2_append_compress(
            _ptr(self._k), _ptr(self._v), self._cap, self.n_kv_heads, self.head_dim, _ptr(k_new), _ptr(v_new),
            n_new, self.n_kv_heads * self.head_dim, f32, l_old, l_new, self._nk_valid, self._nc_valid,
            cfg.kernel_size, cfg.kernel_stride, cfg.coarse_stride, _ptr(self._fine), _ptr(self._fine_hi),
            _ptr(self._fine_lo), self._fine.shape[1], _ptr(self._coarse), _ptr(self._coarse_hi),
            _ptr(self._coarse_lo), self._coarse.shape[1], st), "append/compress")
        self.length = l_new
        self._nk_valid = l_new // cfg.kernel_stride
        self._nc_valid = l_new // cfg.coarse_stride
        self._nc_split = self._nc_valid if split_full else min(self._nc_split, self._nc_valid)

    def _coarse_split(self) -> None:
        """Bring the coarse means' bf16 hi/lo split (approx-LSE mode) up to date
        after batched decode steps, which maintain the float32 means only."""
        a, b = self._nc_split, self._nc_valid
        if a < b:
            c = self._coarse[:, a:b]
            hi = c.to(torch.bfloat16)
            self._coarse_hi[:, a:b].copy_(hi)
            self._coarse_lo[:, a:b].copy_((c - hi.float()).to(torch.bfloat16))
        self._nc_split = b

    def rebuild_kernels(self) -> tuple[torch.Tensor, torch.Tensor]:
        """From-scratch (fine, coarse) means, (count, HKV, D) float32 (sparse.py:135-140)."""
        return (build_kernels(self.keys, self.config.kernel_size, self.config.kernel_stride),
                build_kernels(self.keys, self.config.kernel_size, self.config.coarse_stride))

    # raw device views for the kernels
    def _device_args(self):
        return (self._k, self._v, self._cap, self._fine, self._fine_hi, self._fine_lo, self._fine.shape[1])


class KVCache:
    """One BlockizedLayerCache per layer (model.py:355-369, sparse.py:147-156)."""

    def __init__(self, n_layers: int, layer_factory):
        self.layers = [layer_factory() for _ in range(n_layers)]

    @property
    def length(self) -> int:
        return self.layers[0].length if self.layers else 0

    def truncate(self, new_length: int) -> None:
        for layer in self.layers:
            layer.truncate(new_length)


def blockized_cache(model_config, sparse_config: SparseAttentionConfig, *, capacity: int = 0,
                    device=None) -> KVCache:
    """A KVCache of BlockizedLayerCache layers (sparse.py:147-156)."""
    return KVCache(model_config.n_layers, lambda: BlockizedLayerCache(
        model_config.n_kv_heads, model_config.head_dim, sparse_config, capacity=capacity, device=device))


def build_kernels(keys: torch.Tensor, kernel_size: int, stride: int) -> torch.Tensor:
    """Mean-pool overlapping key windows on the GPU (sparse.py:76-91).

    ``keys`` (L, HKV, D) CUDA tensor (bf16 or float32; float32 is rounded to
    bf16, the cache dtype).  Returns (L // stride, HKV, D) float32.
    """
    if kernel_size <= 0 or stride <= 0:
        raise ValidationError("kernel_size and stride must be positive")
    if keys.dim() != 3:
        raise ValidationError("keys must be (L, HKV, D)")
    length, h, d = keys.shape
    dev = keys.device
    kc = keys.to(torch.bfloat16).transpose(0, 1).contiguous()   # [HKV][L][D]
    count = length // stride
    out = torch.empty((h, count + 1, d), dtype=torch.float32, device=dev)
    lib = _lib.load()
    _lib.check(lib.infllm2_compress(_ptr(kc), max(length, 1), h, d, 0, length, 0, kernel_size, stride,
                                    _ptr(out), None, None, count + 1, _stream(dev)), "build_kernels")
    return out[:, :count].transpose(0, 1)


# --------------------------------------------------------------------------
# the operator (sparse.py:387-468)


def two_stage_attention(q: torch.Tensor, layer: BlockizedLayerCache, config: SparseAttentionConfig,
                        start_position: int, *, stats: Optional[TouchStats] = None,
                        traces: Optional[list] = None, return_selection: bool = False,
                        return_lse: bool = False, out_dtype: Optional[torch.dtype] = None,
                        exact: bool = False, split_p: bool = False, check_finite: bool = False,
                        lse: str = "exact"):
    """Block-sparse attention for ``q`` of shape (n, n_q_heads, head_dim).

    Same semantics as the reference (sparse.py:387-468): row i sits at
    absolute position ``start_position + i``; selection is per (row, KV
    group); forced init/local blocks plus the top-k scored blocks are attended.
    Returns ``out`` (n, HQ, D) in ``out_dtype`` (default: q's dtype), plus the
    int32 selection (n, HKV, max_selected; ascending, -1 padded) and/or the
    float32 LSE (n, HQ) when requested.  ``exact=True`` forces the float64
    CUDA-core scorer (the verifier) instead of the tensor-core one.
    ``check_finite=True`` reproduces the reference's ``NumericError`` for
    non-finite queries or kernel means (sparse.py:176-177); it costs a device
    synchronisation, so it is opt-in.
    ``split_p=True`` makes the tensor-core stage 2 carry the softmax weights as
    bf16 hi + lo (outputs ~1e-5 of the float64 reference instead of ~1e-4, at
    ~1.3x the stage-2 cost); the default uses bf16 weights.
    ``lse="approx"`` is the opt-in approx-LSE selection mode (SURVEY §8f rank 4,
    the paper's LSE-approximated stage 1): each head's kernel weights are
    normalised by ``approx_lse`` over the coarse kernels (sparse.py:292-312)
    instead of the exact softmax, which skips 7/8 of stage 1's first pass but
    changes ~1/3 of the selections; the reference has no such
    driver, so its default ``"exact"`` is what matches the reference.
    """
    if lse not in ("exact", "approx"):
        raise ValidationError(f"unknown lse mode {lse!r}")
    if not isinstance(q, torch.Tensor) or q.dim() != 3:
        raise ValidationError("q must be a (n, n_q_heads, head_dim) tensor")
    n, hq, d = q.shape
    hkv = layer.n_kv_heads
    if hkv and hq % hkv:
        raise ValidationError("query heads not divisible by KV heads")
    if d != layer.head_dim:
        raise ValidationError(f"head_dim {d} != cache head_dim {layer.head_dim}")
    start = int(start_position)
    if n and start + n - 1 >= layer.length:
        raise ValidationError(f"query position {start + n - 1} beyond cache length {layer.length}")
    dev = layer.device
    out_dtype = out_dtype or (q.dtype if q.dtype in (torch.float32, torch.bfloat16) else torch.bfloat16)
    if check_finite and n:
        if not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(layer.fine_means).all())):
            raise NumericError("non-finite values in kernel scoring")
    qb = q.to(device=dev, dtype=torch.bfloat16)
    if qb.stride(2) != 1 or qb.stride(1) != d:
        qb = qb.contiguous()
    geom = config.geometry()
    smax = config.max_selected
    sel = torch.empty((n, hkv, smax), dtype=torch.int32, device=dev)
    out = torch.empty((n, hq, d), dtype=out_dtype, device=dev)
    lse_out = torch.empty((n, hq), dtype=torch.float32, device=dev) if return_lse else None
    sel_scores = torch.empty((n, hkv, smax), dtype=torch.float64, device=dev) if traces is not None else None
    flags = ((_lib.FLAG_EXACT_SIMT if exact else 0) | (_lib.FLAG_OUT_F32 if out_dtype == torch.float32 else 0)
             | (_lib.FLAG_P_SPLIT if split_p else 0))
    lib = _lib.load()
    kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
    ws_bytes = lib.infllm2_select_workspace_bytes(ctypes.byref(geom), n, hq, hkv, d, layer.length, flags)
    ws = _workspace(dev, ws_bytes)
    # below the sparsity threshold every row selects every block: dense causal
    # attention on the tensor cores (8 query rows x 16 heads per MMA tile)
    dense = (n > 0 and not exact and not split_p and hq // hkv == 16 and d == 128
             and lib.infllm2_dense_regime(ctypes.byref(geom), n, start, layer.length) == 1)
    if dense:
        st = _stream(dev)
        if return_selection or stats is not None or traces is not None:
            _lib.check(lib.infllm2_select(
                ctypes.byref(geom), _ptr(qb), qb.stride(0), n, start, hq, hkv, d, _ptr(fine), _ptr(hi), _ptr(lo),
                mcap, layer.length, _ptr(sel), _ptr(sel_scores), _ptr(ws), ws.numel(), flags, st),
                "two_stage_attention")
        _lib.check(lib.infllm2_dense_attend(
            ctypes.byref(geom), _ptr(qb), qb.stride(0), n, start, hq, hkv, d, _ptr(kc), _ptr(vc), cap, layer.length,
            _ptr(out), _ptr(lse_out), flags, st), "two_stage_attention")
    elif n and lse == "approx":
        layer._coarse_split()
        st = _stream(dev)
        _lib.check(lib.infllm2_select_approx(
            ctypes.byref(geom), _ptr(qb), qb.stride(0), n, start, hq, hkv, d, _ptr(fine), _ptr(hi), _ptr(lo), mcap,
            _ptr(layer._coarse), _ptr(layer._coarse_hi), _ptr(layer._coarse_lo), layer._coarse.shape[1],
            layer.length, _ptr(sel), _ptr(sel_scores), _ptr(ws), ws.numel(), flags, st), "two_stage_attention")
        _lib.check(lib.infllm2_attend(
            ctypes.byref(geom), _ptr(qb), qb.stride(0), n, start, hq, hkv, d, _ptr(kc), _ptr(vc), cap,
            layer.length, _ptr(sel), _ptr(out), _ptr(lse_out), flags, st), "two_stage_attention")
    elif n:
        _lib.check(lib.infllm2_forward(
            ctypes.byref(geom), _ptr(qb), qb.stride(0), n, start, hq, hkv, d, _ptr(kc), _ptr(vc), cap,
            layer.length, _ptr(fine), _ptr(hi), _ptr(lo), mcap, _ptr(sel), _ptr(sel_scores), _ptr(out),
            _ptr(lse_out), _ptr(ws), ws.numel(), flags, _stream(dev)), "two_stage_attention")
    if stats is not None or traces is not None:
        _account(sel, sel_scores, start, layer, config, stats, traces)
    if return_selection or return_lse:
        res = (out,)
        if return_selection:
            res += (sel,)
        if return_lse:
            res += (lse_out,)
        return res
    return out


def _account(sel: torch.Tensor, sel_scores: Optional[torch.Tensor], start: int,
             layer: BlockizedLayerCache, cfg: SparseAttentionConfig, stats, traces) -> None:
    """TouchStats and traces derived on the host from the selection tensor
    (sparse.py:456-467); same per-(row, group) order as the reference."""
    s_np = sel.cpu().numpy()
    sc_np = sel_scores.cpu().numpy() if sel_scores is not None else None
    n, hkv, _ = s_np.shape
    m, s = cfg.block_size, cfg.kernel_stride
    nk_total = layer.length // s
    for i in range(n):
        pos = start + i
        n_kernels = min(pos // s + 1, nk_total)
        forced = force_blocks(pos // m + 1, pos // m, cfg.n_init_blocks, cfg.n_local_blocks)
        for g in range(hkv):
            ids = s_np[i, g][s_np[i, g] >= 0]
            touched = int(sum(min((b + 1) * m, pos + 1) - b * m for b in ids))
            if stats is not None:
                stats.add(stage1=n_kernels, stage2=touched, dense_rows=pos + 1)
            if traces is not None:
                traces.append({
                    "query_pos": int(pos),
                    "group": int(g),
                    "forced": [int(b) for b in forced],
                    "selected": [int(b) for b in ids],
                    "scores_topk": [float(x) for x in sc_np[i, g, :ids.size]],
                })
