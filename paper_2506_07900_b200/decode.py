"""Batched single-token decode over S sequences (BASELINE configs[3]).

The reference decodes one sequence at a time by calling two_stage_attention with
n = 1 after appending the new token (model.py:434-444; specdec.py:717-718).  On
the B200 a decode step of S sequences for one layer is one batched call
(`infllm2_decode_step`): append + incremental kernel-mean re-sync, split-K
stage-1 on the tensor cores, block scores, top-k, stage-2 — five launches for
all sequences, no host synchronisation.  Sequences stay independent (each has
its own cache); a multi-GPU deployment partitions sequences across ranks with
no collective.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _lib
from .errors import ValidationError
from .sparse import BlockizedLayerCache, SparseAttentionConfig, _ptr, _stream, two_stage_attention


class DecodeBatch:
    """One layer's caches of S sequences, stepped together."""

    def __init__(self, layers: Sequence[BlockizedLayerCache], config: SparseAttentionConfig, *, concurrent: int = 1):
        """`concurrent`: how many decode batches will run AT THE SAME TIME on
        this device (micro-batches on separate streams, e.g. two halves of the
        sequences pipelined across layers): the fused kernel then sizes its
        thread-block clusters so that many launches are co-resident."""
        if not layers:
            raise ValidationError("empty decode batch")
        l0 = layers[0]
        for l in layers:
            if (l.n_kv_heads, l.head_dim, l.device) != (l0.n_kv_heads, l0.head_dim, l0.device):
                raise ValidationError("decode batch caches must share head geometry and device")
        self.layers = list(layers)
        self.config = config
        if not 1 <= int(concurrent) <= 15:
            raise ValidationError("concurrent must be in 1..15")
        self.concurrent = int(concurrent)
        self.device = l0.device
        self._table: Optional[torch.Tensor] = None
        self._sig = None
        self._ws: Optional[torch.Tensor] = None   # owned scratch: a captured graph keeps its pointer
        self._next: Optional["DecodeBatch"] = None
        self._lib = _lib.load()

    def _signature(self):
        return tuple((l._k.data_ptr(), l._v.data_ptr(), l._cap, l._fine.data_ptr(), l._coarse.data_ptr(), l.length)
                     for l in self.layers)

    def _ensure(self) -> None:
        for l in self.layers:
            l._reserve(l.length + 1)
        sig = self._signature()
        if sig == self._sig:
            return
        n = len(self.layers)
        descs = (_lib.SeqDesc * n)()
        lens = (ctypes.c_int64 * n)()
        for i, l in enumerate(self.layers):
            descs[i] = _lib.SeqDesc(l._k.data_ptr(), l._v.data_ptr(), l._cap, l._fine.data_ptr(), l._fine_hi.data_ptr(),
                                    l._fine_lo.data_ptr(), l._fine.shape[1], l._coarse.data_ptr(), l._coarse.shape[1])
            lens[i] = l.length
        nbytes = self._lib.infllm2_decode_table_bytes(n)
        if self._table is None or self._table.numel() < nbytes:
            self._table = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        _lib.check(self._lib.infllm2_decode_table_build(descs, lens, n, self.layers[0].n_kv_heads,
                                                        self.layers[0].head_dim, self._table.data_ptr(),
                                                        _stream(self.device)), "decode table")
        self._sig = sig
        self._write_link()

    def _write_link(self) -> None:
        nxt = self._next._table.data_ptr() if self._next is not None and self._next._table is not None else None
        _lib.check(self._lib.infllm2_decode_table_link(self._table.data_ptr(), len(self.layers), nxt,
                                                       _stream(self.device)), "decode table link")

    def link_next(self, nxt: Optional["DecodeBatch"]) -> None:
        """Declare the batch of the NEXT layer (same sequences, stepped right
        after this one): this layer's decode step then L2-prefetches the part
        of the next layer's kernel means each CTA streams next, during its own
        dependent tail.  A performance hint only (results are unchanged); the
        next batch's table must exist (call its reserve() first)."""
        if nxt is not None:
            if len(nxt.layers) != len(self.layers) or nxt.device != self.device:
                raise ValidationError("linked decode batches must hold the same number of sequences on one device")
            nxt._ensure()
        self._next = nxt
        self._ensure()
        self._write_link()

    def _fused_ok(self, hq: int, hkv: int, d: int) -> bool:
        """The library's own predicate (infllm2_decode_supported: (G, D) = (16, 128)
        or (8, 64), s = 16, p = 32, m = 64, max_selected <= 80); other geometries
        step each sequence through the prefill kernels."""
        return bool(self._lib.infllm2_decode_supported(ctypes.byref(self.config.geometry()), hq, hkv, d))

    def _step_per_sequence(self, q, k_new, v_new, return_selection, return_lse, out_dtype, bookkeep):
        """One decode step per sequence with the (n = 1) prefill kernels — same
        semantics (append, then attend the new row, model.py:434-444)."""
        if not bookkeep:
            raise ValidationError("graph replay (bookkeep=False) needs the batched decode kernels (G, D = 16, 128 or 8, 64)")
        outs, sels, lses = [], [], []
        for i, layer in enumerate(self.layers):
            layer.append(k_new[i:i + 1], v_new[i:i + 1])
            res = two_stage_attention(q[i:i + 1], layer, self.config, layer.length - 1, return_selection=True,
                                      return_lse=True, out_dtype=out_dtype)
            outs.append(res[0])
            sels.append(res[1])
            lses.append(res[2])
        out = torch.cat(outs)
        if return_selection or return_lse:
            ret = (out,)
            if return_selection:
                ret += (torch.cat(sels),)
            if return_lse:
                ret += (torch.cat(lses),)
            return ret
        return out

    def reserve(self, extra_tokens: int) -> None:
        """Preallocate room for `extra_tokens` more decode steps (no reallocation,
        hence no table rebuild, while they run — required for graph capture)."""
        for l in self.layers:
            l._reserve(l.length + extra_tokens)
        self._ensure()
        l0 = self.layers[0]
        bound = max(l.length for l in self.layers) + max(int(extra_tokens), 1)
        self._workspace(self._lib.infllm2_decode_workspace_bytes(ctypes.byref(self.config.geometry()),
                                                                 len(self.layers), l0.n_kv_heads, bound))

    def _workspace(self, nbytes: int) -> torch.Tensor:
        """This batch's own scratch, grown only outside graph capture: a graph
        captured over step() keeps the pointer, so the buffer lives (and is never
        shared with another stream's calls) as long as the batch does."""
        if self._ws is None or self._ws.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise ValidationError("decode workspace too small inside graph capture: call reserve() first")
            self._ws = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=self.device)
        return self._ws

    def advance(self, n: int = 1) -> None:
        """Host bookkeeping for `n` steps replayed from a captured graph."""
        for l in self.layers:
            l.length += n
            l._nk_valid = l.length // self.config.kernel_stride
            l._nc_valid = l.length // self.config.coarse_stride
        self._sig = self._signature()

    def step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, *, return_selection: bool = False,
             return_lse: bool = False, out_dtype: Optional[torch.dtype] = None, max_len: Optional[int] = None,
             bookkeep: bool = True):
        """Append (S, HKV, D) k_new/v_new and attend (S, HQ, D) q for every sequence.

        `max_len` fixes the length bound that sizes the split-K grid and the
        workspace (default: current max + 1).  Passing a fixed bound (e.g. the
        reserved capacity) makes the launches identical from step to step, so
        a whole multi-layer decode step can be captured in a CUDA graph and
        replayed (`bookkeep=False` inside the capture, then `advance()`).
        """
        n = len(self.layers)
        l0 = self.layers[0]
        hq, d = q.shape[1], q.shape[2]
        if q.shape[0] != n or k_new.shape != (n, l0.n_kv_heads, l0.head_dim) or v_new.shape != k_new.shape:
            raise ValidationError("decode step shapes must be q (S, HQ, D), k/v (S, HKV, D)")
        if hq % l0.n_kv_heads:
            raise ValidationError("query heads not divisible by KV heads")
        if not self._fused_ok(hq, l0.n_kv_heads, l0.head_dim):
            return self._step_per_sequence(q, k_new, v_new, return_selection, return_lse, out_dtype, bookkeep)
        self._ensure()
        dev = self.device
        qb = q.to(device=dev, dtype=torch.bfloat16).contiguous()
        kb = k_new.to(device=dev, dtype=torch.bfloat16).contiguous()
        vb = v_new.to(device=dev, dtype=torch.bfloat16).contiguous()
        out_dtype = out_dtype or (q.dtype if q.dtype in (torch.float32, torch.bfloat16) else torch.bfloat16)
        geom = self.config.geometry()
        smax = self.config.max_selected
        sel = torch.empty((n, l0.n_kv_heads, smax), dtype=torch.int32, device=dev)
        out = torch.empty((n, hq, d), dtype=out_dtype, device=dev)
        lse = torch.empty((n, hq), dtype=torch.float32, device=dev) if return_lse else None
        cur = max(l.length for l in self.layers) + 1
        max_len = cur if max_len is None else int(max_len)
        if max_len < cur:
            raise ValidationError("max_len below the longest sequence")
        ws_bytes = self._lib.infllm2_decode_workspace_bytes(ctypes.byref(geom), n, l0.n_kv_heads, max_len)
        ws = self._workspace(ws_bytes)
        flags = (_lib.FLAG_OUT_F32 if out_dtype == torch.float32 else 0) | (self.concurrent << _lib.DECODE_SHARE_SHIFT)
        _lib.check(self._lib.infllm2_decode_step(
            ctypes.byref(geom), self._table.data_ptr(), n, max_len, hq, l0.n_kv_heads, d, _ptr(qb), _ptr(kb),
            _ptr(vb), _ptr(sel), _ptr(out), _ptr(lse), _ptr(ws), ws.numel(), flags, _stream(dev)), "decode step")
        if bookkeep:                    # the device advanced every length by one
            self.advance(1)
        if return_selection or return_lse:
            res = (out,)
            if return_selection:
                res += (sel,)
            if return_lse:
                res += (lse,)
            return res
        return out
