"""Tree-draft verification through the sparse operator.

The reference scores a speculative draft tree with the DENSE ``forward_tree``
(specdec.py:565-625): node i sits at position ``cache.length + depth_i - 1``,
sees every cached row plus the tree rows its packed ancestor mask admits
(``PackedMask``, specdec.py:117-157), and the cache is never modified.  The
paper's CPM.cu verifies trees through the sparse kernel; the reference has no
such path, so its parity is anchored two ways (tests/test_tree_gpu.py): the
dense backend against the reference's ``forward_tree`` logits, and the sparse
backend against the dense one in the degradation regime (every block
selected), plus the operator against the oracle composition in the sparse
regime.

Definition (sparse backend): node i's attention is the log-sum-exp merge of
  (a) InfLLM v2 two-stage attention of q_i over the prefix cache, as a query at
      position ``base - 1`` (it sees every cached row), and
  (b) dense attention over its ancestor-or-self tree rows;
which is exactly dense attention over prefix ∪ ancestors when (a) selects every
block.

Default path: ONE ``infllm2_forward_tree`` call (the n x n
tree mask travels to the kernel bit-packed in uint64 words).  The draft rows'
K/V are written into the cache at [length, length + n) without advancing its
length; stage 1 scores every node at the broadcast position length - 1 on the
tensor cores (units of 16 nodes share candidates and forced set); stage 2
gathers each node's selected prefix blocks, then the tree rows, admitting tree
row j for node i iff bit j of ``words[i]`` is set - (a) and (b) in one online
softmax, no separate merge.  ``exact=True`` keeps the float64 verifier path:
``infllm2_forward_at`` (float64 scorer) + a float64 masked tree attention merged
by log-sum-exp on the host side of the device.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import torch

from . import _lib
from .errors import ValidationError
from .sparse import BlockizedLayerCache, SparseAttentionConfig, _ptr, _stream, _workspace


@dataclasses.dataclass
class PackedMask:
    """Ancestor-or-self visibility, bit-packed row-wise (specdec.py:117-157):
    bit j of row i (word j // 64, bit j % 64) is set when node j is node i or
    one of its ancestors."""

    words: np.ndarray  # (n, ceil(n/64)) uint64
    n_nodes: int

    @classmethod
    def from_parents(cls, parents) -> "PackedMask":
        parents = np.asarray(parents, dtype=np.int64).reshape(-1)
        n = parents.size
        words = np.zeros((n, max(1, -(-n // 64))), dtype=np.uint64)
        for i in range(n):
            p = int(parents[i])
            if not -1 <= p < i:
                raise ValidationError(f"node {i} parent {p} out of order")
            if p >= 0:
                words[i] = words[p]
            words[i, i // 64] |= np.uint64(1) << np.uint64(i % 64)
        return cls(words=words, n_nodes=n)

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.n_nodes, self.n_nodes), dtype=bool)
        for j in range(self.n_nodes):
            dense[:, j] = (self.words[:, j // 64] >> np.uint64(j % 64)) & np.uint64(1)
        return dense

    def validate(self) -> None:
        if self.words.dtype != np.uint64 or self.words.ndim != 2:
            raise ValidationError("mask words must be a 2-D uint64 array")
        if self.words.shape != (self.n_nodes, max(1, -(-self.n_nodes // 64))):
            raise ValidationError("mask word array has the wrong shape")
        if not self.to_dense().diagonal().all():
            raise ValidationError("every node must see itself")


def _tree_part(q: torch.Tensor, k_tree: torch.Tensor, v_tree: torch.Tensor, vis: torch.Tensor):
    """Dense attention of every node over its visible tree rows: float64
    softmax (model.py:194-226); returns (out (n, HQ, D) f64, lse (n, HQ) f64)."""
    n, hq, d = q.shape
    hkv = k_tree.shape[1]
    g = hq // hkv
    kk = k_tree.double().repeat_interleave(g, dim=1)            # (n, HQ, D)
    vv = v_tree.double().repeat_interleave(g, dim=1)
    s = torch.einsum("ihd,jhd->hij", q.float(), kk.float()).double() * float(np.float32(1.0 / np.sqrt(d)))
    s = s.masked_fill(~vis[None], float("-inf"))
    lse = torch.logsumexp(s, dim=-1)                             # (HQ, n)
    out = torch.einsum("hij,jhd->ihd", torch.exp(s - lse[..., None]), vv)
    return out, lse.transpose(0, 1)


def tree_attention(q: torch.Tensor, layer: BlockizedLayerCache, config: SparseAttentionConfig,
                   k_tree: torch.Tensor, v_tree: torch.Tensor, mask: PackedMask, *, exact: bool = False,
                   split_p: bool = False, return_selection: bool = False):
    """Attention of n tree nodes: q (n, HQ, D) over the prefix cache ``layer``
    (two-stage sparse, each node at position ``layer.length - 1``) merged with
    their ancestor-or-self rows of k_tree/v_tree (n, HKV, D).  The cache is not
    modified.  Returns float32 (n, HQ, D) [, int32 selection (n, HKV, max_sel)]."""
    if q.dim() != 3 or k_tree.dim() != 3 or k_tree.shape != v_tree.shape:
        raise ValidationError("q (n, HQ, D), k_tree/v_tree (n, HKV, D)")
    n = q.shape[0]
    if n == 0 or mask.n_nodes != n or k_tree.shape[0] != n:
        raise ValidationError("tree nodes, K/V rows and mask disagree on node count")
    if layer.length == 0:
        raise ValidationError("tree scoring needs a non-empty prefix cache")
    mask.validate()
    if not exact and _kernel_shape_ok(q.shape[1], layer.n_kv_heads, layer.head_dim, config, n):
        return _tree_attention_kernel(q, layer, config, k_tree, v_tree, mask, split_p, return_selection)
    dev = layer.device
    base = layer.length
    hq, d = q.shape[1], q.shape[2]
    hkv = layer.n_kv_heads
    if hq % hkv or d != layer.head_dim or k_tree.shape[1:] != (hkv, d):
        raise ValidationError("tree node heads / head_dim disagree with the cache")
    qb = q.to(device=dev, dtype=torch.bfloat16).contiguous()
    geom = config.geometry()
    sel = torch.empty((n, hkv, config.max_selected), dtype=torch.int32, device=dev)
    o_p = torch.empty((n, hq, d), dtype=torch.float32, device=dev)
    l_p = torch.empty((n, hq), dtype=torch.float32, device=dev)
    lib = _lib.load()
    kc, vc, cap, fine, _, _, mcap = layer._device_args()
    ws = _workspace(dev, lib.infllm2_forward_at_workspace_bytes(ctypes.byref(geom), n, hkv, base - 1, base))
    flags = (_lib.FLAG_OUT_F32 | (_lib.FLAG_EXACT_SIMT if exact else 0) | (_lib.FLAG_P_SPLIT if split_p else 0))
    _lib.check(lib.infllm2_forward_at(ctypes.byref(geom), _ptr(qb), qb.stride(0), n, base - 1, hq, hkv, d, _ptr(kc),
                                      _ptr(vc), cap, base, _ptr(fine), mcap, _ptr(sel), None, _ptr(o_p), _ptr(l_p),
                                      _ptr(ws), ws.numel(), flags, _stream(dev)), "tree_attention")
    o_p = o_p.double()
    l_p = l_p.double()
    vis = torch.as_tensor(mask.to_dense(), device=dev)
    o_t, l_t = _tree_part(q.to(dev), k_tree.to(dev), v_tree.to(dev), vis)
    m = torch.maximum(l_p, l_t)
    wp, wt = torch.exp(l_p - m), torch.exp(l_t - m)
    out = ((o_p * wp[..., None] + o_t * wt[..., None]) / (wp + wt)[..., None]).float()
    if return_selection:
        return out, sel
    return out


def _kernel_shape_ok(hq: int, hkv: int, d: int, config: SparseAttentionConfig, n: int) -> bool:
    """infllm2_forward_tree's envelope: the tensor-core head geometries
    (G = 16 / D = 128, G = 8 / D = 64), 64-row blocks, <= 80 selected blocks,
    <= 1024 nodes.  Other shapes (e.g. the reference's tiny test models) take
    the float64 path."""
    if hkv <= 0 or hq % hkv:
        return False
    return ((hq // hkv, d) in ((16, 128), (8, 64)) and config.block_size == 64 and config.max_selected <= 80
            and n <= 1024)


def _tree_attention_kernel(q, layer, config, k_tree, v_tree, mask, split_p, return_selection):
    """infllm2_forward_tree: tcgen05 stage 1 at the broadcast position and one
    stage-2 pass over the selected prefix blocks plus the mask-admitted tree
    rows (packed words consumed on the device)."""
    dev = layer.device
    n = q.shape[0]
    base = layer.length
    hq, d = q.shape[1], q.shape[2]
    hkv = layer.n_kv_heads
    if hq % hkv or d != layer.head_dim or k_tree.shape[1:] != (hkv, d):
        raise ValidationError("tree node heads / head_dim disagree with the cache")
    lib = _lib.load()
    layer._reserve(base + n)
    kt = k_tree.to(device=dev).contiguous()
    vt = v_tree.to(device=dev, dtype=kt.dtype).contiguous()
    if kt.dtype not in (torch.bfloat16, torch.float32):
        kt, vt = kt.float(), vt.float()
    # the draft rows go to [base, base + n): scratch past the cache length
    _lib.check(lib.infllm2_append_kv(_ptr(layer._k), _ptr(layer._v), layer._cap, hkv, d, _ptr(kt), _ptr(vt), n,
                                     hkv * d, 1 if kt.dtype == torch.float32 else 0, base, _stream(dev)), "tree rows")
    words = torch.as_tensor(np.ascontiguousarray(mask.words).view(np.int64), device=dev)
    qb = q.to(device=dev, dtype=torch.bfloat16).contiguous()
    geom = config.geometry()
    sel = torch.empty((n, hkv, config.max_selected), dtype=torch.int32, device=dev)
    out = torch.empty((n, hq, d), dtype=torch.float32, device=dev)
    kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
    ws = _workspace(dev, lib.infllm2_forward_tree_workspace_bytes(ctypes.byref(geom), n, hq, hkv, d, base))
    flags = _lib.FLAG_OUT_F32 | (_lib.FLAG_P_SPLIT if split_p else 0)
    _lib.check(lib.infllm2_forward_tree(ctypes.byref(geom), _ptr(qb), qb.stride(0), n, hq, hkv, d, _ptr(kc), _ptr(vc),
                                        cap, base, _ptr(fine), _ptr(hi), _ptr(lo), mcap, _ptr(words),
                                        words.shape[1], _ptr(sel), None, _ptr(out), None, _ptr(ws), ws.numel(),
                                        flags, _stream(dev)), "tree_attention")
    if return_selection:
        return out, sel
    return out
