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
block.  (a) is one ``infllm2_forward_at`` call for all nodes (every row at the
same position: shared candidates and forced set; float64 scorer, tensor-core
stage 2); (b) is a tiny masked float64 attention.
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
