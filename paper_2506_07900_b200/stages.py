"""Per-stage functions of the reference surface on CUDA tensors.

The reference's tests and callers import the individual stages of the sparse
path directly (``deskinfer.sparse``: ``kernel_scores``, ``group_scores``,
``block_scores``, ``RelevanceScores``, ``select_topk``, ``exact_lse``,
``approx_lse``, ``sparse_attend``; reference ``test_sparse.py:10-27``).  The
fused kernels in ``libinfllm2.so`` never materialise these intermediates, so
these are small GPU restatements of each stage for API completeness and for
per-stage checks; the hot path is ``two_stage_attention``.  Semantics follow the
reference line by line: float32 dot products, float64 softmax / group mean /
block max, (score desc, id asc) tie order, the same exceptions.

Inputs may be CUDA tensors or numpy arrays (moved to the current CUDA device);
results are CUDA tensors (scalars for the LSE functions).
"""

from __future__ import annotations

import dataclasses
import math
from typing import Sequence

import numpy as np
import torch

from .errors import NumericError, ValidationError


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_07900_b200 stage functions need a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def _t(x, dtype=torch.float32) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=x.device if x.is_cuda else _dev(), dtype=dtype)
    return torch.as_tensor(np.asarray(x), device=_dev()).to(dtype)


def _softmax_f64(s: torch.Tensor) -> torch.Tensor:
    """softmax_f64 (model.py:185-191): -inf entries get exactly zero mass."""
    m = s.max()
    m = torch.where(torch.isneginf(m), torch.zeros_like(m), m)
    e = torch.exp(s - m)
    return e / e.sum()


def _logsumexp_f64(s: torch.Tensor) -> float:
    """logsumexp (model.py:172-182)."""
    if s.numel() == 0:
        raise ValueError("logsumexp of an empty score vector")
    m = float(s.max())
    if math.isinf(m) and m < 0:
        return float("-inf")
    if not math.isfinite(m):
        raise NumericError("non-finite scores in logsumexp")
    return m + float(torch.log(torch.exp(s - m).sum()))


def kernel_scores(q_head, kernel_means) -> torch.Tensor:
    """Softmax over kernels of the scaled query/kernel dots (sparse.py:163-180).

    ``q_head`` (D,), ``kernel_means`` (n_kernels, D); float32 dots, float64
    softmax.  Returns a float64 simplex vector on the GPU."""
    q = _t(q_head)
    km = _t(kernel_means)
    if km.dim() != 2 or q.shape[-1] != km.shape[-1]:
        raise ValidationError(f"kernel mean shape {tuple(km.shape)} incompatible with query dim {q.shape[-1]}")
    if km.shape[0] == 0:
        raise ValidationError("no kernels to score")
    if not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(km).all())):
        raise NumericError("non-finite values in kernel scoring")
    scale = np.float32(1.0 / np.sqrt(q.shape[-1]))
    dots = (km @ q) * float(scale)                        # float32, as the reference's sgemv
    return _softmax_f64(dots.double())


def group_scores(per_head_scores) -> torch.Tensor:
    """Mean of the per-head kernel scores of one KV group (sparse.py:183-188)."""
    arr = _t(per_head_scores, torch.float64)
    if arr.dim() != 2 or arr.shape[0] == 0:
        raise ValidationError("expected (n_heads, n_kernels) score matrix")
    acc = arr[0].clone()
    for h in range(1, arr.shape[0]):                      # sequential in h, as numpy's reduce
        acc = acc + arr[h]
    return acc / arr.shape[0]


def _kernel_range(block, kernel_size: int, stride: int, n_kernels: int):
    start, end = block
    lo = 0 if start < kernel_size else (start - kernel_size) // stride + 1
    hi = min(n_kernels, -(-end // stride))
    return min(lo, n_kernels), hi


def block_scores(group_kernel_scores, blocks: Sequence[tuple[int, int]], kernel_size: int,
                 stride: int) -> torch.Tensor:
    """Per-block relevance: max over the kernels whose window meets the block,
    0.0 for an empty range (sparse.py:201-215)."""
    s = _t(group_kernel_scores, torch.float64)
    nk = s.shape[0]
    ranges = [_kernel_range(b, kernel_size, stride, nk) for b in blocks]
    if not ranges:
        return torch.zeros(0, dtype=torch.float64, device=s.device)
    width = max(1, max(hi - lo for lo, hi in ranges))
    lo = torch.tensor([r[0] for r in ranges], device=s.device)
    n = torch.tensor([max(0, r[1] - r[0]) for r in ranges], device=s.device)
    j = torch.arange(width, device=s.device)
    idx = (lo[:, None] + j[None, :]).clamp(max=max(nk - 1, 0))
    vals = s[idx] if nk else torch.zeros((len(ranges), width), dtype=torch.float64, device=s.device)
    vals = torch.where(j[None, :] < n[:, None], vals, torch.full_like(vals, -math.inf))
    out = vals.max(dim=1).values
    return torch.where(n > 0, out, torch.zeros_like(out))


@dataclasses.dataclass
class RelevanceScores:
    """Stage-1 output for one (query token, KV group) (sparse.py:230-244)."""

    scores: torch.Tensor
    forced: torch.Tensor

    def __post_init__(self) -> None:
        if tuple(self.scores.shape) != tuple(self.forced.shape):
            raise ValidationError("scores/forced shape mismatch")


def select_topk(scores, k: int, forced, *, forced_consume_budget: bool = False) -> torch.Tensor:
    """Forced blocks plus the k best others by (score desc, id asc), ids
    ascending (sparse.py:247-277)."""
    s = _t(scores, torch.float64)
    if k <= 0:
        raise ValidationError("k must be positive")
    n = s.shape[0]
    f = _t(forced, torch.int64).reshape(-1)
    if f.numel() and (int(f.min()) < 0 or int(f.max()) >= n):
        raise ValidationError("forced block id out of range")
    fset = torch.unique(f)
    budget = max(0, k - fset.numel()) if forced_consume_budget else k
    is_forced = torch.zeros(n, dtype=torch.bool, device=s.device)
    is_forced[fset] = True
    cand = torch.nonzero(~is_forced).reshape(-1)            # ascending ids
    if cand.numel() and budget > 0:
        order = torch.sort(-s[cand], stable=True).indices  # stable: equal scores keep id order
        chosen = cand[order[:budget]]
    else:
        chosen = cand[:0]
    return torch.sort(torch.cat([fset, chosen])).values


def exact_lse(q_head, fine_means) -> float:
    """Log-sum-exp of the scaled query/kernel dots over every fine kernel (sparse.py:284-289)."""
    fm = _t(fine_means)
    if fm.shape[0] == 0:
        raise ValidationError("no kernels for exact_lse")
    q = _t(q_head)
    scale = float(np.float32(1.0 / np.sqrt(q.shape[-1])))
    return _logsumexp_f64(((fm @ q) * scale).double())


def approx_lse(q_head, coarse_means, kernel_stride: int, coarse_stride: int) -> float:
    """Coarse-kernel estimate of the fine-kernel log-sum-exp plus
    ln(coarse_stride / kernel_stride) (sparse.py:292-312)."""
    cm = _t(coarse_means)
    if cm.shape[0] == 0:
        raise ValidationError("no coarse kernels for approx_lse")
    if coarse_stride < kernel_stride or coarse_stride % kernel_stride:
        raise ValidationError("coarse_stride must be a multiple of kernel_stride")
    q = _t(q_head)
    scale = float(np.float32(1.0 / np.sqrt(q.shape[-1])))
    return _logsumexp_f64(((cm @ q) * scale).double()) + float(np.log(coarse_stride / kernel_stride))


def sparse_attend(q_heads, keys, values, selected, blocks: Sequence[tuple[int, int]], position: int,
                  group: int, group_size: int) -> tuple[torch.Tensor, int]:
    """Attention of one query token over the selected blocks of one KV group
    (sparse.py:347-384): rows after ``position`` excluded; float32 dots,
    float64 softmax and weighted sum, float32 output.  Returns (out, rows)."""
    sel = _t(selected, torch.int64).reshape(-1).tolist()
    if len(sel) == 0:
        raise ValidationError("empty block selection")
    gather = []
    for b in sel:
        start, end = blocks[int(b)]
        end = min(end, position + 1)
        if start <= position:
            gather.append(torch.arange(start, end))
    if not gather:
        raise ValidationError("selection contains no causally visible rows")
    qh = _t(q_heads)
    rows = torch.cat(gather).to(qh.device)
    k = _t(keys)[rows, group, :]
    v = _t(values)[rows, group, :].double()
    scale = float(np.float32(1.0 / np.sqrt(qh.shape[-1])))
    out = torch.empty_like(qh, dtype=torch.float32)
    for h in range(qh.shape[0]):
        probs = _softmax_f64(((k @ qh[h]) * scale).double())
        out[h] = (probs @ v).float()
    return out, int(rows.numel())
