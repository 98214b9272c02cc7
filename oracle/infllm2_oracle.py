"""CPU oracle for InfLLM v2 two-stage block-sparse attention.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the
``paper_2506_07900_b200`` package, its CUDA library, ``bench.py``'s own arm)
may import or call this module.  It is used by ``tests/`` as the checker, by
``__graft_entry__.smoke()`` as the checker, and by ``bench.py`` only for the
``cpu_baseline`` leg and the ``--impl reference`` arm.

This is a restatement, in vectorised numpy, of the reference's algorithm in
``/root/reference/pkg/src/deskinfer/sparse.py`` (abbreviated ``sparse.py``)
and of the numeric helpers in ``/root/reference/pkg/src/deskinfer/model.py``
(``model.py``).  Every function cites the reference lines it follows.  The
arithmetic is kept in the reference's order wherever the order affects
rounding:

* kernel means: sequential float64 sum over the window rows, float64 divide by
  the clipped window width, round-to-nearest float32 (``sparse.py:70-73``);
* stage-1 scores: per-head softmax in float64 (``model.py:185-191``), the
  group mean as a sequential float64 sum over heads divided by the group size
  (``sparse.py:183-188``), block max over intersecting kernels
  (``sparse.py:191-215``), forced blocks and top-k with the lower-id
  tie-break (``sparse.py:218-277``);
* stage-2: float64 softmax over the gathered rows, float64 value mix, float32
  output (``sparse.py:347-384``).

The only arithmetic the reference leaves to a third-party library is the
float32 dot product (``sparse.py:179,381``), which numpy hands to OpenBLAS
``sgemv`` with a CPU-kernel-specific summation order.  ``dot="sgemv"``
reproduces that call shape exactly (one matrix-vector product per head), so on
the same numpy/OpenBLAS build the oracle is bit-identical to the reference;
``dot="f64"`` forms every dot product in float64 instead, which is
machine-independent.  Parity is pinned by ``tests/golden/`` fixtures that the
reference itself produced (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np


class OracleValidationError(ValueError):
    """Mirror of ``container.ValidationError`` (container.py:48-49)."""


# --------------------------------------------------------------------------
# geometry (sparse.py:31-51)


@dataclasses.dataclass(frozen=True)
class Geometry:
    block_size: int = 64          # m
    kernel_size: int = 32         # p
    kernel_stride: int = 16       # s
    coarse_stride: int = 128      # s_c
    top_k: int = 8                # k
    n_init_blocks: int = 1
    n_local_blocks: int = 2
    forced_consume_budget: bool = False

    def __post_init__(self) -> None:  # sparse.py:42-51
        if min(self.block_size, self.kernel_size, self.kernel_stride,
               self.coarse_stride, self.top_k) <= 0:
            raise OracleValidationError("sizes must be positive")
        if self.kernel_stride > self.kernel_size:
            raise OracleValidationError("kernel_stride must not exceed kernel_size")
        if self.coarse_stride < self.kernel_stride or self.coarse_stride % self.kernel_stride:
            raise OracleValidationError("coarse_stride must be a multiple of kernel_stride")
        if self.n_init_blocks < 0 or self.n_local_blocks < 0:
            raise OracleValidationError("forced block counts must be non-negative")

    @property
    def max_selected(self) -> int:
        """Upper bound on |selection| (forced + top-k), ``SPEC.md`` BlockSelection."""
        return self.top_k + self.n_init_blocks + self.n_local_blocks


# --------------------------------------------------------------------------
# partitioning and kernel means (sparse.py:58-140)


def partition_blocks(length: int, block_size: int) -> list[tuple[int, int]]:
    """[(j*m, min((j+1)*m, L))]; the last block may be short (sparse.py:58-67)."""
    if block_size <= 0 or length < 0:
        raise OracleValidationError("bad partition arguments")
    return [(b, min(b + block_size, length)) for b in range(0, length, block_size)]


def window_means(keys: np.ndarray, kernel_size: int, stride: int,
                 first: int = 0) -> np.ndarray:
    """Mean-pooled windows ``[j*s, min(j*s+p, L))`` for ``first <= j < L//s``.

    Restates ``_window_mean``/``build_kernels`` (sparse.py:70-91): each window
    is summed row by row in float64 (numpy's axis-0 reduction is sequential),
    divided in float64 by its clipped width and rounded to float32.  The loop
    runs over the row offset inside the window so that every window keeps that
    sequential order while all windows advance together.
    """
    if kernel_size <= 0 or stride <= 0:
        raise OracleValidationError("kernel_size and stride must be positive")
    keys = np.asarray(keys)
    length = keys.shape[0]
    count = length // stride
    first = min(max(first, 0), count)
    starts = np.arange(first, count, dtype=np.int64) * stride
    widths = np.minimum(starts + kernel_size, length) - starts
    acc = np.zeros((count - first,) + keys.shape[1:], dtype=np.float64)
    for r in range(kernel_size):
        live = widths > r
        if not live.any():
            break
        acc[live] += keys[starts[live] + r].astype(np.float64)
    shape = (-1,) + (1,) * (keys.ndim - 1)
    return (acc / widths.reshape(shape).astype(np.float64)).astype(np.float32)


def first_dirty_window(boundary: int, kernel_size: int, stride: int, count: int) -> int:
    """First window whose contents change at ``boundary`` (sparse.py:119-120)."""
    first = 0 if boundary < kernel_size else (boundary - kernel_size) // stride + 1
    return min(first, count)


def updated_means(old_means: np.ndarray, keys: np.ndarray, kernel_size: int,
                  stride: int, boundary: int) -> np.ndarray:
    """Incremental re-sync after append/truncate (sparse.py:111-133).

    One deliberate deviation: ``first`` is also clipped to the number of
    windows that already exist.  The reference clips only to the new count
    (``sparse.py:120``), so when ``stride > kernel_size`` (the default coarse
    stride 128 > kernel 32) an append that crosses a stride multiple from an
    old length with ``old % stride >= kernel_size`` raises a numpy broadcast
    error at ``sparse.py:122``.  Clipping
    restores the reference's own invariant, incremental == rebuild
    (``test_sparse.py:276-290``).
    """
    count = keys.shape[0] // stride
    first = min(first_dirty_window(boundary, kernel_size, stride, count), old_means.shape[0])
    out = np.empty((count,) + keys.shape[1:], dtype=np.float32)
    out[:first] = old_means[:first]
    out[first:] = window_means(keys, kernel_size, stride, first)
    return out


# --------------------------------------------------------------------------
# numeric helpers (model.py:172-191)


def softmax_f64(scores: np.ndarray, axis: int = -1) -> np.ndarray:
    """Max-subtracted float64 softmax; -inf rows get zero mass (model.py:185-191)."""
    s = np.asarray(scores, dtype=np.float64)
    mx = np.max(s, axis=axis, keepdims=True)
    mx = np.where(np.isneginf(mx), 0.0, mx)
    e = np.exp(s - mx)
    return e / np.sum(e, axis=axis, keepdims=True)


def logsumexp_f64(scores: np.ndarray, axis: int = -1) -> np.ndarray:
    """log(sum(exp)) with max subtraction in float64 (model.py:172-182)."""
    s = np.asarray(scores, dtype=np.float64)
    mx = np.max(s, axis=axis, keepdims=True)
    return (mx + np.log(np.sum(np.exp(s - mx), axis=axis, keepdims=True))).squeeze(axis)


def scaled_dots(rows: np.ndarray, q_heads: np.ndarray, dot: str) -> np.ndarray:
    """(H, R) float64 scores ``f64(rows @ q_h) * (1/sqrt(D))`` (sparse.py:178-179,378-381).

    ``dot="sgemv"`` issues one float32 matrix-vector product per head, exactly
    the call the reference makes; ``dot="f64"`` forms the products in float64.
    """
    scale = 1.0 / np.sqrt(q_heads.shape[-1])       # numpy float64 scalar
    if dot == "sgemv":
        # Keep the caller's (possibly strided) view: numpy picks its BLAS path
        # from the operand layout, and the reference passes strided views.
        rows32 = rows if rows.dtype == np.float32 else rows.astype(np.float32)
        q32 = np.asarray(q_heads, dtype=np.float32)
        return np.stack([(rows32 @ q32[h]) * scale for h in range(q32.shape[0])])
    if dot == "f64":
        return (np.asarray(q_heads, np.float64) @ np.asarray(rows, np.float64).T) * scale
    raise ValueError(f"unknown dot mode {dot!r}")


# --------------------------------------------------------------------------
# stage 1 (sparse.py:163-277)


def kernel_range_for_block(start: int, end: int, kernel_size: int, stride: int,
                           n_kernels: int) -> tuple[int, int]:
    """Half-open kernel range intersecting [start, end) (sparse.py:191-198)."""
    lo = 0 if start < kernel_size else (start - kernel_size) // stride + 1
    hi = min(n_kernels, -(-end // stride))
    return min(lo, n_kernels), hi


def group_kernel_scores(q_heads: np.ndarray, means: np.ndarray, dot: str) -> np.ndarray:
    """S_j = mean_h softmax_j(z_hj) over the group's heads (sparse.py:163-188).

    ``means`` is (nk_t, D) for one KV group.  The per-head softmax rows are
    stacked (G, nk_t) and averaged along axis 0, i.e. a sequential float64 sum
    over heads divided by G, as ``group_scores`` does.
    """
    if means.shape[0] == 0:
        raise OracleValidationError("no kernels to score")
    z = scaled_dots(means, q_heads, dot)
    if not np.isfinite(z).all():
        raise OracleValidationError("non-finite values in kernel scoring")
    per_head = np.stack([softmax_f64(z[h]) for h in range(z.shape[0])])
    return per_head.mean(axis=0)


def block_scores(gscores: np.ndarray, pos: int, geom: Geometry) -> np.ndarray:
    """R_b for candidate blocks b = 0..pos//m, clipped to pos+1 (sparse.py:201-215,421-425)."""
    m, p, s = geom.block_size, geom.kernel_size, geom.kernel_stride
    n_cand = pos // m + 1
    nk = gscores.shape[0]
    out = np.zeros(n_cand, dtype=np.float64)
    for b in range(n_cand):
        lo, hi = kernel_range_for_block(b * m, min((b + 1) * m, pos + 1), p, s, nk)
        if hi > lo:
            out[b] = gscores[lo:hi].max()
    return out


def force_blocks(n_blocks: int, query_block: int, n_init: int, n_local: int) -> np.ndarray:
    """Leading ``n_init`` plus the ``n_local`` blocks ending at the query's (sparse.py:218-227)."""
    if not 0 <= query_block < max(n_blocks, 1):
        raise OracleValidationError("query block out of range")
    forced = set(range(min(n_init, n_blocks)))
    if n_local > 0:
        forced.update(range(max(0, query_block - n_local + 1), query_block + 1))
    return np.asarray(sorted(forced), dtype=np.int64)


def select_topk(scores: np.ndarray, k: int, forced: np.ndarray,
                forced_consume_budget: bool = False) -> np.ndarray:
    """Forced ∪ best ``budget`` non-forced ids by (-score, id), ascending (sparse.py:247-277)."""
    scores = np.asarray(scores, dtype=np.float64)
    if k <= 0:
        raise OracleValidationError("k must be positive")
    n = scores.shape[0]
    forced = np.asarray(forced, dtype=np.int64)
    if forced.size and (forced.min() < 0 or forced.max() >= n):
        raise OracleValidationError("forced block id out of range")
    is_forced = np.zeros(n, dtype=bool)
    is_forced[forced] = True
    budget = max(0, k - int(is_forced.sum())) if forced_consume_budget else k
    cand = np.flatnonzero(~is_forced)
    chosen = cand[np.argsort(-scores[cand], kind="stable")[:budget]] if budget else cand[:0]
    return np.union1d(forced, chosen).astype(np.int64)


def selection_margin(scores: np.ndarray, selected: np.ndarray, forced: np.ndarray) -> float:
    """Gap between the weakest chosen and the strongest rejected candidate.

    Used only to report how ambiguous a selection mismatch was.
    """
    cand = np.setdiff1d(np.arange(scores.shape[0]), forced)
    chosen = np.intersect1d(cand, selected)
    rejected = np.setdiff1d(cand, selected)
    if chosen.size == 0 or rejected.size == 0:
        return math.inf
    return float(scores[chosen].min() - scores[rejected].max())


# --------------------------------------------------------------------------
# stage 2 (sparse.py:347-384) and the driver (sparse.py:387-468)


def selected_rows(selected: np.ndarray, pos: int, block_size: int) -> np.ndarray:
    """Rows of the selected blocks clipped causally to ``pos`` (sparse.py:367-375)."""
    parts = [np.arange(b * block_size, min((b + 1) * block_size, pos + 1))
             for b in selected if b * block_size <= pos]
    if not parts:
        raise OracleValidationError("selection contains no causally visible rows")
    return np.concatenate(parts)


def sparse_attend(q_heads: np.ndarray, keys_g: np.ndarray, values_g: np.ndarray,
                  rows: np.ndarray, dot: str) -> tuple[np.ndarray, np.ndarray]:
    """Per-head float64 softmax over ``rows`` and value mix (sparse.py:376-383).

    Returns (out float32 (G, D), lse float64 (G,)).  The LSE is not returned
    by the reference; it is the natural-log normaliser of the same
    scores.
    """
    z = scaled_dots(keys_g[rows], q_heads, dot)
    v = values_g[rows].astype(np.float64)
    probs = softmax_f64(z, axis=-1)
    return (probs @ v).astype(np.float32), logsumexp_f64(z, axis=-1)


@dataclasses.dataclass
class OracleResult:
    out: np.ndarray            # (n, HQ, D) float32
    selection: np.ndarray      # (n, HKV, max_selected) int32, ascending, -1 padded
    lse: np.ndarray            # (n, HQ) float64
    stage1_rows: int = 0       # TouchStats.stage1 (sparse.py:319-344)
    stage2_rows: int = 0
    dense_rows: int = 0
    samples: int = 0
    margins: Optional[np.ndarray] = None   # (n, HKV) float64 selection margins
    scores: Optional[list] = None          # per (row, group) block scores if kept


def approx_group_kernel_scores(q_heads: np.ndarray, means: np.ndarray, coarse: np.ndarray,
                               geom: Geometry, dot: str) -> np.ndarray:
    """S_j under the approx-LSE selection mode (opt-in).

    The reference has no driver for this mode: ``approx_lse`` (sparse.py:292-312)
    is its only LSE estimator.  Definition used here and by the GPU (DESIGN §4
    K2p): head h's weights are P_hj = exp(z_hj - approx_lse(q_h, coarse[:nc_t]))
    in float64, with nc_t = min(t // s_c + 1, L // s_c) coarse kernels (the
    causal analogue of nk_t, sparse.py:426) passed in as ``coarse``; then the
    group mean in head order (sparse.py:183-188).  With no coarse kernel
    (L < s_c) the exact softmax is used.
    """
    if coarse.shape[0] == 0:
        return group_kernel_scores(q_heads, means, dot)
    z = scaled_dots(means, q_heads, dot)
    if not np.isfinite(z).all():
        raise OracleValidationError("non-finite values in kernel scoring")
    per_head = np.stack([np.exp(z[h] - approx_lse(q_heads[h], coarse, geom.kernel_stride,
                                                   geom.coarse_stride, dot))
                         for h in range(z.shape[0])])
    return per_head.mean(axis=0)


def two_stage_attention(q: np.ndarray, keys: np.ndarray, values: np.ndarray,
                        fine_means: np.ndarray, geom: Geometry, start_position: int,
                        *, rows: Optional[np.ndarray] = None, dot: str = "f64",
                        keep_scores: bool = False, lse_mode: str = "exact",
                        coarse_means: Optional[np.ndarray] = None) -> OracleResult:
    """Restatement of ``two_stage_attention`` (sparse.py:387-468).

    ``keys``/``values`` are the whole cache (L, HKV, D); ``fine_means`` its
    (L//s, HKV, D) float32 kernel means.  ``rows`` optionally restricts the
    computation to a subset of query rows (results for other rows are zero /
    -1); rows are independent given the cache.  ``lse_mode="approx"``
    (with ``coarse_means`` (L//s_c, HKV, D)) normalises stage 1 by approx_lse
    instead of the exact softmax (see ``approx_group_kernel_scores``).
    """
    if lse_mode not in ("exact", "approx"):
        raise OracleValidationError(f"unknown lse_mode {lse_mode!r}")
    if lse_mode == "approx" and coarse_means is None:
        raise OracleValidationError("approx lse_mode needs coarse_means")
    n, hq, d = q.shape
    length, hkv, _ = keys.shape
    if hkv and hq % hkv:
        raise OracleValidationError("query heads not divisible by KV heads")
    g_size = hq // hkv
    m, s = geom.block_size, geom.kernel_stride
    nk_total = fine_means.shape[0]
    smax = geom.max_selected
    res = OracleResult(
        out=np.zeros((n, hq, d), np.float32),
        selection=np.full((n, hkv, smax), -1, np.int32),
        lse=np.zeros((n, hq), np.float64),
        margins=np.full((n, hkv), np.inf),
        scores=[] if keep_scores else None,
    )
    row_ids = range(n) if rows is None else [int(r) for r in rows]
    for i in row_ids:
        pos = start_position + i
        if pos >= length:
            raise OracleValidationError(f"query position {pos} beyond cache length {length}")
        n_cand = pos // m + 1
        n_kernels = min(pos // s + 1, nk_total)          # sparse.py:426
        forced = force_blocks(n_cand, pos // m, geom.n_init_blocks, geom.n_local_blocks)
        for g in range(hkv):
            qh = q[i, g * g_size:(g + 1) * g_size, :]
            if n_kernels > 0 and lse_mode == "approx":
                nc_t = min(pos // geom.coarse_stride + 1, coarse_means.shape[0])
                gs = approx_group_kernel_scores(qh, fine_means[:n_kernels, g, :], coarse_means[:nc_t, g, :],
                                                geom, dot)
                bs = block_scores(gs, pos, geom)
            elif n_kernels > 0:
                gs = group_kernel_scores(qh, fine_means[:n_kernels, g, :], dot)
                bs = block_scores(gs, pos, geom)
            else:
                bs = np.zeros(n_cand, dtype=np.float64)
            sel = select_topk(bs, geom.top_k, forced, geom.forced_consume_budget)
            res.selection[i, g, :sel.size] = sel
            res.margins[i, g] = selection_margin(bs, sel, forced)
            if keep_scores:
                res.scores.append((i, g, bs))
            r = selected_rows(sel, pos, m)
            o, lse = sparse_attend(qh, keys[:, g, :], values[:, g, :], r, dot)
            res.out[i, g * g_size:(g + 1) * g_size] = o
            res.lse[i, g * g_size:(g + 1) * g_size] = lse
            res.stage1_rows += n_kernels
            res.stage2_rows += int(r.size)
            res.dense_rows += pos + 1
            res.samples += 1
    return res


# --------------------------------------------------------------------------
# LSE estimators (sparse.py:284-312) and dense attention (model.py:194-253)


def exact_lse(q_head: np.ndarray, fine_means: np.ndarray, dot: str = "sgemv") -> float:
    """logsumexp over every fine kernel (sparse.py:284-289)."""
    if fine_means.shape[0] == 0:
        raise OracleValidationError("no kernels for exact_lse")
    return float(logsumexp_f64(scaled_dots(fine_means, q_head[None], dot)[0]))


def approx_lse(q_head: np.ndarray, coarse_means: np.ndarray, kernel_stride: int,
               coarse_stride: int, dot: str = "sgemv") -> float:
    """Coarse-kernel logsumexp plus ln(s_c/s) (sparse.py:292-312)."""
    if coarse_means.shape[0] == 0:
        raise OracleValidationError("no coarse kernels for approx_lse")
    if coarse_stride < kernel_stride or coarse_stride % kernel_stride:
        raise OracleValidationError("coarse_stride must be a multiple of kernel_stride")
    base = float(logsumexp_f64(scaled_dots(coarse_means, q_head[None], dot)[0]))
    return base + float(np.log(coarse_stride / kernel_stride))


def dense_attention(q: np.ndarray, keys: np.ndarray, values: np.ndarray,
                    causal_offset: int, dot: str = "f64") -> tuple[np.ndarray, np.ndarray]:
    """Causal GQA attention, float64 softmax (model.py:194-253).

    ``q`` (n, HQ, D), ``keys``/``values`` (L, HKV, D).  Returns (out float32,
    lse float64 (n, HQ)).
    """
    n, hq, d = q.shape
    length, hkv, _ = keys.shape
    if causal_offset < 0 or causal_offset + n > length:
        raise OracleValidationError("causal_offset out of range")
    g_size = hq // hkv
    out = np.empty((n, hq, d), np.float32)
    lse = np.empty((n, hq), np.float64)
    for i in range(n):
        pos = causal_offset + i
        for g in range(hkv):
            qh = q[i, g * g_size:(g + 1) * g_size]
            z = scaled_dots(keys[:pos + 1, g], qh, dot)
            probs = softmax_f64(z, axis=-1)
            out[i, g * g_size:(g + 1) * g_size] = (
                probs @ values[:pos + 1, g].astype(np.float64)).astype(np.float32)
            lse[i, g * g_size:(g + 1) * g_size] = logsumexp_f64(z, axis=-1)
    return out, lse


def stage2_rows_closed_form(pos: int, geom: Geometry) -> int:
    """Stage-2 rows per (query, group) (SURVEY §8(a) closed form, n_local >= 1)."""
    m = geom.block_size
    n_cand = pos // m + 1
    forced = force_blocks(n_cand, pos // m, geom.n_init_blocks, geom.n_local_blocks)
    budget = geom.top_k - forced.size if geom.forced_consume_budget else geom.top_k
    if n_cand - forced.size <= max(budget, 0):
        return pos + 1
    return (forced.size + max(budget, 0) - 1) * m + (pos % m) + 1
