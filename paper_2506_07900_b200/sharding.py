"""Query-sequence sharding of InfLLM v2 prefill over N ranks (one process per GPU).

Rows are independent given the cache (chunked calls of the reference
are bitwise equal to one call), but every rank needs the GLOBAL cache: kernel
windows and nk_t depend on the full length L.  So:

* rank r owns query chunks r and 2N-1-r of 2N equal chunks ("zig-zag"): stage-1
  work grows linearly with position, so every rank's pair sums to the same work;
* each rank holds the K/V rows of its own tokens; one all-gather per chunk half
  (NCCL over NVLink on B200, gloo in the CPU tests) rebuilds the full K/V in
  natural order, which every rank appends to its blockized cache and compresses;
* outputs stay sharded (rank r's rows), no further collective.

Batched decode partitions whole sequences across ranks and needs no collective.
"""

from __future__ import annotations

from typing import Sequence

import torch
import torch.distributed as dist


def zigzag_chunks(seq: int, world: int, rank: int) -> list[tuple[int, int]]:
    """Row ranges [lo, hi) owned by `rank`: chunks rank and 2*world-1-rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    nch = 2 * world
    size = seq // nch
    bounds = [(c * size, (c + 1) * size if c < nch - 1 else seq) for c in range(nch)]
    return [bounds[rank], bounds[nch - 1 - rank]]


def natural_order(world: int) -> list[tuple[int, int]]:
    """For natural chunk c: (which gathered half, source rank)."""
    out = []
    for c in range(2 * world):
        out.append((0, c) if c < world else (1, 2 * world - 1 - c))
    return out


def _all_gather(dst: torch.Tensor, src: torch.Tensor, group=None) -> None:
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(dst, src, group=group)
    else:
        parts = list(dst.unbind(0))
        dist.all_gather(parts, src.contiguous(), group=group)


def gather_rows(local: Sequence[torch.Tensor], world: int, group=None) -> list[torch.Tensor]:
    """All-gather the per-rank chunk pairs of a row-major tensor (rows first).

    `local` = [rows of chunk rank, rows of chunk 2N-1-rank] (equal sizes across
    ranks; the last chunk may be longer only when world == 1).  Returns the 2N
    chunks in natural row order (views into two gather buffers).
    """
    if world == 1:
        return [local[0], local[1]]
    halves = []
    for h in range(2):
        src = local[h]
        buf = torch.empty((world,) + tuple(src.shape), dtype=src.dtype, device=src.device)
        _all_gather(buf, src, group)
        halves.append(buf)
    return [halves[h][r] for h, r in natural_order(world)]


def fill_layer_cache(cache, k_local: Sequence[torch.Tensor], v_local: Sequence[torch.Tensor], world: int,
                     group=None) -> None:
    """Rebuild the full-length cache on this rank from every rank's K/V shard."""
    cache.truncate(0)
    ks = gather_rows(k_local, world, group)
    vs = gather_rows(v_local, world, group)
    cache.append(torch.cat(ks), torch.cat(vs))


def sharded_prefill(q_local: Sequence[torch.Tensor], cache, config, chunks, attention):
    """Run `attention(q_chunk, cache, config, start)` on this rank's chunks."""
    return [attention(q, cache, config, lo) for q, (lo, _) in zip(q_local, chunks)]
