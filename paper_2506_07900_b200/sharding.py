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

from typing import Optional, Sequence

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
    """dst[(world, ...)] <- every rank's src.  NCCL gathers in place on the
    device; gloo (the CPU test transport, also used to run several ranks on one
    GPU) stages CUDA tensors through host memory."""
    backend = dist.get_backend(group)
    if backend == "nccl" and hasattr(dist, "all_gather_into_tensor"):
        dist.all_gather_into_tensor(dst, src.contiguous(), group=group)
        return
    if src.is_cuda:
        host = torch.empty(dst.shape, dtype=dst.dtype)
        dist.all_gather(list(host.unbind(0)), src.detach().cpu().contiguous(), group=group)
        dst.copy_(host)
        return
    dist.all_gather(list(dst.unbind(0)), src.contiguous(), group=group)


def gather_rows(local: Sequence[torch.Tensor], world: int, group=None) -> list[torch.Tensor]:
    """All-gather the per-rank chunk pairs of a row-major tensor (rows first).

    `local` = [rows of chunk rank, rows of chunk 2N-1-rank] (equal sizes across
    ranks; the last chunk may be longer only when world == 1).  Returns the 2N
    chunks in natural row order (views into two gather buffers).
    """
    return [c for run in _natural_runs(_gather_halves(local, world, group), world) for c in run]


def _gather_halves(local: Sequence[torch.Tensor], world: int, group=None) -> list[torch.Tensor]:
    if world == 1:
        return [local[0].unsqueeze(0), local[1].unsqueeze(0)]
    halves = []
    for h in range(2):
        src = local[h]
        buf = torch.empty((world,) + tuple(src.shape), dtype=src.dtype, device=src.device)
        _all_gather(buf, src, group)
        halves.append(buf)
    return halves


def _natural_runs(halves: list[torch.Tensor], world: int) -> list[list[torch.Tensor]]:
    """The gathered halves as runs of natural-order chunks: half 0 holds chunks
    0..N-1 in rank order (one contiguous run); half 1 holds chunks 2N-1..N in
    rank order, i.e. reversed (one run per chunk)."""
    h0, h1 = halves
    first = [h0.reshape((-1,) + tuple(h0.shape[2:]))] if world > 1 else [h0[0]]
    return [first, [h1[r] for r in range(world - 1, -1, -1)]]


class LayerGather:
    """One layer's K/V all-gather, optionally issued on a side stream so it
    overlaps the previous layer's attention; ``fill`` waits for it and appends
    the rows to the cache in natural order with no concatenation: the gathered
    buffers are read once by the fused append + compress kernel
    (infllm2_append_compress), which writes the cache and its kernel means."""

    def __init__(self, k_local: Sequence[torch.Tensor], v_local: Sequence[torch.Tensor], world: int, group=None,
                 stream: Optional[torch.cuda.Stream] = None):
        self.world = world
        self.event = None
        dev = k_local[0].device
        if stream is not None and dev.type == "cuda":
            main = torch.cuda.current_stream(dev)
            stream.wait_stream(main)            # the shards were produced on the main stream
            with torch.cuda.stream(stream):
                self.k = _gather_halves(k_local, world, group)
                self.v = _gather_halves(v_local, world, group)
                self.event = torch.cuda.Event()
                self.event.record(stream)
            for t in self.k + self.v:
                t.record_stream(main)           # consumed on the main stream
        else:
            self.k = _gather_halves(k_local, world, group)
            self.v = _gather_halves(v_local, world, group)

    def fill(self, cache) -> None:
        if self.event is not None:
            torch.cuda.current_stream(self.k[0].device).wait_event(self.event)
        cache.truncate(0)
        for krun, vrun in zip(_natural_runs(self.k, self.world), _natural_runs(self.v, self.world)):
            for kk, vv in zip(krun, vrun):
                cache.append(kk, vv)


def fill_layer_cache(cache, k_local: Sequence[torch.Tensor], v_local: Sequence[torch.Tensor], world: int,
                     group=None) -> None:
    """Rebuild the full-length cache on this rank from every rank's K/V shard."""
    LayerGather(k_local, v_local, world, group).fill(cache)


def sharded_prefill(q_local: Sequence[torch.Tensor], cache, config, chunks, attention):
    """Run `attention(q_chunk, cache, config, start)` on this rank's chunks."""
    return [attention(q, cache, config, lo) for q, (lo, _) in zip(q_local, chunks)]
