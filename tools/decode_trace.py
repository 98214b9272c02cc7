"""Phase timeline of one fused decode launch (INFLLM2_DECODE_TRACE=1).

Prints, per phase, min / median / max over CTAs of the %globaltimer stamp
relative to the earliest CTA start (microseconds)."""
import ctypes
import os
import sys

os.environ["INFLLM2_DECODE_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P
from paper_2506_07900_b200 import _lib

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
batches = []
for layer in range(4):          # 4 layers, one graph: the trace ring holds all 4 launches
    caches = []
    for s in range(S):
        c = P.BlockizedLayerCache(2, 128, cfg, capacity=L + 64)
        c.append(torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16),
                 torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16))
        caches.append(c)
    b = P.DecodeBatch(caches, cfg)
    b.reserve(32)
    batches.append(b)
for i in range(3):                # layer i prefetches layer i+1's means (INFLLM2_DECODE_PREFETCH=1: on)
    batches[i].link_next(batches[i + 1])
q = torch.randn((S, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
kn = torch.randn((S, 2, 128), generator=g, device="cuda").to(torch.bfloat16)


def step(bookkeep=True):
    for b in batches:
        b.step(q, kn, kn, max_len=L + 32, bookkeep=bookkeep)


side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
graph = torch.cuda.CUDAGraph()
with torch.cuda.stream(side):
    step()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=side):
        step(bookkeep=False)
for _ in range(3):
    graph.replay()
    for b in batches:
        b.advance(1)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (4 * 160 * 24))()
lib.infllm2_debug_decode_trace(buf, 4 * 160 * 24)
ring = np.array(buf, dtype=np.float64).reshape(4, 160, 24)
smid = ring[3, :, 11].copy()
early = ring[:, :, 21].copy()
print("early flag per launch (CTA 0):", early[:, 0])
ring[:, :, 21] = 0
ring[ring == 0] = np.nan
for i in range(3):
    gap = np.nanmin(ring[i + 1, :, 0]) - np.nanmax(ring[i, :, 10])
    dur = np.nanmax(ring[i, :, 10]) - np.nanmin(ring[i, :, 0])
    print(f"launch {i}: duration {dur / 1e3:.2f} us, gap to next launch {gap / 1e3:.2f} us")
t = ring[3]
t0 = np.nanmin(t[:, 0])
ok = ~np.isnan(t[:, 15]) & ~np.isnan(t[:, 11])
mhz = (t[ok, 11] - t[ok, 15]) / (t[ok, 10] - t[ok, 0]) * 1e3
print(f"SM clock inside the kernel: median {np.median(mhz):.0f} MHz (min {mhz.min():.0f}, max {mhz.max():.0f})")
names = ["start", "prod: stage-1 TMA issued", "epi: stage-1 partial", "epi: segment stage-1 complete",
         "epi: block scores", "epi: local top-k", "merge published", "prod: selection seen",
         "epi: first stage-2 partial", "epi: segment done", "CTA end", "(smid)", "epi: first z tile", "epi: append done",
         "combine start (after x3)", "-", "lengths read", "prod: past pdl_wait", "mma: q ready",
         "mma: tile 0 ready", "epi: past pdl_wait"]
for i, n in enumerate(names):
    if i in (11, 15, 21):
        continue
    col = (t[:, i] - t0) / 1e3
    col = col[~np.isnan(col)]
    if col.size:
        print(f"{n:34s} n={col.size:4d} min={col.min():7.2f} med={np.median(col):7.2f} max={col.max():7.2f} us")

order = np.argsort(-np.nan_to_num(t[:, 2] - t0, nan=-1))
print("slowest stage-1 CTAs: cta smid first_tile tma_done partial append")
for c in order[:12]:
    print(f"  {c:4d} {int(smid[c]):4d} {(t[c,12]-t0)/1e3:7.2f} {(t[c,1]-t0)/1e3:7.2f} {(t[c,2]-t0)/1e3:7.2f} {(t[c,13]-t0)/1e3:7.2f}")
print("fastest:")
for c in order[-150:][::-1][:0]:
    pass
fin = np.nan_to_num(t[:144, 2] - t0, nan=0) / 1e3
cb = (ctypes.c_longlong * (160 * 32))()
lib.infllm2_debug_decode_cycles(cb, 160 * 32)
cy = np.array(cb, dtype=np.float64).reshape(160, 32)[:8, :18]
steps = ["x1->LSE", "LSE->S_j", "S_j->R_b", "R_b->localtopk", "topk->x2", "x2->merge loads", "loads->rank",
         "(7)", "(8)", "rank->sel_s", "sel_s->s2_full", "s2_full->tilemax", "tilemax->o_full",
         "o_full->partial(unused)", "tiles->x3", "x3->combine loads", "loads->end"]
d = np.diff(cy, axis=1)
print("cycles per phase (cluster 0, pieces 0..7):")
for i, n in enumerate(steps):
    print(f"  {n:22s} " + " ".join(f"{v:7.0f}" for v in d[:, i]))
