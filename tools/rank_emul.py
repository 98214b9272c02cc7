"""Per-rank work of the query-sharded prefill at N ranks, emulated on one GPU:
rank r's two zig-zag chunks of a 128K, 32-layer step (select + attend on their
own streams after the layer's fused append), timed with CUDA events.  The
all-gather is not included (NVLink, overlapped on a side stream in the bench).
Prints ms per step for each emulated rank and the scaling efficiency the
slowest rank implies against the N = 1 step: t1 / (N * max_r t_r)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import sharding as S  # noqa: E402

L, LAYERS, HQ, HKV, D = 131072, int(sys.argv[2]) if len(sys.argv) > 2 else 8, 32, 2, 128
NS = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
cfg = P.SparseAttentionConfig(top_k=16)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(5)
q = torch.randn((L, HQ, D), generator=g, device=dev).to(torch.bfloat16)
caches = []
for layer in range(LAYERS):
    k = torch.randn((L, HKV, D), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((L, HKV, D), generator=g, device=dev).to(torch.bfloat16)
    c = P.BlockizedLayerCache(HKV, D, cfg, capacity=L, device=dev)
    c.append(k, v)
    caches.append((c, k, v))
streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]


def rank_step(chunks):
    cur = torch.cuda.current_stream(dev)
    for c, k, v in caches:
        c.truncate(0)
        c.append(k, v)                        # the fused append + compress of the full layer
        for (lo, hi), st in zip(chunks, streams):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                P.two_stage_attention(q[lo:hi], c, cfg, lo)
        for st in streams:
            cur.wait_stream(st)


t1 = None
for n in NS:
    times = []
    for r in range(n):
        chunks = S.zigzag_chunks(L, n, r)
        rank_step(chunks)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            rank_step(chunks)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 2 * 32 / LAYERS)
    if n == 1:
        t1 = times[0]
    eff = t1 / (n * max(times)) if t1 else float("nan")
    print(f"N={n}: per-rank ms per 32-layer step min {min(times):.1f} max {max(times):.1f}; "
          f"implied efficiency vs N=1 {eff:.3f}", flush=True)
