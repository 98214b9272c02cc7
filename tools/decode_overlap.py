"""Do two decode micro-batches on separate streams overlap?  Times 32 layer
steps of micro-batch A alone, then A and B concurrently (graph-captured)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402

L, S, layers, mb = 131072, 8, 32, 2
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
share = int(sys.argv[1]) if len(sys.argv) > 1 else 2
bat = [[], []]
for layer in range(layers):
    cs = []
    for s in range(S):
        c = P.BlockizedLayerCache(2, 128, cfg, capacity=L + 256)
        c.append(torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16),
                 torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16))
        cs.append(c)
    for m in range(mb):
        b = P.DecodeBatch(cs[m * 4:(m + 1) * 4], cfg, concurrent=share)
        b.reserve(200)
        bat[m].append(b)
q = torch.randn((4, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
kn = torch.randn((4, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
st = [torch.cuda.Stream(), torch.cuda.Stream()]


def run(which):
    cur = torch.cuda.current_stream()
    for m in which:
        st[m].wait_stream(cur)
        with torch.cuda.stream(st[m]):
            for i in range(layers):
                bat[m][i].step(q, kn, kn, max_len=L + 256, bookkeep=False)
    for m in which:
        cur.wait_stream(st[m])


for which in ([0], [1], [0, 1]):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        run(which)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=side):
            run(which)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"share={share} micro-batches {which}: {e0.elapsed_time(e1) / 10 * 1e3 / layers:.1f} us per layer", flush=True)
