"""Two-micro-batch decode pipeline probe: S sequences split in MB halves, each
on its own stream (layer l+1 after layer l per micro-batch), with micro-batch
m's chain started `m * offset` SM cycles late (torch.cuda._sleep) so one's
means stream runs during the other's dependent tail.  Prints us per layer-step
(all sequences) for each offset.

usage: python tools/decode_mb.py [S] [L] [NL] [MB] [offsets_cycles,...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
NL = int(sys.argv[3]) if len(sys.argv) > 3 else 8
MB = int(sys.argv[4]) if len(sys.argv) > 4 else 2
OFFS = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [0, 10000, 20000, 30000, 40000]
REPS = 10
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
bounds = [(m * S // MB, (m + 1) * S // MB) for m in range(MB)]
batches = [[] for _ in range(MB)]
for layer in range(NL):
    caches = []
    for s in range(S):
        c = P.BlockizedLayerCache(2, 128, cfg, capacity=L + 512)
        c.append(torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16),
                 torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16))
        caches.append(c)
    for m, (lo, hi) in enumerate(bounds):
        b = P.DecodeBatch(caches[lo:hi], cfg, concurrent=MB)
        b.reserve(400)
        batches[m].append(b)
allb = [b for row in batches for b in row]
q = torch.randn((NL, S, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
kn = torch.randn((NL, S, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
bound = L + 400
streams = [torch.cuda.Stream() for _ in range(MB)]


def step(offset, bookkeep=True):
    cur = torch.cuda.current_stream()
    for m, st in enumerate(streams):
        st.wait_stream(cur)
        lo, hi = bounds[m]
        with torch.cuda.stream(st):
            if m and offset:
                torch.cuda._sleep(m * offset)
            for i in range(NL):
                batches[m][i].step(q[i, lo:hi], kn[i, lo:hi], kn[i, lo:hi], max_len=bound, bookkeep=bookkeep)
    for st in streams:
        cur.wait_stream(st)


side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
for off in OFFS:
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        step(off)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=side):
            step(off, bookkeep=False)
    torch.cuda.synchronize()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(REPS):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    for b in allb:
        b.advance(REPS + 3)
    us = e0.elapsed_time(e1) * 1e3 / REPS
    # the sleep itself: one kernel of `offset` cycles at the start of each step
    print(f"S={S} MB={MB} NL={NL} offset={off} cycles: {us:.1f} us per step, {us / NL:.2f} us per layer-step "
          f"(all sequences), {us / NL * 32 / S:.1f} us/token at 32 layers")
