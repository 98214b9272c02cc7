"""Decode timing probe: S sequences x L cached tokens, NL layers; eager and CUDA-graph steps."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2506_07900_b200 as P

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
NL = int(sys.argv[3]) if len(sys.argv) > 3 else 4
REPS = 8
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
batches = []
for layer in range(NL):
    caches = []
    for s in range(S):
        c = P.BlockizedLayerCache(2, 128, cfg, capacity=L + 256)
        k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
        c.append(k, torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16))
        caches.append(c)
    b = P.DecodeBatch(caches, cfg)
    b.reserve(200)
    batches.append(b)
q = torch.randn((NL, S, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
kn = torch.randn((NL, S, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
bound = L + 200
def step(bookkeep=True):
    for i, b in enumerate(batches):
        b.step(q[i], kn[i], kn[i], max_len=bound, bookkeep=bookkeep)
step(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    step()
e1.record(); torch.cuda.synchronize()
eager = e0.elapsed_time(e1) * 1e3 / (REPS * NL)
graph = torch.cuda.CUDAGraph()
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_):
    step(); torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=s_):
        step(bookkeep=False)
torch.cuda.synchronize()
e0.record()
for _ in range(REPS):
    graph.replay()
e1.record(); torch.cuda.synchronize()
for b in batches:
    b.advance(REPS)
gr = e0.elapsed_time(e1) * 1e3 / (REPS * NL)
nk = L // 16
bytes_layer = S * (2 * nk * 128 * 4 + 2 * 1216 * 128 * 2 * 2)
for name, us in (("eager", eager), ("graph", gr)):
    print(f"{name}: S={S} L={L}: {us:.1f} us per layer-step; 32-layer step {us*32/1e3:.3f} ms; "
          f"{us*32/S:.1f} us/token aggregate; {bytes_layer/us/1e3:.0f} GB/s algorithmic")
