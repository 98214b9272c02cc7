"""Decode timing probe: S sequences x L cached tokens, a few layers; per-layer decode_step time."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2506_07900_b200 as P

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
NL = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
batches = []
for layer in range(NL):
    caches = []
    for s in range(S):
        c = P.BlockizedLayerCache(2, 128, cfg, capacity=L + 64)
        k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
        c.append(k, torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16))
        caches.append(c)
    batches.append(P.DecodeBatch(caches, cfg))
q = torch.randn((S, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
kn = torch.randn((S, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
for b in batches:
    b.step(q, kn, kn)
torch.cuda.synchronize()
reps = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    for b in batches:
        b.step(q, kn, kn)
e1.record(); torch.cuda.synchronize()
per_layer_us = e0.elapsed_time(e1) * 1e3 / (reps * NL)
nk = L // 16
bytes_layer = S * (2 * nk * 128 * 4 + 2 * 1216 * 128 * 2 * 2)
print(f"S={S} L={L}: {per_layer_us:.1f} us per layer-step; 32-layer step {per_layer_us*32/1e3:.3f} ms; "
      f"{per_layer_us*32/S:.1f} us/token aggregate; HBM {bytes_layer/per_layer_us/1e3:.0f} GB/s algorithmic")
