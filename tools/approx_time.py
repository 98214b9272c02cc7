import sys, torch
sys.path.insert(0, ".")
import paper_2506_07900_b200 as P
L = 131072
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L); layer.append(k, v)
for mode in ("exact", "approx", "exact", "approx"):
    P.two_stage_attention(q, layer, cfg, 0, lse=mode); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): P.two_stage_attention(q, layer, cfg, 0, lse=mode)
    e1.record(); torch.cuda.synchronize()
    print(mode, "ms/layer (select+attend)", e0.elapsed_time(e1) / 3)
