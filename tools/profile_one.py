"""One prefill forward (select + attend) at a given length, for ncu captures."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2506_07900_b200 as P

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
layer.append(k, v)
for _ in range(2):
    P.two_stage_attention(q, layer, cfg, 0)
torch.cuda.synchronize()
print("done")
