"""One prefill forward (select + attend) at a given length, for ncu captures:
python tools/profile_one.py [L] [hq hkv d]   (default 32 q / 2 KV heads, d 128)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2506_07900_b200 as P

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
HQ, HKV, D = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (32, 2, 128)
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((L, HQ, D), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, HKV, D), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, HKV, D), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(HKV, D, cfg, capacity=L)
layer.append(k, v)
for _ in range(2):
    P.two_stage_attention(q, layer, cfg, 0)
torch.cuda.synchronize()
print("done")
