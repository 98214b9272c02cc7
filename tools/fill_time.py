"""Time the per-layer cache fill of the prefill bench (all-gather + append + compress of one 128K layer)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2506_07900_b200 as P
from paper_2506_07900_b200 import sharding as S
L = 131072
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
k = [torch.randn((L // 2, 2, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(2)]
v = [torch.randn((L // 2, 2, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(2)]
cache = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
for _ in range(3): S.fill_layer_cache(cache, k, v, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): S.fill_layer_cache(cache, k, v, 1)
e1.record(); torch.cuda.synchronize()
print("fill_layer_cache ms", e0.elapsed_time(e1) / 10)
import time
t = time.perf_counter()
for _ in range(10): S.fill_layer_cache(cache, k, v, 1)
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t) * 100)
