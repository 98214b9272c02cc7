import sys, time, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests/golden')
import paper_2506_07900_b200 as P
from inputs import make_qkv
for L in (256, 2048, 8192):
    cfg = P.SparseAttentionConfig(top_k=16)
    q, k, v = make_qkv(5, L, L, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    o1, s1 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, exact=True)
    torch.cuda.synchronize(); t=time.time()
    o2, s2 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True)
    torch.cuda.synchronize(); dt=time.time()-t
    diff = (s1 != s2).any(-1)
    print(f"L={L} tc-vs-simt selection mismatches {int(diff.sum())}/{diff.numel()} time {dt*1e3:.1f}ms", flush=True)
    if diff.any():
        idx = diff.nonzero()[:3]
        for i, g in idx.tolist():
            print(i, g, s1[i, g].tolist(), s2[i, g].tolist())
