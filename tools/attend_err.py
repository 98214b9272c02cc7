"""Locate stage-2 tensor-core error vs the float64 CUDA-core path."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import paper_2506_07900_b200 as P
from inputs import make_qkv

for L in (256, 2048):
    cfg = P.SparseAttentionConfig(top_k=16)
    q, k, v = make_qkv(5, L, L, 32, 2, 128)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
    qd = torch.from_numpy(q).cuda()
    o1, s1, l1 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True, out_dtype=torch.float32, exact=True)
    o2, s2, l2 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True, out_dtype=torch.float32)
    dl = (l1 - l2).abs().cpu().numpy()
    do = (o1 - o2).abs().amax(-1).cpu().numpy()
    print(f"L={L} mean|dLSE| {dl.mean():.2e} max {dl.max():.2e}; mean max|dO| {do.mean():.2e}")
    i, h = np.unravel_index(dl.argmax(), dl.shape)
    print("  worst (row, head)", i, h, "lse", l1[i, h].item(), l2[i, h].item())
    print("  per-head mean dLSE", np.round(dl.mean(0), 5).tolist())
    print("  per-row-bucket mean dLSE", [float(np.round(dl[j:j+64].mean(), 5)) for j in range(0, L, max(64, L // 16))])
    # error vs number of rows attended
    nsel = (s1[:, :, :] >= 0).sum(-1).cpu().numpy()
    print("  rows<64 mean", dl[:64].mean(), " rows 64..127", dl[64:128].mean())
