"""Full-layer selection census at BASELINE's headline size: the tensor-core
stage 1 vs the float64 CUDA-core verifier (exact=True) on EVERY (row, group)
pair of a 131072-row layer; mismatching pairs are re-scored by the CPU oracle
(float64 dots and the reference's float32 sgemv shape) with their margins."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from oracle import infllm2_oracle as O  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
for top_k in (16, 64):
    cfg = P.SparseAttentionConfig(top_k=top_k)
    g = torch.Generator(device="cuda").manual_seed(1_000_003 + top_k)   # the test_config2 layer
    k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(k, v)
    s_tc = P.two_stage_attention(q, layer, cfg, 0, return_selection=True)[1]
    torch.cuda.synchronize()
    t0 = time.time()
    s_x = torch.cat([P.two_stage_attention(q[i:i + 8192], layer, cfg, i, return_selection=True, exact=True)[1]
                     for i in range(0, L, 8192)])
    torch.cuda.synchronize()
    t_x = time.time() - t0
    bad = torch.nonzero((s_tc != s_x).any(-1)).cpu().numpy()
    kh, vh = k.float().cpu().numpy(), v.float().cpu().numpy()
    fine = O.window_means(kh, 32, 16)
    geom = O.Geometry(top_k=top_k)
    tc_f64 = tc_sg = x_f64 = 0
    margins = []
    for r, gg in bad:
        qr = q[r:r + 1].float().cpu().numpy()
        f = O.two_stage_attention(qr, kh, vh, fine, geom, int(r), keep_scores=True)
        sg = O.two_stage_attention(qr, kh, vh, fine, geom, int(r), dot="sgemv")
        bs = [x[2] for x in f.scores if x[1] == gg][0]
        margins.append(f.margins[0, gg] / bs.max())
        tc_f64 += np.array_equal(s_tc[r, gg].cpu().numpy(), f.selection[0, gg])
        x_f64 += np.array_equal(s_x[r, gg].cpu().numpy(), f.selection[0, gg])
        tc_sg += np.array_equal(s_tc[r, gg].cpu().numpy(), sg.selection[0, gg])
    m = np.array(margins) if margins else np.zeros(1)
    print(f"L={L} k={top_k}: {len(bad)} of {2 * L} (row, group) pairs differ between the tensor-core and the "
          f"float64 verifier (verifier ran {t_x:.1f} s); of those the CPU float64 oracle agrees with the verifier "
          f"{x_f64}, with the tensor cores {tc_f64}; the tensor cores agree with the sgemv oracle {tc_sg}; relative "
          f"float64 margins max {m.max():.2e}, median {np.median(m):.2e}", flush=True)
    del k, v, q, layer, s_tc, s_x
