"""Near-tie census of the tensor-core stage 1 at 131072 rows.

Candidate (row, group) pairs = those whose selection moves when pass 1 is
perturbed (mu_hi only, INFLLM2_SELECT_P1HI=1): the near-ties.  For each, the
CPU oracle (the reference's algorithm) gives the float64-dot selection, the
reference-shaped float32 sgemv selection, and the float64 margin between the
weakest chosen and strongest rejected block (relative to the block score).
Reports how many of ALL pairs the default path selects differently from the
float64 oracle and how close those ties were."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402
from oracle import infllm2_oracle as O  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072


def select(layer, q, cfg, hi_only):
    os.environ["INFLLM2_SELECT_P1HI"] = "1" if hi_only else "0"
    return P.two_stage_attention(q, layer, cfg, 0, return_selection=True)[1]


for top_k in (16, 64):
    cfg = P.SparseAttentionConfig(top_k=top_k)
    g = torch.Generator(device="cuda").manual_seed(100 * top_k + 1)
    k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(k, v)
    s_tc = select(layer, q, cfg, False)
    s_hi = select(layer, q, cfg, True)
    cand = torch.nonzero((s_tc != s_hi).any(-1)).cpu().numpy()
    kh, vh = k.float().cpu().numpy(), v.float().cpu().numpy()
    fine = O.window_means(kh, 32, 16)
    geom = O.Geometry(top_k=top_k)
    tc_np = s_tc.cpu().numpy()
    stats = dict(cand=len(cand), tc_ne_f64=0, tc_eq_sgemv_when_ne_f64=0, f64_ne_sgemv=0)
    margins = []
    for r, gg in cand:
        qr = q[r:r + 1].float().cpu().numpy()
        f = O.two_stage_attention(qr, kh, vh, fine, geom, int(r), keep_scores=True)
        sg = O.two_stage_attention(qr, kh, vh, fine, geom, int(r), dot="sgemv")
        bs = [x[2] for x in f.scores if x[1] == gg][0]
        rel = f.margins[0, gg] / bs.max()
        if not np.array_equal(tc_np[r, gg], f.selection[0, gg]):
            stats["tc_ne_f64"] += 1
            margins.append(rel)
            if np.array_equal(tc_np[r, gg], sg.selection[0, gg]):
                stats["tc_eq_sgemv_when_ne_f64"] += 1
        if not np.array_equal(f.selection[0, gg], sg.selection[0, gg]):
            stats["f64_ne_sgemv"] += 1
    m = np.array(margins) if margins else np.zeros(1)
    print(f"L={L} k={top_k}: {stats}; relative f64 margins of the TC!=f64 pairs: "
          f"max {m.max():.2e} median {np.median(m):.2e}", flush=True)
    del k, v, q, layer
