"""Experiment: stage-1 pass 1 (the softmax normaliser) over mu_hi only
(INFLLM2_SELECT_P1HI=1) vs the default hi + lo, on full 131072-row layers:
selection mismatches over ALL (row, group) pairs, which side the float64
verifier agrees with, and the stage-1 time per layer."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072


def select(layer, q, cfg, hi_only):
    os.environ["INFLLM2_SELECT_P1HI"] = "1" if hi_only else "0"
    lib = _lib.load()
    geom = cfg.geometry()
    n = q.shape[0]
    kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
    sel = torch.empty((n, 2, cfg.max_selected), dtype=torch.int32, device="cuda")
    wsb = lib.infllm2_select_workspace_bytes(ctypes.byref(geom), n, 32, 2, 128, layer.length, 0)
    ws = P.sparse._workspace(torch.device("cuda", 0), wsb)
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.infllm2_select(ctypes.byref(geom), q.data_ptr(), q.stride(0), n, 0, 32, 2, 128, fine.data_ptr(),
                                      hi.data_ptr(), lo.data_ptr(), mcap, layer.length, sel.data_ptr(), None,
                                      ws.data_ptr(), ws.numel(), 0, st), "select")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sel, min(ts)


for top_k in (16, 64):
    for seed in (1, 2):
        cfg = P.SparseAttentionConfig(top_k=top_k)
        g = torch.Generator(device="cuda").manual_seed(100 * top_k + seed)
        k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
        q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
        layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
        layer.append(k, v)
        s_full, t_full = select(layer, q, cfg, False)
        s_hi, t_hi = select(layer, q, cfg, True)
        diff = (s_full != s_hi).any(-1)
        rows = torch.nonzero(diff.any(-1)).flatten()
        agree_full = agree_hi = neither = 0
        for r in rows[:200].tolist():
            o, s_ex = P.two_stage_attention(q[r:r + 1], layer, cfg, r, exact=True, return_selection=True)
            for gg in range(2):
                if not diff[r, gg]:
                    continue
                if torch.equal(s_ex[0, gg], s_full[r, gg]):
                    agree_full += 1
                elif torch.equal(s_ex[0, gg], s_hi[r, gg]):
                    agree_hi += 1
                else:
                    neither += 1
        print(f"L={L} k={top_k} seed={seed}: stage1 hi+lo {t_full:.2f} ms, p1-hi-only {t_hi:.2f} ms; "
              f"mismatching (row, group) pairs {int(diff.sum())} of {L * 2}; f64 verifier agrees with "
              f"hi+lo {agree_full}, hi-only {agree_hi}, neither {neither}", flush=True)
        del k, v, q, layer
