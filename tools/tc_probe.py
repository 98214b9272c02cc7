"""GPU probe: tensor-core kernels vs the float64 CUDA-core verifier, plus per-kernel timings.

Run on the GPU box:  python tools/tc_probe.py [L ...]
"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402
from inputs import make_qkv  # noqa: E402


def timed_split(layer, q, cfg, reps=3):
    lib = _lib.load()
    geom = cfg.geometry()
    dev = layer.device
    n = q.shape[0]
    kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
    sel = torch.empty((n, 2, cfg.max_selected), dtype=torch.int32, device=dev)
    out = torch.empty((n, 32, 128), dtype=torch.bfloat16, device=dev)
    wsb = lib.infllm2_select_workspace_bytes(ctypes.byref(geom), n, 32, 2, 128, layer.length, 0)
    ws = P.sparse._workspace(dev, wsb)
    st = torch.cuda.current_stream().cuda_stream
    ts, ta = [], []
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        _lib.check(lib.infllm2_select(ctypes.byref(geom), q.data_ptr(), q.stride(0), n, 0, 32, 2, 128, fine.data_ptr(),
                                      hi.data_ptr(), lo.data_ptr(), mcap, layer.length, sel.data_ptr(), None,
                                      ws.data_ptr(), ws.numel(), 0, st), "select")
        e[1].record()
        _lib.check(lib.infllm2_attend(ctypes.byref(geom), q.data_ptr(), q.stride(0), n, 0, 32, 2, 128, kc.data_ptr(),
                                      vc.data_ptr(), cap, layer.length, sel.data_ptr(), out.data_ptr(), None, 0, st),
                   "attend")
        e[2].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
        ta.append(e[1].elapsed_time(e[2]))
    return min(ts), min(ta)


def main():
    lengths = [int(x) for x in sys.argv[1:]] or [256, 2048, 8192, 32768]
    for L in lengths:
        cfg = P.SparseAttentionConfig(top_k=16)
        q, k, v = make_qkv(5, L, L, 32, 2, 128)
        layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
        layer.append(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda())
        qd = torch.from_numpy(q).cuda()
        o2, s2, l2 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True,
                                           out_dtype=torch.float32)
        torch.cuda.synchronize()
        if L <= 8192:
            o1, s1, l1 = P.two_stage_attention(qd, layer, cfg, 0, return_selection=True, return_lse=True,
                                               out_dtype=torch.float32, exact=True)
            diff = (s1 != s2).any(-1)
            do = (o1 - o2).abs()
            rel = (do / (o1.abs() + 1e-3)).max().item()
            print(f"L={L} sel mismatches {int(diff.sum())}/{diff.numel()}  max|dO|={do.max().item():.2e} "
                  f"maxrel={rel:.2e} max|dLSE|={(l1 - l2).abs().max().item():.2e}", flush=True)
            if diff.any():
                for i, g in diff.nonzero()[:3].tolist():
                    print("  ", i, g, s1[i, g].tolist(), s2[i, g].tolist())
        ts, ta = timed_split(layer, qd, cfg)
        print(f"L={L} select {ts:.3f} ms  attend {ta:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
