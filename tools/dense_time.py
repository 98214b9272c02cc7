"""Time infllm2_dense_attend (causal GQA, 32 q heads / 2 KV groups, D = 128) over
a full prefill of L rows, with the library named by INFLLM2_LIB_PATH:
  INFLLM2_LIB_PATH=variants/x.so python tools/dense_time.py [L ...]
Prints ms per call and algorithmic causal TF/s (4 * D * HQ * L(L+1)/2 flops)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402
from paper_2506_07900_b200.sparse import _ptr, _stream  # noqa: E402

lib = _lib.load()
for L in [int(a) for a in sys.argv[1:]] or [4096, 16384, 32768]:
    cfg = P.SparseAttentionConfig(top_k=64)
    g = torch.Generator(device="cuda").manual_seed(L)
    q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    kk = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
    layer.append(kk, kk)
    kc, vc, cap, *_ = layer._device_args()
    out = torch.empty((L, 32, 128), dtype=torch.bfloat16, device="cuda")
    geom = cfg.geometry()
    st = _stream(torch.device("cuda"))

    def run():
        _lib.check(lib.infllm2_dense_attend(ctypes.byref(geom), _ptr(q), 32 * 128, L, 0, 32, 2, 128, _ptr(kc),
                                            _ptr(vc), cap, L, _ptr(out), None, 0, st), "dense")
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{os.environ.get('INFLLM2_LIB_PATH', 'in-tree')} L={L}: {ms:.3f} ms  {4 * 128 * 32 * L * (L + 1) / 2 / ms / 1e9:.0f} TF/s")
