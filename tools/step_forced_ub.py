"""Step-level upper bound of forced-block sharing in stage 2 (power-capped
context): a 32-layer 128K prefill (select + attend per layer, caches filled
once) timed with stage 2 fed (a) each layer's real selection and (b) the same
selection with the forced blocks (0, qb-1, qb) removed from rows >= 4096."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
NL = int(sys.argv[2]) if len(sys.argv) > 2 else 32
HQ, HKV, D = 32, 2, 128
cfg = P.SparseAttentionConfig(top_k=16)
geom = cfg.geometry()
lib = _lib.load()
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
gen = torch.Generator(device=dev)
layers = []
for layer in range(NL):
    gen.manual_seed(1_000_003 * layer + 17)
    q = torch.randn((L, HQ, D), generator=gen, device=dev).to(torch.bfloat16)
    k = torch.randn((L, HKV, D), generator=gen, device=dev).to(torch.bfloat16)
    v = torch.randn((L, HKV, D), generator=gen, device=dev).to(torch.bfloat16)
    c = P.BlockizedLayerCache(HKV, D, cfg, capacity=L, device=dev)
    c.append(k, v)
    del k, v
    layers.append((q, c))
sel_buf = torch.empty((L, HKV, cfg.max_selected), dtype=torch.int32, device=dev)
out = torch.empty((L, HQ, D), dtype=torch.bfloat16, device=dev)
wsb = lib.infllm2_select_workspace_bytes(ctypes.byref(geom), L, HQ, HKV, D, L, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)


def select(q, c, sel):
    kc, vc, cap, fine, hi, lo, mcap = c._device_args()
    _lib.check(lib.infllm2_select(ctypes.byref(geom), q.data_ptr(), q.stride(0), L, 0, HQ, HKV, D, fine.data_ptr(),
                                  hi.data_ptr(), lo.data_ptr(), mcap, c.length, sel.data_ptr(), None, ws.data_ptr(),
                                  ws.numel(), 0, stream.cuda_stream), "select")


def attend(q, c, sel):
    kc, vc, cap, fine, hi, lo, mcap = c._device_args()
    _lib.check(lib.infllm2_attend(ctypes.byref(geom), q.data_ptr(), q.stride(0), L, 0, HQ, HKV, D, kc.data_ptr(),
                                  vc.data_ptr(), cap, c.length, sel.data_ptr(), out.data_ptr(), None, 0,
                                  stream.cuda_stream), "attend")


pos = torch.arange(L, device=dev).view(L, 1, 1)
real, mod = [], []
big = torch.iinfo(torch.int32).max
for q, c in layers:
    s = torch.empty_like(sel_buf)
    select(q, c, s)
    real.append(s)
    forced = ((s == 0) | (s == pos // 64) | (s == pos // 64 - 1)) & (pos >= 4096)
    s2 = torch.where(forced | (s < 0), torch.full_like(s, big), s).sort(dim=-1).values
    mod.append(torch.where(s2 == big, torch.full_like(s2, -1), s2).contiguous())
torch.cuda.synchronize()
for name, sels in (("real", real), ("forced removed", mod), ("real", real), ("forced removed", mod)):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for (q, c), s in zip(layers, sels):
            select(q, c, sel_buf)
            attend(q, c, s)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{name}: {ms:.1f} ms per {NL}-layer step ({L / (ms / 1e3):.0f} tok/s)", flush=True)
