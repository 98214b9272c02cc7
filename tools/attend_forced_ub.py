"""Upper bound of forced-block sharing in stage 2: time the attend kernel over
a 128K layer with the full selection and with the forced blocks (init block 0,
local blocks qb-1, qb) removed from every row's list (what a per-query-block
shared pass would leave per row)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
layer.append(k, v)
out, sel = P.two_stage_attention(q, layer, cfg, 0, return_selection=True)
pos = torch.arange(L, device="cuda").view(L, 1, 1)
qb = pos // 64
forced = ((sel == 0) | (sel == qb) | (sel == qb - 1)) & (pos >= 4096)   # early rows keep theirs (never empty)
big = torch.iinfo(torch.int32).max
s2 = torch.where(forced | (sel < 0), torch.full_like(sel, big), sel).sort(dim=-1).values
s2 = torch.where(s2 == big, torch.full_like(s2, -1), s2).contiguous()
lib = _lib.load()
geom = cfg.geometry()
kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
st = torch.cuda.current_stream().cuda_stream
for name, s in (("full selection", sel), ("forced removed", s2), ("full selection", sel)):
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.infllm2_attend(ctypes.byref(geom), q.data_ptr(), q.stride(0), L, 0, 32, 2, 128, kc.data_ptr(),
                                      vc.data_ptr(), cap, L, s.data_ptr(), out.data_ptr(), None, 0, st), "attend")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name}: stage 2 at L={L}: {min(ts[1:]):.3f} ms (reps {['%.3f' % t for t in ts]})")
