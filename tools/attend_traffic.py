"""Stage-2 time per 128K layer (CUDA events, 3 reps) for A/B of L2 policies;
run under ncu for DRAM bytes."""
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
lib = _lib.load()
geom = cfg.geometry()
kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
st = torch.cuda.current_stream().cuda_stream
ts = []
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.infllm2_attend(ctypes.byref(geom), q.data_ptr(), q.stride(0), L, 0, 32, 2, 128, kc.data_ptr(),
                                  vc.data_ptr(), cap, L, sel.data_ptr(), out.data_ptr(), None, 0, st), "attend")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"stage 2 at L={L}: {min(ts[1:]):.3f} ms (reps {['%.3f' % t for t in ts]})")
