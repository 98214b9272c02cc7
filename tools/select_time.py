"""Stage-1 time per 128K layer (CUDA events, best of 4) and a checksum of the
selection, for A/B runs of select_tc variants (INFLLM2_LIB_PATH)."""
import ctypes
import hashlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
top_k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = P.SparseAttentionConfig(top_k=top_k)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
layer.append(k, k)
lib = _lib.load()
geom = cfg.geometry()
kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
sel = torch.empty((L, 2, cfg.max_selected), dtype=torch.int32, device="cuda")
wsb = lib.infllm2_select_workspace_bytes(ctypes.byref(geom), L, 32, 2, 128, L, 0)
ws = P.sparse._workspace(torch.device("cuda", 0), wsb)
st = torch.cuda.current_stream().cuda_stream
ts = []
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.infllm2_select(ctypes.byref(geom), q.data_ptr(), q.stride(0), L, 0, 32, 2, 128, fine.data_ptr(),
                                  hi.data_ptr(), lo.data_ptr(), mcap, L, sel.data_ptr(), None, ws.data_ptr(),
                                  ws.numel(), 0, st), "select")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
h = hashlib.sha256(sel.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"stage 1 L={L} k={top_k}: {min(ts):.3f} ms (reps {['%.2f' % t for t in ts]}) selection sha {h}", flush=True)
