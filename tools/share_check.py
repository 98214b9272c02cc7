"""attend_share.cu vs attend_tc.cu on one prefill layer: run with
INFLLM2_ATTEND_SHARE=0 and without, same inputs; `--compare` diffs the two saved
outputs/LSEs and checks sampled rows against the float64 verifier."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
tag = "off" if os.environ.get("INFLLM2_ATTEND_SHARE") == "0" else "on"
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(3)
q = torch.randn((L, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(2, 128, cfg, capacity=L)
layer.append(k, v)
out, sel, lse = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                      out_dtype=torch.float32)
lib = _lib.load()
geom = cfg.geometry()
kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
st = torch.cuda.current_stream().cuda_stream
o2 = torch.empty((L, 32, 128), dtype=torch.bfloat16, device="cuda")
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.infllm2_attend(ctypes.byref(geom), q.data_ptr(), q.stride(0), L, 0, 32, 2, 128, kc.data_ptr(),
                                  vc.data_ptr(), cap, L, sel.data_ptr(), o2.data_ptr(), None, 0, st), "attend")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"[{tag}] stage 2 at L={L}: {min(ts[1:]):.3f} ms")
torch.save({"out": out.cpu(), "lse": lse.cpu(), "sel": sel.cpu()}, f"/tmp/share_{tag}.pt")
if "--compare" in sys.argv and tag == "on":
    ref = torch.load("/tmp/share_off.pt")
    assert torch.equal(ref["sel"], sel.cpu())
    d = (ref["out"] - out.cpu()).abs()
    dl = (ref["lse"] - lse.cpu()).abs()
    print(f"max |out_share - out_tc| = {d.max().item():.3e} (rows >= 256: {d[256:].max().item():.3e}, "
          f"rows < 256: {d[:256].max().item():.3e}); max |dLSE| = {dl.max().item():.3e}")
    rows = torch.tensor([256, 257, 300, 1023, 4096, 5000, L // 2 + 3, L - 4, L - 1])
    ex, _, exl = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                       out_dtype=torch.float32, exact=True)
    for name, o, l in (("share", out.cpu(), lse.cpu()), ("tc", ref["out"], ref["lse"])):
        e = (o[rows] - ex.cpu()[rows]).abs()
        bar = 1e-3 + 1e-2 * ex.cpu()[rows].abs()
        el = (l[rows] - exl.cpu()[rows]).abs().max().item()
        print(f"{name}: max |out - f64| = {e.max().item():.3e}, within bar: {bool((e <= bar).all())}, "
              f"max |dLSE| vs f64 = {el:.3e}")
