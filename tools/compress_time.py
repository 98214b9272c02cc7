"""K1 timing: one 131072-row prefill append into an empty blockized cache
(infllm2_append_compress: K/V rows in, fine + coarse means and the bf16 hi/lo
splits out) and a full re-sync pass (compress only), with CUDA events.
Algorithmic bytes: append = L*HKV*D*2 (K in) *2 (V) + same out + means
(nk + nc) * HKV * D * (4 + 2 + 2); compress-only = K read + means written."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
HKV, D = 2, 128
cfg = P.SparseAttentionConfig(top_k=16)
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((L, HKV, D), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((L, HKV, D), generator=g, device="cuda").to(torch.bfloat16)
layer = P.BlockizedLayerCache(HKV, D, cfg, capacity=L)
means_bytes = (L // 16 + L // 128) * HKV * D * (4 + 2 + 2)
REPS = 20
for what in ("append", "resync"):
    # back-to-back launches: the host enqueues faster than one launch runs, so
    # the events bracket GPU time (one launch alone would include the Python
    # call's ~30 us)
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(REPS):
            if what == "append":
                layer.length = layer._nk_valid = layer._nc_valid = 0     # empty the cache (no kernel)
                layer.append(k, v)
            else:
                layer._nk_valid = layer._nc_valid = 0
                layer._sync(0, L)
        e1.record()
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / REPS
    nbytes = (4 * L * HKV * D * 2 if what == "append" else L * HKV * D * 2) + means_bytes
    print(f"{what}: L={L} {t * 1e6:.1f} us per launch ({REPS} back to back), algorithmic {nbytes / 1e6:.1f} MB -> "
          f"{nbytes / t / 1e9:.0f} GB/s")
f, c = layer.rebuild_kernels()
assert torch.equal(layer.fine_means.contiguous(), f.contiguous())
assert torch.equal(layer.coarse_means.contiguous(), c.contiguous())
print("means == rebuild: ok")
