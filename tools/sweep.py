"""BASELINE configs[4]: one InfLLM v2 layer, prefill over L in 4K..128K and
top-k in 8..64, for the MiniCPM4-8B attention shape (32 q / 2 KV heads,
d = 128) and the MiniCPM4-0.5B shape (16 q / 2 KV heads, d = 64; the
reference has no 0.5B config, SURVEY F17 - this is the public model card's
attention geometry).  Reports ms per layer (CUDA events, after warm-up),
tok/s for a 32-layer stack, the split stage-1 / stage-2 time, and whether the
layer is in the dense regime (every row selects every block: ceil(L/m) - |F|
<= k).  Usage: python tools/sweep.py [--quick] > profiles/r1_sweep.md
"""

import argparse
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_07900_b200 as P  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402
from paper_2506_07900_b200.sparse import _ptr, _stream, _workspace  # noqa: E402

SHAPES = {"8B": (32, 2, 128), "0.5B": (16, 2, 64)}


def time_layer(hq, hkv, d, L, k, reps=3, attend_too=True):
    cfg = P.SparseAttentionConfig(top_k=k)
    g = torch.Generator(device="cuda").manual_seed(L + k)
    q = torch.randn((L, hq, d), generator=g, device="cuda").to(torch.bfloat16)
    kk = torch.randn((L, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    vv = torch.randn((L, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(hkv, d, cfg, capacity=L)
    layer.append(kk, vv)
    lib = _lib.load()
    geom = cfg.geometry()
    sel = torch.empty((L, hkv, cfg.max_selected), dtype=torch.int32, device="cuda")
    out = torch.empty((L, hq, d), dtype=torch.bfloat16, device="cuda")
    kc, vc, cap, fine, hi, lo, mcap = layer._device_args()
    ws_bytes = lib.infllm2_select_workspace_bytes(ctypes.byref(geom), L, hq, hkv, d, L, 0)
    ws = _workspace(torch.device("cuda"), ws_bytes)
    st = _stream(torch.device("cuda"))

    def select():
        _lib.check(lib.infllm2_select(ctypes.byref(geom), _ptr(q), hq * d, L, 0, hq, hkv, d, _ptr(fine), _ptr(hi),
                                      _ptr(lo), mcap, L, _ptr(sel), None, _ptr(ws), ws.numel(), 0, st), "select")

    dense_path = hq // hkv == 16 and d == 128 and lib.infllm2_dense_regime(ctypes.byref(geom), L, 0, L) == 1

    def attend():
        if dense_path:      # what two_stage_attention runs below the sparsity threshold
            _lib.check(lib.infllm2_dense_attend(ctypes.byref(geom), _ptr(q), hq * d, L, 0, hq, hkv, d, _ptr(kc),
                                                _ptr(vc), cap, L, _ptr(out), None, 0, st), "dense attend")
            return
        _lib.check(lib.infllm2_attend(ctypes.byref(geom), _ptr(q), hq * d, L, 0, hq, hkv, d, _ptr(kc), _ptr(vc), cap, L,
                                      _ptr(sel), _ptr(out), None, 0, st), "attend")

    if not attend_too:      # stage 1 only (e.g. timing experiments that leave the selection invalid)
        attend = lambda: None  # noqa: E731
    for _ in range(2):
        select()
        attend()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_sel = t_att = 0.0
    for _ in range(reps):
        e[0].record()
        select()
        e[1].record()
        attend()
        e[2].record()
        torch.cuda.synchronize()
        t_sel += e[0].elapsed_time(e[1])
        t_att += e[1].elapsed_time(e[2])
    n_forced = cfg.n_init_blocks + cfg.n_local_blocks
    dense = -(-L // cfg.block_size) - n_forced <= k
    return t_sel / reps, t_att / reps, dense


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--shapes", default="8B,0.5B")
    ap.add_argument("--lengths", default="")
    ap.add_argument("--topks", default="8,16,32,64")
    args = ap.parse_args()
    lengths = [4096, 16384, 65536] if args.quick else [4096, 8192, 16384, 32768, 65536, 131072]
    if args.lengths:
        lengths = [int(x) for x in args.lengths.split(",")]
    ks = [int(x) for x in args.topks.split(",")]
    print("| shape | L | top-k | dense regime | stage 1 ms | stage 2 ms | ms/layer | tok/s (32 layers) |")
    print("|---|---|---|---|---|---|---|---|")
    for name, (hq, hkv, d) in SHAPES.items():
        if name not in args.shapes.split(","):
            continue
        for L in lengths:
            for k in ks:
                ts, ta, dense = time_layer(hq, hkv, d, L, k)
                ms = ts + ta
                print(f"| {name} | {L} | {k} | {'yes' if dense else 'no'} | {ts:.3f} | {ta:.3f} | {ms:.3f} | "
                      f"{L / (32 * ms / 1e3):,.0f} |", flush=True)
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
