"""Batched decode timing for the MiniCPM4-0.5B head geometry (16 q heads, 2 KV
heads, D = 64): the cluster kernel and the five-launch path (eager and
CUDA-graph replay) vs stepping every sequence through the prefill kernels.

    python tools/decode_05b.py [--seqs 8] [--len 131072] [--steps 20]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_07900_b200 as P  # noqa: E402

HQ, HKV, D = 16, 2, 64


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=8)
    ap.add_argument("--len", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--topk", type=int, default=16)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = P.SparseAttentionConfig(top_k=a.topk)
    S, L, n = a.seqs, a.len, a.steps
    extra = 8 * n + 32
    gen = torch.Generator(device="cuda").manual_seed(3)
    layers = []
    for _ in range(S):
        c = P.BlockizedLayerCache(HKV, D, cfg, capacity=L + extra)
        c.append(torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16),
                 torch.randn((L, HKV, D), generator=gen, device="cuda").to(torch.bfloat16))
        layers.append(c)
    q = torch.randn((S, HQ, D), generator=gen, device="cuda").to(torch.bfloat16)
    kn = torch.randn((S, HKV, D), generator=gen, device="cuda").to(torch.bfloat16)
    batch = P.DecodeBatch(layers, cfg)
    batch.reserve(extra)
    bound = L + extra

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3          # us per step

    res = {"seqs": S, "len": L, "top_k": a.topk}

    def measure(tag):
        res[f"{tag}_eager_us"] = timed(lambda: batch.step(q, kn, kn, max_len=bound), n)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                batch.step(q, kn, kn, max_len=bound, bookkeep=False)
        torch.cuda.synchronize()

        def replay():
            graph.replay()
            batch.advance(1)

        res[f"{tag}_graph_us"] = timed(replay, n)

    measure("fused")
    os.environ["INFLLM2_DECODE_LEGACY"] = "1"
    measure("five_launch")
    del os.environ["INFLLM2_DECODE_LEGACY"]
    res["per_sequence_us"] = timed(lambda: batch._step_per_sequence(q, kn, kn, False, False, None, True), n)
    nk = L // 16
    per_seq = HKV * nk * D * 4 + HKV * (a.topk + 3) * 64 * D * 2 * 2
    res["algorithmic_bytes_per_step"] = per_seq * S
    res["fused_graph_hbm_GBps"] = per_seq * S / (res["fused_graph_us"] * 1e-6) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
