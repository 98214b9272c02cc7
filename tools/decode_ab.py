"""configs[3] decode step timing alone (bench.run_decode), for A/B runs:
  python tools/decode_ab.py [--layers 32] [--decode-seqs 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2506_07900_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=bench.SEQ)
ap.add_argument("--layers", type=int, default=bench.LAYERS)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--decode-seqs", type=int, default=8)
ap.add_argument("--decode-microbatches", type=int, default=1)
args = ap.parse_args()
dev = torch.device("cuda", 0)
cfg = P.SparseAttentionConfig(top_k=16)
res = bench.run_decode(args, P, cfg, 1, 0, dev, lambda: torch.cuda.synchronize(dev), None)
print(json.dumps({k: res[k] for k in ("ms_per_step", "us_per_token", "microbatches")} | {"roofline_frac": res["roofline"]["frac"],
                  "e2e_ms": res["e2e"]["ms_per_step"]}))
