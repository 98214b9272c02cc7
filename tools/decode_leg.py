"""Run only bench.py's decode leg (configs[3]) and print its us/token:
python tools/decode_leg.py [--steps K --warmup W ...] (bench.py's flags)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_07900_b200 as P  # noqa: E402

sys.argv = [sys.argv[0]] + sys.argv[1:]
args = bench.parse()
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
cfg = P.SparseAttentionConfig(top_k=16)
res = bench.run_decode(args, P, cfg, 1, 0, dev, lambda: torch.cuda.synchronize(dev), None)
print(json.dumps({"us_per_token": res["us_per_token"], "e2e_us_per_token": res["e2e"]["us_per_token"],
                  "ms_per_step": res["ms_per_step"],
                  "frac": res["roofline"]["frac"], "early_env": os.environ.get("INFLLM2_DECODE_NOEARLY")}))
