"""Per-CTA cycle split of select_tc (needs a -DSEL_PROFILE variant build):
  tools/build_variant.sh variants/prof.so paper_2506_07900_b200/csrc/select_tc.cu -DSEL_PROFILE
  INFLLM2_LIB_PATH=variants/prof.so python tools/select_profile.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ".")
from sweep import time_layer  # noqa: E402
from paper_2506_07900_b200 import _lib  # noqa: E402

time_layer(32, 2, 128, int(os.environ.get("AB_LEN", "131072")), 16, reps=1, attend_too=False)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * (160 * 8))()
rc = lib.infllm2_debug_select_cycles(buf, 160 * 8)
a = np.frombuffer(buf, dtype=np.int64).reshape(160, 8)[:148].astype(np.float64)
# 3 launches were accumulated (2 warm-up + 1 timed): ratios only
names = ["epi total", "epi acc_full wait", "epi pass-1", "mma total", "mma mu_full wait", "mma acc_empty wait"]
for i, n in enumerate(names):
    print(f"{n:22s} {a[:, i].mean() / a[:, 0].mean() * 100:6.1f} % of epilogue total")
