"""Per-CTA cycle split of attend_tc (needs a -DATT_PROFILE variant build):
  tools/build_variant.sh variants/aprof.so paper_2506_07900_b200/csrc/attend_tc.cu -DATT_PROFILE
  INFLLM2_LIB_PATH=variants/aprof.so python tools/attend_profile.py
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

shape = (16, 2, 64) if os.environ.get("AB_SHAPE") == "0.5B" else (32, 2, 128)
print("shape", shape, "select, attend ms:", time_layer(*shape, int(os.environ.get("AB_LEN", "131072")),
                                                      int(os.environ.get("AB_TOPK", "16")), reps=1))
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (160 * 24))()
_lib.load().infllm2_debug_attend_cycles(buf, 160 * 24)
a = np.frombuffer(buf, dtype=np.int64).reshape(160, 24)[:148].astype(np.float64).mean(axis=0)
names = {0: "QK total", 2: "QK s_empty wait", 3: "PV total", 4: "PV v_full wait", 5: "PV p_full wait",
         7: "softmax total", 1: "softmax in tile loops", 8: "softmax s_full wait", 15: "softmax S TMEM ld+wait",
         9: "softmax vote barrier", 10: "softmax need path", 11: "softmax p_empty wait",
         6: "softmax P fence+arrive", 19: "softmax sel/mask", 20: "softmax P compute+store",
         16: "softmax item sel take", 17: "softmax st_empty wait", 18: "softmax stats write", 14: "K TMA total", 12: "K TMA k_empty wait", 13: "V TMA v_empty wait"}
for i, n in names.items():
    tot = a[0] if i in (0, 2) else a[3] if i in (3, 4, 5) else a[14] if i in (12, 13, 14) else a[7]
    print(f"{n:24s} {a[i] / tot * 100:6.1f} %")
