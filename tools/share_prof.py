"""Per-role wait split of attend_share_kernel (a role that rarely waits paces the kernel):
  tools/build_variant.sh variants/sprof.so paper_2506_07900_b200/csrc/attend_share.cu -DSHARE_PROF
  INFLLM2_LIB_PATH=variants/sprof.so AB_SHAPE=0.5B|8B AB_TOPK=16 python tools/share_prof.py"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from sweep import time_layer
shape = (16, 2, 64) if os.environ.get("AB_SHAPE") == "0.5B" else (32, 2, 128)
lib = ctypes.CDLL(os.environ["INFLLM2_LIB_PATH"])
print(shape, time_layer(*shape, 131072, int(os.environ.get("AB_TOPK", "16")), reps=1))
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (160 * 16))()
lib.infllm2_debug_share_cycles(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(160, 16)[:148].astype(np.float64).mean(axis=0)
names = {1: ("K prod ring_empty wait", 0), 3: ("V prod ring_empty wait", 2), 5: ("QK k_full wait", 4), 6: ("QK s_empty wait", 4),
         8: ("PV v_full wait", 7), 9: ("PV p_full wait", 7), 10: ("PV o_empty wait", 7), 12: ("softmax s_full wait", 11),
         13: ("softmax p_empty wait", 11), 15: ("epilogue o_full wait", 14)}
for i, (n, t) in names.items():
    print(f"{n:26s} {a[i] / a[t] * 100:6.1f} %   (total {a[t]/1e6:.2f} Mcyc)")
