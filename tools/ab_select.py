"""Time one 128K layer's stage 1 / stage 2 (8B shape, top-k 16) with the
library named by INFLLM2_LIB_PATH (default: the in-tree build), for A/B runs
of kernel variants built with tools/build_variant.sh:
  for v in base new; do INFLLM2_LIB_PATH=variants/$v.so python tools/ab_select.py $v; done
AB_STAGE1_ONLY=1 skips stage 2 (for experiments that leave the selection invalid).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ".")
from sweep import time_layer  # noqa: E402

L = int(os.environ.get("AB_LEN", "131072"))
ts, ta, _ = time_layer(32, 2, 128, L, 16, attend_too=os.environ.get("AB_STAGE1_ONLY") != "1")
print(sys.argv[1] if len(sys.argv) > 1 else "lib", f"stage 1 {ts:.3f} ms  stage 2 {ta:.3f} ms")
