"""Stage-1 time per 128K layer at top-k 16/32/64 (8B shape), for A/B of top-k variants."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ".")
from sweep import time_layer  # noqa: E402
for k in (16, 32, 64):
    ts, ta, _ = time_layer(32, 2, 128, 131072, k, attend_too=False)
    print(sys.argv[1] if len(sys.argv) > 1 else "lib", f"k={k} stage 1 {ts:.3f} ms")
