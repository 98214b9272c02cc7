"""One 128K layer's stage 1 only (8B shape, top-k 16), for ncu captures of
select_tc experiments (INFLLM2_SELECT_DBG) that leave the selection invalid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ".")
from sweep import time_layer  # noqa: E402
time_layer(32, 2, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 131072, 16, reps=1, attend_too=False)
