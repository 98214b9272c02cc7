"""Parity bars shared by the GPU tests, set at ~2x the measured
envelope (tests/envelope.py records it; profiles/r2_envelope.jsonl).

* OUT_ABS + OUT_REL*|ref|: float32 outputs of the tensor-core stage 2 (bf16
  softmax weights; convex-combination error ~2^-9 |V| / sqrt(rows)), measured
  max 8.4e-4 abs at 128K over 2048 (row, group) pairs;
* LSE_TC: natural-log LSE of the tensor-core paths vs float64, measured max
  1.3e-6 at 128K (the survey's bar is 1e-5);
* SPLIT_*: split_p=True (bf16 hi + lo weights), measured 2.2e-6 at 8K.
"""

OUT_ABS, OUT_REL = 1e-3, 1e-2
LSE_TC = 5e-6
SPLIT_ABS, SPLIT_REL = 2e-5, 1e-4
