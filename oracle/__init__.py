"""CPU oracle — test infrastructure only (see infllm2_oracle.py header)."""
