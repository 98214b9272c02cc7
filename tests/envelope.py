"""Measured error envelopes of the GPU parity tests.

Each parity test asserts its bar AND records the worst error it saw here; with
INFLLM2_ENVELOPE_LOG=<path> set, the records are appended to that file as JSON
lines (DESIGN.md §5 quotes them when setting the bars)."""

from __future__ import annotations

import json
import os


def record(test: str, **values) -> None:
    path = os.environ.get("INFLLM2_ENVELOPE_LOG")
    line = {"test": test, **{k: float(v) for k, v in values.items()}}
    print("envelope", json.dumps(line))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(line) + "\n")
