"""Shared loaders for the committed golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from inputs import digest
from cases import CASES, build_inputs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return meta, {k: z[k] for k in z.files if k != "meta"}


def case_names():
    return sorted(CASES)


def case_inputs(meta):
    q, k, v = build_inputs(meta["seed"], meta["length"], meta["n_q"], meta["hq"],
                           meta["hkv"], meta["d"], meta["scale"], meta["kind"])
    assert digest(q, k, v) == meta["input_sha"], "input generator drifted from the fixture"
    return q, k, v


def available() -> list[str]:
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
