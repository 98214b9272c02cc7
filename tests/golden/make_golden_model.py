"""Golden fixture for the model seam (forward(..., backend=...) / make_cache),
produced by the UNMODIFIED reference in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_model.py

A tiny seeded ``random_bundle`` (2 layers, 8 query / 2 KV heads, head_dim 8)
runs a 300-token prefill and then three single-token decode steps through
``deskinfer.model.forward`` with ``make_cache(bundle, backend)`` for both
backends (sparse: top_k=2, n_local_blocks=1 -> a real sparse regime).  The
fixture stores the config, the parameters, the tokens and every step's logits.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from deskinfer.model import ModelConfig, forward, random_bundle  # noqa: E402
from deskinfer.sparse import SparseAttentionConfig  # noqa: E402
from deskinfer.specdec import make_cache  # noqa: E402

CFG = dict(hidden_dim=64, n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=8, vocab_size=256,
           max_seq_len=4096, ffn_dim=128)
SPARSE = dict(top_k=2, n_local_blocks=1)


def main() -> None:
    cfg = ModelConfig(**CFG)
    bundle = random_bundle(cfg, seed=2506, scale=0.2)
    rng = np.random.default_rng(7900)
    tokens = rng.integers(0, cfg.vocab_size, size=303)
    out = {"tokens": tokens}
    for backend in ("dense", "sparse"):
        sc = SparseAttentionConfig(**SPARSE) if backend == "sparse" else None
        cache = make_cache(bundle, backend, sc)
        steps = [forward(bundle, tokens[:300], cache, backend=backend, sparse_config=sc).logits]
        for t in range(300, 303):
            steps.append(forward(bundle, tokens[t:t + 1], cache, backend=backend, sparse_config=sc).logits)
        out[f"logits_{backend}"] = np.concatenate(steps)
    for name, a in bundle.params.items():
        out["param:" + name] = a
    out["config"] = np.frombuffer(repr(CFG).encode(), dtype=np.uint8)
    out["sparse"] = np.frombuffer(repr(SPARSE).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "model_seam.npz"), **out)
    print("wrote model_seam.npz", {k: v.shape for k, v in out.items() if not k.startswith("param:")})


if __name__ == "__main__":
    main()
