"""Golden fixture for tree-draft verification: the UNMODIFIED reference's dense
``forward_tree`` (specdec.py:565-625) on the model-seam bundle.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_tree.py

Same seeded ``random_bundle`` as make_golden_model.py (its parameters are in
model_seam.npz); the first 300 tokens of model_seam.npz's sequence are
prefilled into a dense cache with ``forward``, then a 12-node draft tree (two
roots, branching, depths 1..4) is scored with ``PackedMask.from_parents``.
Stores the tree tokens, parents, depths and the reference's logits.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from deskinfer.model import ModelConfig, forward, random_bundle  # noqa: E402
from deskinfer.specdec import PackedMask, forward_tree, make_cache  # noqa: E402

sys.path.insert(0, HERE)
from make_golden_model import CFG  # noqa: E402

PARENTS = [-1, 0, 0, 1, 1, 2, 3, 3, 5, 6, -1, 10]


def main() -> None:
    cfg = ModelConfig(**CFG)
    bundle = random_bundle(cfg, seed=2506, scale=0.2)
    seam = np.load(os.path.join(HERE, "model_seam.npz"))
    prefix = seam["tokens"][:300]
    cache = make_cache(bundle, "dense", None)
    forward(bundle, prefix, cache, backend="dense")
    parents = np.asarray(PARENTS, dtype=np.int64)
    depths = np.zeros_like(parents)
    for i, p in enumerate(parents):
        depths[i] = 1 if p < 0 else depths[p] + 1
    tokens = np.random.default_rng(565).integers(0, cfg.vocab_size, size=parents.size)
    res = forward_tree(bundle, cache, tokens, depths, PackedMask.from_parents(parents))
    assert cache.length == 300
    np.savez_compressed(os.path.join(HERE, "model_tree.npz"), parents=parents, depths=depths, tokens=tokens,
                        prefix_len=np.int64(300), logits=res.logits)
    print("wrote model_tree.npz", res.logits.shape)


if __name__ == "__main__":
    main()
