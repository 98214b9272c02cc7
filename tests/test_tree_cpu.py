"""PackedMask (specdec.py:117-157) host logic, no GPU: bit layout, multi-word
rows, validation."""

import numpy as np
import pytest

from paper_2506_07900_b200.errors import ValidationError
from paper_2506_07900_b200.tree import PackedMask


def test_chain_packs_as_documented():
    m = PackedMask.from_parents([-1, 0, 1])          # specdec.py:121-123: rows 0b001, 0b011, 0b111
    assert m.words[:, 0].tolist() == [0b001, 0b011, 0b111]
    m.validate()


def test_branching_tree_and_dense_view():
    parents = [-1, 0, 0, 1, -1, 4]
    d = PackedMask.from_parents(parents).to_dense()
    for i, p in enumerate(parents):
        anc = {i}
        while p >= 0:
            anc.add(p)
            p = parents[p]
        assert set(np.flatnonzero(d[i]).tolist()) == anc


def test_more_than_64_nodes_use_two_words():
    parents = [-1] + list(range(69))                 # a 70-node chain
    m = PackedMask.from_parents(parents)
    assert m.words.shape == (70, 2)
    assert m.to_dense()[69].all()
    assert int(m.words[69, 1]) == (1 << 6) - 1


def test_validation():
    with pytest.raises(ValidationError):
        PackedMask.from_parents([0])                 # a node cannot be its own parent
    with pytest.raises(ValidationError):
        PackedMask(words=np.zeros((2, 1), np.uint64), n_nodes=2).validate()
    with pytest.raises(ValidationError):
        PackedMask(words=np.zeros((2, 2), np.uint64), n_nodes=2).validate()
