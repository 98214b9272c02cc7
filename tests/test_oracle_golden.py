"""Pin the CPU oracle to what the reference itself produced (tests/golden/*.npz).

Fixtures were made by tests/golden/make_golden.py running the unmodified
reference (/root/reference/pkg/src/deskinfer).  These tests run everywhere
(no GPU) and check the restatement in oracle/infllm2_oracle.py:

* kernel means bit-identical (sha256) to ``BlockizedLayerCache.fine_means`` /
  ``coarse_means`` (sparse.py:106-127);
* block selections identical per (row, group) to the reference traces
  (sparse.py:458-467), in both dot modes;
* the selected blocks' float64 relevance scores identical to the traces'
  ``scores_topk`` with the reference's own dot arithmetic (``dot="sgemv"``);
* outputs within 1e-6 (sgemv) / 2e-6 (f64 dots) of the reference's float32
  outputs;
* TouchStats totals equal to the reference's (sparse.py:319-344,456-457).
"""

import numpy as np
import pytest

from golden_util import case_inputs, case_names, load
from inputs import digest
from oracle import infllm2_oracle as O

FAST = [n for n in case_names() if not n.startswith("b8_2k") and n != "b8_1300_ragged"]


def _geom(meta):
    return O.Geometry(**meta["geometry"])


def _run(name, dot):
    meta, z = load(name)
    q, k, v = case_inputs(meta)
    geom = _geom(meta)
    fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
    rows = z["rows"]
    res = O.two_stage_attention(q, k, v, fine, geom, meta["start"], rows=rows, dot=dot,
                                keep_scores=True)
    return meta, z, q, k, v, geom, fine, res


@pytest.mark.parametrize("name", case_names())
def test_kernel_means_bitwise(name):
    meta, _ = load(name)
    _, k, _ = case_inputs(meta)
    g = _geom(meta)
    assert digest(O.window_means(k, g.kernel_size, g.kernel_stride)) == meta["fine_sha"]
    assert digest(O.window_means(k, g.kernel_size, g.coarse_stride)) == meta["coarse_sha"]


@pytest.mark.parametrize("name", FAST + ["b8_2k_prefill"])
def test_selection_scores_and_outputs_sgemv(name):
    meta, z, q, k, v, geom, fine, res = _run(name, "sgemv")
    rows = z["rows"]
    got = res.selection[rows]
    want = z["selection"]
    bad = np.argwhere((got != want).any(axis=-1))
    assert bad.size == 0, f"{len(bad)} (row, group) selections differ, first {bad[:5].tolist()}"
    # scores of the selected blocks, bit-for-bit
    by_key = {(i, g): s for i, g, s in res.scores}
    for j, r in enumerate(rows):
        for g in range(meta["hkv"]):
            sel = want[j, g][want[j, g] >= 0]
            np.testing.assert_array_equal(by_key[(int(r), g)][sel], z["scores_topk"][j, g, :sel.size])
    out = res.out[z["out_rows"]]
    assert np.max(np.abs(out - z["out"])) <= 1e-6
    if len(rows) == meta["n_q"]:
        assert res.stage1_rows == meta["stage1_rows"]
        assert res.stage2_rows == meta["stage2_rows"]
        assert res.dense_rows == meta["dense_rows"]


@pytest.mark.parametrize("name", FAST)
def test_selection_and_outputs_f64_dots(name):
    meta, z, q, k, v, geom, fine, res = _run(name, "f64")
    got = res.selection[z["rows"]]
    bad = np.argwhere((got != z["selection"]).any(axis=-1))
    assert bad.size == 0, f"{len(bad)} selections differ with f64 dots"
    assert np.max(np.abs(res.out[z["out_rows"]] - z["out"])) <= 2e-6


@pytest.mark.parametrize("name", ["inc_small", "inc_b8"])
def test_incremental_means_equal_rebuild(name):
    """Incremental append/truncate re-sync == rebuild (sparse.py:111-133, F18 fix)."""
    meta, z = load(name)
    geom = O.Geometry(**meta["geometry"])
    keys = np.zeros((0, meta["hkv"], meta["d"]), np.float32)
    fine = np.zeros((0, meta["hkv"], meta["d"]), np.float32)
    coarse = fine.copy()
    from inputs import make_qkv
    for step, (op, arg) in enumerate(z["ops"]):
        if op == 0:
            boundary = keys.shape[0]
            kk = make_qkv(meta["seed"] + step, int(arg), 1, 1, meta["hkv"], meta["d"])[1]
            keys = np.concatenate([keys, kk])
        else:
            keys = keys[:arg]
            boundary = int(arg)
        fine = O.updated_means(fine, keys, geom.kernel_size, geom.kernel_stride, boundary)
        coarse = O.updated_means(coarse, keys, geom.kernel_size, geom.coarse_stride, boundary)
        assert digest(fine) == meta["fine_sha"][step], step
        assert digest(coarse) == meta["coarse_sha"][step], step
        assert keys.shape[0] == meta["lengths"][step]


def test_reference_defect_f18_is_recorded():
    """The reference's own incremental path raised on the s_c > p geometry."""
    meta, _ = load("inc_b8")
    assert 0 in meta["ref_incremental"]
    first_fail = meta["ref_incremental"].index(0)
    assert all(s == 2 for s in meta["ref_incremental"][:first_fail])
    meta, _ = load("inc_small")
    assert all(s == 2 for s in meta["ref_incremental"])


def test_dense_degradation_oracle():
    """Budget-covering selection == dense attention (test_acceptance.py:68-106)."""
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(40):
        m = int(rng.choice([8, 16, 32]))
        geom = O.Geometry(block_size=m, kernel_size=m // 2, kernel_stride=m // 4,
                          coarse_stride=m // 2, top_k=int(rng.integers(1, 5)),
                          n_init_blocks=int(rng.integers(0, 3)),
                          n_local_blocks=int(rng.integers(0, 3)))
        n_blocks = int(rng.integers(1, geom.max_selected + 1))
        length = max(n_blocks * m - int(rng.integers(0, m)), 1)
        k = rng.standard_normal((length, 2, 8)).astype(np.float32)
        v = rng.standard_normal((length, 2, 8)).astype(np.float32)
        q = rng.standard_normal((1, 4, 8)).astype(np.float32)
        fine = O.window_means(k, geom.kernel_size, geom.kernel_stride)
        res = O.two_stage_attention(q, k, v, fine, geom, length - 1)
        dense, _ = O.dense_attention(q, k, v, length - 1)
        worst = max(worst, float(np.abs(res.out - dense).max()))
    assert worst < 1e-5


def test_force_and_topk_kats():
    """KATs from test_sparse.py:162-213 and test_acceptance.py:113-137."""
    assert O.force_blocks(10, 5, 1, 2).tolist() == [0, 4, 5]
    assert O.force_blocks(10, 0, 2, 2).tolist() == [0, 1]
    assert O.force_blocks(3, 2, 0, 1).tolist() == [2]
    assert O.force_blocks(1, 0, 4, 4).tolist() == [0]
    e = np.array([], dtype=np.int64)
    assert O.select_topk(np.array([0.5, 0.9, 0.9, 0.9, 0.1]), 2, e).tolist() == [1, 2]
    assert O.select_topk(np.ones(6), 3, e).tolist() == [0, 1, 2]
    s = np.array([0.1, 0.2, 0.3, 0.4])
    assert O.select_topk(s, 2, np.array([0])).tolist() == [0, 2, 3]
    assert O.select_topk(s, 2, np.array([0]), True).tolist() == [0, 3]
    rng = np.random.default_rng(102)
    for _ in range(300):
        n = int(rng.integers(1, 41))
        k = int(rng.integers(1, 11))
        sc = rng.integers(0, 5, size=n) / 4.0
        forced = rng.choice(n, size=int(rng.integers(0, min(3, n) + 1)), replace=False)
        consume = bool(rng.integers(0, 2))
        fs = set(int(b) for b in forced)
        budget = max(0, k - len(fs)) if consume else k
        order = sorted((i for i in range(n) if i not in fs), key=lambda i: (-sc[i], i))
        assert O.select_topk(sc, k, forced, consume).tolist() == sorted(fs | set(order[:budget]))


def test_partition_and_kernel_counts():
    """test_sparse.py:57-92 and SPEC.md:142,166."""
    assert O.partition_blocks(20, 8) == [(0, 8), (8, 16), (16, 20)]
    keys = np.zeros((17, 1, 2), np.float32)
    assert O.window_means(keys, 4, 2).shape[0] == 8
    assert O.window_means(keys, 4, 16).shape[0] == 1
    assert O.window_means(keys, 4, 18).shape[0] == 0
    # l=48, p=32, s=16 -> windows [0,32), [16,48), [32,48)
    k = np.arange(48, dtype=np.float32).reshape(48, 1, 1)
    got = O.window_means(k, 32, 16)[:, 0, 0]
    np.testing.assert_array_equal(got, [15.5, 31.5, 39.5])
    assert O.kernel_range_for_block(0, 64, 32, 16, 100) == (0, 4)
    assert O.kernel_range_for_block(64, 128, 32, 16, 100) == (3, 8)


def test_touch_ratio_closed_form():
    """Canonical touch ratios 1.0625 / 0.40625 / 0.1484375 (test_acceptance.py:171-173)."""
    geom = O.Geometry()
    for length, want in ((512, 1.0625), (2048, 0.40625), (8192, 0.1484375)):
        pos = length - 1
        rows = O.stage2_rows_closed_form(pos, geom)
        assert (length // 16 + rows) / length == want
