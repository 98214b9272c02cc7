"""Generate golden fixtures by running the UNMODIFIED reference in this container.

Usage (from the repo root, in the build container where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``deskinfer`` read-only from ``/root/reference/pkg/src`` and, for
each case below, records what the reference itself computes:

* ``selection``   — per (row, KV group) selected block ids from ``traces``
                    (``sparse.py:458-467``), -1 padded;
* ``scores_topk`` — the float64 relevance scores of those blocks;
* ``out``         — ``two_stage_attention`` outputs for the stored rows;
* ``fine_sha`` / ``coarse_sha`` — sha256 of ``BlockizedLayerCache``'s
                    float32 kernel means (``sparse.py:106-127``).

Inputs are regenerated from (seed, shape) by ``tests/golden/inputs.py``; the
fixture stores their sha256 so a drifted generator fails loudly.  The GPU box
never runs this script (``/root/reference`` does not exist there); it only
reads the committed ``*.npz`` files.
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from inputs import digest, make_qkv  # noqa: E402
from cases import B8, CASES, SMALL, build_inputs, sample_rows  # noqa: E402,F401

def run_case(name):
    from deskinfer.sparse import BlockizedLayerCache, SparseAttentionConfig, two_stage_attention

    geom, seed, length, n_q, start, hq, hkv, d, rows, out_rows, scale, kind = CASES[name]
    cfg = SparseAttentionConfig(**geom)
    q, k, v = build_inputs(seed, length, n_q, hq, hkv, d, scale, kind)
    layer = BlockizedLayerCache(hkv, d, cfg)
    layer.append(k, v)
    row_ids = np.arange(n_q) if rows is None else sample_rows(n_q, start, seed)
    smax = cfg.top_k + cfg.n_init_blocks + cfg.n_local_blocks
    sel = np.full((row_ids.size, hkv, smax), -1, np.int32)
    scores = np.full((row_ids.size, hkv, smax), np.nan, np.float64)
    if out_rows is None or out_rows >= row_ids.size:
        keep_out = np.arange(row_ids.size)
    else:
        keep_out = np.unique(np.linspace(0, row_ids.size - 1, out_rows).round().astype(np.int64))
    outs = np.zeros((keep_out.size, hq, d), np.float32)
    keep_pos = {int(j): idx for idx, j in enumerate(keep_out)}
    stage1 = stage2 = dense = 0
    from deskinfer.sparse import TouchStats
    for j, r in enumerate(row_ids):
        traces = []
        stats = TouchStats()
        o = two_stage_attention(q[r:r + 1], layer, cfg, start + int(r), stats=stats, traces=traces)
        stage1 += stats.stage1
        stage2 += stats.stage2
        dense += stats.dense_rows
        for t in traces:
            g = t["group"]
            sel[j, g, :len(t["selected"])] = t["selected"]
            scores[j, g, :len(t["scores_topk"])] = t["scores_topk"]
        if j in keep_pos:
            outs[keep_pos[j]] = o[0]
    meta = dict(name=name, geometry=geom, seed=seed, length=length, n_q=n_q, start=start,
                hq=hq, hkv=hkv, d=d, scale=scale, kind=kind,
                input_sha=digest(q, k, v),
                fine_sha=digest(layer.fine_means), coarse_sha=digest(layer.coarse_means),
                stage1_rows=stage1, stage2_rows=stage2, dense_rows=dense)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        meta=np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8),
        rows=row_ids.astype(np.int32), selection=sel, scores_topk=scores,
        out_rows=row_ids[keep_out].astype(np.int32), out=outs)
    return name, row_ids.size


def run_incremental(name, geom, hkv, d, steps, seed):
    """Append/truncate sequences; record the reference's kernel means after each step.

    The recorded truth is the reference's ``build_kernels`` over the current
    keys (its own invariant: incremental == rebuild, test_sparse.py:276-290).
    The reference's incremental ``BlockizedLayerCache`` is driven alongside;
    ``ref_incremental`` records per step whether it ran (1), matched the
    rebuild bit-for-bit (2), or raised (0 — the s_c > p defect, F18).
    """
    from deskinfer.sparse import BlockizedLayerCache, SparseAttentionConfig, build_kernels

    cfg = SparseAttentionConfig(**geom)
    layer = BlockizedLayerCache(hkv, d, cfg)
    layer_alive = True
    rng = np.random.default_rng(seed)
    ops, fine, coarse, lengths, status = [], [], [], [], []
    keys = np.zeros((0, hkv, d), np.float32)
    for op, arg in steps(rng):
        if op == "append":
            kk = make_qkv(seed + len(ops), arg, 1, 1, hkv, d)[1]
            keys = np.concatenate([keys, kk])
            ops.append((0, arg))
        else:
            keys = keys[:arg]
            ops.append((1, arg))
        want_f = build_kernels(keys, cfg.kernel_size, cfg.kernel_stride)
        want_c = build_kernels(keys, cfg.kernel_size, cfg.coarse_stride)
        st = 0
        if layer_alive:
            try:
                if op == "append":
                    layer.append(kk, kk)
                else:
                    layer.truncate(arg)
                st = 1 + int(np.array_equal(layer.fine_means, want_f)
                             and np.array_equal(layer.coarse_means, want_c))
            except ValueError:
                layer_alive = False
        status.append(st)
        fine.append(digest(want_f))
        coarse.append(digest(want_c))
        lengths.append(int(keys.shape[0]))
    meta = dict(name=name, geometry=geom, hkv=hkv, d=d, seed=seed,
                fine_sha=fine, coarse_sha=coarse, lengths=lengths,
                ref_incremental=status)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        meta=np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8),
        ops=np.asarray(ops, dtype=np.int64))
    return name, len(ops)


def small_steps(rng):
    length = 0
    for step in range(40):
        n_new = int(rng.integers(1, 5))
        yield "append", n_new
        length += n_new
        if step % 7 == 3 and length > 4:
            length -= int(rng.integers(1, 4))
            yield "truncate", length


def b8_steps(rng):
    yield "append", 8192
    for _ in range(256):
        yield "append", 1
    yield "truncate", 8192 + 100
    yield "truncate", 8190
    for _ in range(40):
        yield "append", int(rng.integers(1, 40))


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        futs = [ex.submit(run_case, nm) for nm in names if nm in CASES]
        if "inc_small" in names or not sys.argv[1:]:
            futs.append(ex.submit(run_incremental, "inc_small", SMALL, 2, 4, small_steps, 10))
        if "inc_b8" in names or not sys.argv[1:]:
            futs.append(ex.submit(run_incremental, "inc_b8", B8, 2, 128, b8_steps, 30))
        for f in futs:
            print(*f.result(), flush=True)
