"""BASELINE configs[2] parity at the headline size: one 131 072-token layer of
the 8B-shaped stack (32 q / 2 KV heads, d 128, m 64, p 32, s 16, init 1,
local 2) — and, for configs[4]'s MiniCPM4-0.5B shape, 16 q / 2 KV heads, d 64 —
all rows prefilled through ``two_stage_attention`` on the B200 (the
exact product call bench.py times), checked against the CPU oracle (the
reference's algorithm, /root/reference/pkg/src/deskinfer/sparse.py:387-468,
float64 dots) on >= 1024 sampled rows: seeded rows, the first/last rows,
block-size multiples +-1 and the zig-zag shard boundaries of 2/4/8 ranks.

Bars: selections bit-exact per (row, group); outputs and LSE within the
tensor-core bars of DESIGN.md §5.  The oracle fans rows out over the host
cores (rows are independent given the cache).
"""

import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

from bars import LSE_TC, OUT_ABS, OUT_REL, SPLIT_ABS, SPLIT_REL  # noqa: F401
from envelope import record
from oracle import infllm2_oracle as O

pytestmark = pytest.mark.gpu

import paper_2506_07900_b200 as P  # noqa: E402

L = 131072
_ST = {}


def _oracle_rows(rows):
    st = _ST
    res = []
    for r in rows:
        o = O.two_stage_attention(st["q"][r][None], st["k"], st["v"], st["fine"], st["geom"], int(st["pos"][r]))
        res.append((r, o.selection[0], o.out[0], o.lse[0]))
    return res


def sample_positions(seed: int, count: int = 1024) -> np.ndarray:
    rng = np.random.default_rng(seed)
    picks = {0, 1, 2, 63, 64, 65, 127, 128, L - 2, L - 1}
    for b in np.linspace(2, L // 64 - 1, 24).round().astype(int):
        picks.update({b * 64 - 1, b * 64, b * 64 + 1})
    for world in (2, 4, 8):
        size = L // (2 * world)
        for c in range(1, 2 * world):
            picks.update({c * size - 1, c * size})
    while len(picks) < count:
        picks.add(int(rng.integers(0, L)))
    return np.asarray(sorted(picks), dtype=np.int64)


@pytest.mark.parametrize("top_k,shape,rows", [(16, (32, 2, 128), 1024), (64, (32, 2, 128), 1024),
                                              (16, (16, 2, 64), 512)], ids=["8B-k16", "8B-k64", "0.5B-k16"])
def test_config2_128k_layer_vs_oracle(top_k, shape, rows):
    torch.cuda.set_device(0)
    hq, hkv, d = shape
    cfg = P.SparseAttentionConfig(top_k=top_k)
    g = torch.Generator(device="cuda").manual_seed(1_000_003 + top_k + (0 if d == 128 else d))
    k = torch.randn((L, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((L, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn((L, hq, d), generator=g, device="cuda").to(torch.bfloat16)
    layer = P.BlockizedLayerCache(hkv, d, cfg, capacity=L)
    layer.append(k, v)
    out, sel, lse = P.two_stage_attention(q, layer, cfg, 0, return_selection=True, return_lse=True,
                                          out_dtype=torch.float32)
    pos = sample_positions(top_k + (0 if d == 128 else d), rows)
    idx = torch.as_tensor(pos, device="cuda")
    got_sel = sel[idx].cpu().numpy()
    got_out = out[idx].cpu().numpy()
    got_lse = lse[idx].cpu().numpy()
    k_h = k.float().cpu().numpy()
    _ST.update(k=k_h, v=v.float().cpu().numpy(), q=q[idx].float().cpu().numpy(), pos=pos,
               fine=O.window_means(k_h, 32, 16), geom=O.Geometry(top_k=top_k))
    assert np.array_equal(layer.fine_means.contiguous().cpu().numpy(), _ST["fine"])
    cores = os.cpu_count() or 1
    chunks = [list(range(i, pos.size, cores * 4)) for i in range(cores * 4)]
    with mp.get_context("fork").Pool(cores) as pool:
        results = [x for part in pool.map(_oracle_rows, chunks) for x in part]
    results.sort(key=lambda x: x[0])
    ref_sel = np.stack([x[1] for x in results])
    ref_out = np.stack([x[2] for x in results])
    ref_lse = np.stack([x[3] for x in results])
    bad = np.argwhere((got_sel != ref_sel).any(-1))
    assert bad.size == 0, f"{len(bad)} of {pos.size * 2} (row, group) selections differ: " \
                          f"{[(int(pos[i]), int(gg)) for i, gg in bad[:4]]}"
    err = np.abs(got_out - ref_out)
    lerr = np.abs(got_lse - ref_lse)
    record(f"config2_k{top_k}_d{d}", rows=pos.size, out_max_abs=err.max(),
           out_max_rel=(err / (np.abs(ref_out) + 1e-3)).max(), lse_max_abs=lerr.max())
    assert (err <= OUT_ABS + OUT_REL * np.abs(ref_out)).all(), err.max()
    assert lerr.max() <= LSE_TC, lerr.max()
