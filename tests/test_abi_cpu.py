"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/infllm2.h declares, and its host-only entry points (geometry
validation, error strings) behave like the reference's validation
(sparse.py:42-51).  No compute call is made (no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_07900_b200 import _lib
    return _lib.load()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "infllm2.h")).read()
    return sorted(set(re.findall(r"\b(infllm2_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lib):
    from paper_2506_07900_b200 import _lib
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (infllm2_\w+)", nm))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.SIGNATURES), "ctypes signature table out of sync"


def test_library_is_sm100a(lib):
    from paper_2506_07900_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_geometry_validation_matches_reference(lib):
    from paper_2506_07900_b200 import _lib
    import paper_2506_07900_b200 as P
    ok = P.SparseAttentionConfig().geometry()
    assert lib.infllm2_validate_geometry(ctypes.byref(ok)) == 0
    assert lib.infllm2_max_selected(ctypes.byref(ok)) == 11
    bad = [dict(block_size=0), dict(kernel_stride=24, kernel_size=16), dict(coarse_stride=24),
           dict(top_k=0), dict(n_init_blocks=-1)]
    for kw in bad:
        with pytest.raises(P.ValidationError):
            P.SparseAttentionConfig(**kw)
        g = _lib.Geometry(64, 32, 16, 128, 8, 1, 2, 0)
        for k, v in kw.items():
            setattr(g, k, v)
        assert lib.infllm2_validate_geometry(ctypes.byref(g)) == _lib.ERR_CONFIG, kw
    assert lib.infllm2_strerror(-3) == b"query position beyond cache length"


def test_host_helpers_match_reference_kats():
    import paper_2506_07900_b200 as P
    assert P.partition_blocks(20, 8) == [(0, 8), (8, 16), (16, 20)]
    assert P.force_blocks(10, 5, 1, 2).tolist() == [0, 4, 5]
    assert P.force_blocks(1, 0, 4, 4).tolist() == [0]
    assert P.kernel_range_for_block((64, 128), 32, 16, 100) == (3, 8)
    with pytest.raises(P.ValidationError):
        P.force_blocks(3, 3, 1, 1)


def test_workspace_query_is_host_only(lib):
    import paper_2506_07900_b200 as P
    g = P.SparseAttentionConfig(top_k=16).geometry()
    n = lib.infllm2_select_workspace_bytes(ctypes.byref(g), 8192, 32, 2, 128, 8192, 0)
    assert n > 0
