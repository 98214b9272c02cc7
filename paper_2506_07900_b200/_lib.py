"""ctypes binding of libinfllm2.so (include/infllm2.h).

The library is built in-tree (``paper_2506_07900_b200/libinfllm2.so``, see
``build.py``).  There is no fallback: if the library is missing or fails to
load, every operator raises ``RuntimeError`` instead of silently computing
something else.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NumericError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libinfllm2.so")

c_i32, c_i64, c_sz, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p


class Geometry(ctypes.Structure):
    """``infllm2_geometry`` — mirrors SparseAttentionConfig (sparse.py:31-40)."""

    _fields_ = [("block_size", c_i32), ("kernel_size", c_i32), ("kernel_stride", c_i32),
                ("coarse_stride", c_i32), ("top_k", c_i32), ("n_init_blocks", c_i32),
                ("n_local_blocks", c_i32), ("forced_consume_budget", c_i32)]


OK = 0
ERR_CONFIG, ERR_SHAPE, ERR_POSITION, ERR_CAPACITY = -1, -2, -3, -4
ERR_WORKSPACE, ERR_UNSUPPORTED, ERR_CUDA, ERR_NUMERIC, ERR_EMPTY = -5, -6, -7, -8, -9
FLAG_EXACT_SIMT, FLAG_CHECK_FINITE, FLAG_OUT_F32, FLAG_P_SPLIT = 1, 2, 4, 8
DECODE_SHARE_SHIFT = 8          # infllm2_decode_step flags bits 8..11: concurrent decode batches

# Exported symbols and their signatures (restype, argtypes); tests check every
# symbol declared in include/infllm2.h is exported.
SIGNATURES = {
    "infllm2_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "infllm2_version": (ctypes.c_int, []),
    "infllm2_validate_geometry": (ctypes.c_int, [ctypes.POINTER(Geometry)]),
    "infllm2_max_selected": (c_i32, [ctypes.POINTER(Geometry)]),
    "infllm2_launch_count": (ctypes.c_uint64, []),
    "infllm2_decode_early_count": (ctypes.c_uint64, []),
    "infllm2_append_kv": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_i64, c_i64,
                                         c_i32, c_i64, c_vp]),
    "infllm2_compress": (ctypes.c_int, [c_vp, c_i64, c_i32, c_i32, c_i64, c_i64, c_i64, c_i32, c_i32,
                                        c_vp, c_vp, c_vp, c_i64, c_vp]),
    "infllm2_append_compress": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_i64, c_i64, c_i32,
                                               c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                               c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "infllm2_select_workspace_bytes": (c_sz, [ctypes.POINTER(Geometry), c_i64, c_i32, c_i32, c_i32,
                                              c_i64, c_i32]),
    "infllm2_select": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i64, c_i32, c_i32,
                                      c_i32, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_sz,
                                      c_i32, c_vp]),
    "infllm2_select_approx": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i64, c_i32, c_i32,
                                             c_i32, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64,
                                             c_vp, c_vp, c_vp, c_sz, c_i32, c_vp]),
    "infllm2_attend": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i64, c_i32, c_i32,
                                      c_i32, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "infllm2_forward": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i64, c_i32, c_i32,
                                       c_i32, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_sz, c_i32, c_vp]),
}

class SeqDesc(ctypes.Structure):
    """``infllm2_seq_desc`` — one sequence's blockized cache (batched decode)."""

    _fields_ = [("k_cache", c_vp), ("v_cache", c_vp), ("cap", c_i64), ("fine_means", c_vp), ("means_hi", c_vp),
                ("means_lo", c_vp), ("means_cap", c_i64), ("coarse_means", c_vp), ("coarse_cap", c_i64)]


SIGNATURES.update({
    "infllm2_forward_at": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32,
                                          c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz,
                                          c_i32, c_vp]),
    "infllm2_forward_tree": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i32, c_i32, c_i32, c_vp,
                                            c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_i32, c_vp, c_vp,
                                            c_vp, c_vp, c_vp, c_sz, c_i32, c_vp]),
    "infllm2_forward_tree_workspace_bytes": (c_sz, [ctypes.POINTER(Geometry), c_i64, c_i32, c_i32, c_i32, c_i64]),
    "infllm2_forward_at_workspace_bytes": (c_sz, [ctypes.POINTER(Geometry), c_i64, c_i32, c_i64, c_i64]),
    "infllm2_dense_attend": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32,
                                            c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i32, c_vp]),
    "infllm2_dense_regime": (ctypes.c_int, [ctypes.POINTER(Geometry), c_i64, c_i64, c_i64]),
    "infllm2_decode_supported": (ctypes.c_int, [ctypes.POINTER(Geometry), c_i32, c_i32, c_i32]),
    "infllm2_decode_table_bytes": (c_sz, [c_i32]),
    "infllm2_decode_table_build": (ctypes.c_int, [ctypes.POINTER(SeqDesc), ctypes.POINTER(c_i64), c_i32, c_i32,
                                                  c_i32, c_vp, c_vp]),
    "infllm2_decode_table_link": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "infllm2_decode_table_lengths": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_i64), c_vp]),
    "infllm2_decode_workspace_bytes": (c_sz, [ctypes.POINTER(Geometry), c_i32, c_i32, c_i64]),
    "infllm2_decode_step": (ctypes.c_int, [ctypes.POINTER(Geometry), c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_vp,
                                           c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_i32, c_vp]),
})

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load (once) and return the library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            # INFLLM2_LIB_PATH: an alternative build of the same ABI (A/B timing of kernel variants)
            path = os.environ.get("INFLLM2_LIB_PATH", LIB_PATH)
            if not os.path.exists(path):
                raise RuntimeError(
                    f"libinfllm2.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; "
                    "g.build()'` — there is no CPU fallback")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    """Map a library return code to the reference's exception types."""
    if rc == OK:
        return
    msg = f"{what}: {load().infllm2_strerror(rc).decode()} (code {rc})"
    if rc == ERR_NUMERIC:
        raise NumericError(msg)
    if rc in (ERR_CONFIG, ERR_SHAPE, ERR_POSITION, ERR_CAPACITY, ERR_EMPTY):
        raise ValidationError(msg)
    raise RuntimeError(msg)
