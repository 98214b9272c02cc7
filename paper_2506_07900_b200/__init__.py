"""B200-native InfLLM v2 two-stage block-sparse attention (arXiv 2506.07900).

Drop-in for the reference's sparse-attention surface (``deskinfer.sparse``):
``SparseAttentionConfig``, ``BlockizedLayerCache``, ``blockized_cache``,
``build_kernels`` and ``two_stage_attention`` on CUDA tensors, computed by the
hand-written sm_100a kernels in ``libinfllm2.so`` (C ABI: ``include/infllm2.h``).
"""

from . import model, stages, tree
from .decode import DecodeBatch
from .errors import NumericError, ValidationError
from .tree import PackedMask, tree_attention
from .sparse import (BlockizedLayerCache, KVCache, SparseAttentionConfig, TouchStats,
                     blockized_cache, build_kernels, force_blocks, kernel_range_for_block,
                     partition_blocks, two_stage_attention)

__all__ = [
    "model", "stages", "tree", "DecodeBatch", "BlockizedLayerCache", "KVCache", "NumericError", "SparseAttentionConfig", "TouchStats",
    "ValidationError", "blockized_cache", "build_kernels", "force_blocks",
    "kernel_range_for_block", "partition_blocks", "two_stage_attention", "PackedMask", "tree_attention",
]
