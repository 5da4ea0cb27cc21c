"""B200-native BinaryAttention forward path (arXiv 2603.09582) behind the reference's operator shape.

    binary_attention(Q, K, V, bias, scale) -> O

Python is only the host-side convenience layer over the C ABI in include/binattn_cuda.h
(libbinattn_cuda.so, hand-written CUDA for sm_100a).  There is no CPU path here: importing works without
a GPU (so the build can be checked), every compute call needs one.
"""
from .api import (BinaryAttention, BinAttnError, ShapeError, ValidationError, CudaError, UnsupportedError,
                  binary_attention, binary_attention_fused, AttentionConfig, AttentionOutput, Relative1dBias, Relative2dBias,
                  FidelityReport, load_library)
from .launcher import shard_range, shard_heads, shard_plan, shard_units, ShardedBinaryAttention

__all__ = ["BinaryAttention", "BinAttnError", "ShapeError", "ValidationError", "CudaError", "UnsupportedError",
           "binary_attention", "binary_attention_fused", "AttentionConfig", "AttentionOutput", "Relative1dBias", "Relative2dBias", "FidelityReport", "load_library",
           "shard_range", "shard_heads", "shard_plan", "shard_units", "ShardedBinaryAttention"]
