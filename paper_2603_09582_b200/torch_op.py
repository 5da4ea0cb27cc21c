"""torch.library registration of the operator ("the caller side"):

    torch.ops.binattn.binary_attention(Q, K, V, bias, scale) -> O          (dense bias table or None)
    torch.ops.binattn.binary_attention_rel1d(Q, K, V, offsets, scale) -> O (Relative1dBias offsets)
    torch.ops.binattn.binary_attention_ex(Q, K, V, bias, scale, quantize_pv, out_bf16) -> O
                                   (quantize_pv: the reference's default integer P.V arithmetic; out_bf16: bfloat16 output)

so model code (and torch.compile / export graphs, through the fake kernels below) can call the batched [B,H,N,d]
forward like any other op.  Forward only -- the reference path is forward-only too (qat.cpp's toys are out of scope).
The CUDA implementation is the C ABI (api.BinaryAttention.forward); there is no CPU kernel registered: calling the op
with CPU tensors fails loudly, like the rest of this package.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import api

_lib_defined = False


def register() -> None:
    """Idempotent; called on import of this module."""
    global _lib_defined
    if _lib_defined:
        return
    _lib_defined = True

    @torch.library.custom_op("binattn::binary_attention", mutates_args=(), device_types="cuda")
    def binary_attention(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, bias: Optional[torch.Tensor],
                         scale: Optional[float]) -> torch.Tensor:
        return api._handle_for(Q.device).forward(Q, K, V, bias, scale)

    @binary_attention.register_fake
    def _(Q, K, V, bias, scale):
        return Q.new_empty(Q.shape, dtype=torch.float32)

    @torch.library.custom_op("binattn::binary_attention_ex", mutates_args=(), device_types="cuda")
    def binary_attention_ex(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, bias: Optional[torch.Tensor], scale: Optional[float],
                            quantize_pv: bool, out_bf16: bool) -> torch.Tensor:
        return api._handle_for(Q.device).forward(Q, K, V, bias, scale, quantize_pv=quantize_pv,
                                                 out_dtype=torch.bfloat16 if out_bf16 else torch.float32)

    @binary_attention_ex.register_fake
    def _(Q, K, V, bias, scale, quantize_pv, out_bf16):
        return Q.new_empty(Q.shape, dtype=torch.bfloat16 if out_bf16 else torch.float32)

    @torch.library.custom_op("binattn::binary_attention_rel1d", mutates_args=(), device_types="cuda")
    def binary_attention_rel1d(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, offsets: torch.Tensor,
                               scale: Optional[float]) -> torch.Tensor:
        return api._handle_for(Q.device).forward(Q, K, V, api.Relative1dBias(offsets), scale)

    @binary_attention_rel1d.register_fake
    def _(Q, K, V, offsets, scale):
        return Q.new_empty(Q.shape, dtype=torch.float32)


register()
