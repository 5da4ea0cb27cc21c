"""ctypes binding of include/binattn_cuda.h plus the host-side mirror of the reference's operator API.

Mirrors (names, argument meaning, error behaviour):
  binattn::AttentionConfig / AttentionConfig::make   proj/include/binattn/attention.hpp:29-41, src/attention.cpp:45-53
  binattn::AttentionOutput                           attention.hpp:43-48
  binattn::binary_attention_fused                    attention.hpp:69-71, attention.cpp:250-382
  binattn::ShapeError / ValidationError              errors.hpp:16-25
PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_PKG, "libbinattn_cuda.so")

BA_BF16, BA_F16, BA_F32 = 0, 1, 2
KERNELS = {"auto": 0, "simt": 1, "tcgen05": 2}
_DTYPES = {torch.bfloat16: BA_BF16, torch.float16: BA_F16, torch.float32: BA_F32}


class BinAttnError(RuntimeError):
    """binattn::Error (errors.hpp:10-13)."""


class ShapeError(BinAttnError):
    """binattn::ShapeError (errors.hpp:16-19)."""


class ValidationError(BinAttnError):
    """binattn::ValidationError (errors.hpp:22-25)."""


class CudaError(BinAttnError):
    pass


class UnsupportedError(BinAttnError):
    pass


_STATUS = {1: ShapeError, 2: ValidationError, 3: CudaError, 4: UnsupportedError}


class _Params(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("N", C.c_int32), ("d", C.c_int32), ("in_dtype", C.c_int32),
                ("bias_mode", C.c_int32), ("bias_heads", C.c_int32), ("bias_dtype", C.c_int32),
                ("bias_ld", C.c_int64), ("inv_tau", C.c_float), ("kernel", C.c_int32),
                ("quantize_pv", C.c_int32), ("block_cols", C.c_int32), ("unit_begin", C.c_int64), ("unit_end", C.c_int64),
                ("out_bf16", C.c_int32), ("bias_on_device", C.c_int32)]


_lib = None


class _Fidelity(C.Structure):  # ba_fidelity (include/binattn_cuda.h)
    _fields_ = [("cos_sim", C.c_double), ("relative_l1", C.c_double), ("rmse", C.c_double), ("precision_at_k", C.c_double)]


@dataclass
class FidelityReport:
    """binattn::FidelityReport (fidelity.hpp:12-18)."""
    cos_sim: float
    relative_l1: float
    rmse: float
    precision_at_k: float
    k: int


def load_library() -> C.CDLL:
    """Load libbinattn_cuda.so (built in-tree by paper_2603_09582_b200/build.py).  Fails loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback for this package)")
    lib = C.CDLL(_LIB_PATH)
    vp, i64 = C.c_void_p, C.c_int64
    lib.ba_create.argtypes = [C.c_int, C.POINTER(vp)]
    lib.ba_destroy.argtypes = [vp]
    lib.ba_workspace_bytes.argtypes = [C.POINTER(_Params)]
    lib.ba_workspace_bytes.restype = C.c_size_t
    lib.ba_pack_signs.argtypes = [vp, C.POINTER(_Params), vp, vp, vp, vp]
    lib.ba_binary_logits.argtypes = [vp, C.POINTER(_Params), vp, vp, i64, vp, vp]
    lib.ba_quantize_values.argtypes = [vp, C.POINTER(_Params), vp, vp, vp, vp]
    lib.ba_binary_attention_fwd.argtypes = [vp, C.POINTER(_Params), vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.ba_attention_probs.argtypes = [vp, C.POINTER(_Params), C.c_int, vp, vp, vp, i64, vp, C.c_int, vp, vp]
    lib.ba_attention_fidelity.argtypes = [vp, vp, vp, i64, i64, i64, C.POINTER(_Fidelity), vp]
    lib.ba_binary_attention_host.argtypes = [vp, C.POINTER(_Params), vp, vp, vp, vp, vp, vp, vp]
    lib.ba_shard_range.argtypes = [i64, C.c_int, C.c_int, C.POINTER(i64), C.POINTER(i64)]
    lib.ba_shard_units.argtypes = [C.POINTER(_Params), C.c_int, C.c_int, C.POINTER(i64), C.POINTER(i64)]
    lib.ba_select_kernel.argtypes = [C.POINTER(_Params)]
    lib.ba_launch_count.argtypes = [vp]
    lib.ba_launch_count.restype = i64
    lib.ba_profile_begin.argtypes = [vp, C.c_int]
    lib.ba_profile_end.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.ba_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc:
        raise _STATUS.get(rc, BinAttnError)(load_library().ba_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


@dataclass
class Relative1dBias:
    """binattn::Relative1dBias (attention.hpp:18-21): b_ij = offsets[i - j + N - 1].  offsets: [2N-1] or [1|H, 2N-1],
    fp32 or bf16.  Pass it as `bias`: the kernels generate the bias from the table, no N x N tensor is ever built
    (attention.cpp:65-76 materialises one)."""
    offsets: torch.Tensor


@dataclass
class Relative2dBias:
    """binattn::Relative2dBias (attention.hpp:22-26): N = g*g tokens on a g x g grid,
    b_ij = row_offsets[ri - rj + g - 1] + col_offsets[ci - cj + g - 1], both tables of length 2g-1 (or [1|H, 2g-1]).
    Passed to the C ABI as BA_BIAS_REL2D: generated inside the second-generation tcgen05 kernel from the two tables (N >= 512,
    g % 32 == 0), else expanded once on the device to the table materialize_bias builds (attention.cpp:78-96).
    `materialize` is that table, for tests and for callers of the dense path."""
    row_offsets: torch.Tensor
    col_offsets: torch.Tensor

    def materialize(self, n: int) -> torch.Tensor:
        g = int(round(math.sqrt(n)))
        if g * g != n:
            raise ShapeError("bias: relative-2d requires N to be a perfect square")  # attention.cpp:79-81
        ro, co = self.row_offsets, self.col_offsets
        ro = ro.unsqueeze(0) if ro.dim() == 1 else ro
        co = co.unsqueeze(0) if co.dim() == 1 else co
        if ro.shape[-1] != 2 * g - 1 or co.shape[-1] != 2 * g - 1 or ro.shape[0] != co.shape[0]:
            raise ShapeError("bias: relative-2d tables must have length 2*sqrt(N)-1")  # attention.cpp:82-83
        idx = torch.arange(n, device=ro.device)
        r, c = idx // g, idx % g
        dr = r[:, None] - r[None, :] + (g - 1)
        dc = c[:, None] - c[None, :] + (g - 1)
        return ro[:, dr] + co[:, dc]  # [Hb, N, N]


@dataclass
class AttentionConfig:
    """binattn::AttentionConfig (attention.hpp:29-41).  block_rows/block_cols are accepted and validated like the
    reference's (attention.cpp:26-28) but do not change the result: the CUDA kernels pick their own tiles and the
    reference itself is tile-invariant to 1e-12 (test_attention.cpp:254-272).  quantize_pv=True runs the integer P.V
    mode on the CUDA cores, where block_cols (<= 64) DOES shape the result, exactly as in the reference.

    DELIBERATE DEVIATION: quantize_pv defaults to False here, to True in the reference (attention.hpp:35).  False is the
    fp P.V mode the tensor-core product path implements and O-parity is defined against; set
    quantize_pv=True to get the reference's default arithmetic when porting `AttentionConfig::make(n, d)`."""
    seq_len: int = 0
    head_dim: int = 0
    temperature: float = 1.0
    block_rows: int = 64
    block_cols: int = 64
    quantize_pv: bool = False
    bias: Optional[object] = None  # dense [N,N] (or [Hb,N,N]) table == materialize_bias output, or a Relative1dBias

    @staticmethod
    def make(n: int, d: int) -> "AttentionConfig":  # attention.cpp:45-53
        return AttentionConfig(seq_len=n, head_dim=d, temperature=math.sqrt(d), block_rows=min(64, n),
                               block_cols=min(64, n))


@dataclass
class AttentionOutput:
    """binattn::AttentionOutput (attention.hpp:43-48); probs is never produced by the fused kernels."""
    output: torch.Tensor
    row_max: torch.Tensor
    row_sum: torch.Tensor


class BinaryAttention:
    """One ba_handle bound to one CUDA device."""

    def __init__(self, device: int | torch.device | None = None):
        self.lib = load_library()
        if not torch.cuda.is_available():
            raise CudaError("no CUDA device: paper_2603_09582_b200 has no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        h = C.c_void_p()
        _check(self.lib.ba_create(dev.index, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.ba_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ------------------------------------------------------------------------------------------
    def _params(self, B, H, N, d, dtype, bias=None, scale=None, kernel="auto", quantize_pv=False, block_cols=None) -> _Params:
        if dtype not in _DTYPES:
            raise ValidationError(f"unsupported input dtype {dtype}")
        p = _Params(B=B, H=H, N=N, d=d, in_dtype=_DTYPES[dtype], kernel=KERNELS[kernel])
        p.quantize_pv, p.block_cols = int(bool(quantize_pv)), int(block_cols or 0)
        p.inv_tau = (1.0 / math.sqrt(d)) if scale is None else float(scale)
        if isinstance(bias, Relative2dBias):
            tb = bias.row_offsets  # (_check_bias packed both tables into one [Hb, 2, 2g-1] tensor and stored it here)
            if tb.dtype not in (torch.bfloat16, torch.float32):
                raise ValidationError("bias must be bfloat16 or float32")
            p.bias_mode, p.bias_heads, p.bias_dtype, p.bias_ld = 3, tb.shape[0], _DTYPES[tb.dtype], 0
        elif isinstance(bias, Relative1dBias):
            off = bias.offsets
            if off.dtype not in (torch.bfloat16, torch.float32):
                raise ValidationError("bias must be bfloat16 or float32")
            p.bias_mode, p.bias_heads, p.bias_dtype, p.bias_ld = 2, off.shape[0], _DTYPES[off.dtype], 0
        elif bias is not None:
            if bias.dtype not in (torch.bfloat16, torch.float32):
                raise ValidationError("bias must be bfloat16 or float32")
            p.bias_mode, p.bias_heads, p.bias_dtype = 1, bias.shape[0], _DTYPES[bias.dtype]
            p.bias_ld = bias.stride(1)
        return p

    @staticmethod
    def _check_bias(bias, H, N):
        """Shape rules of materialize_bias (attention.cpp:59-67); returns the tensor whose pointer goes to the C ABI."""
        if bias is None:
            return None, None
        if isinstance(bias, Relative2dBias):
            g = int(round(math.sqrt(N)))
            if g * g != N:
                raise ShapeError("bias: relative-2d requires N to be a perfect square")  # attention.cpp:79-81
            ro, co = bias.row_offsets, bias.col_offsets
            ro = ro.unsqueeze(0) if ro.dim() == 1 else ro
            co = co.unsqueeze(0) if co.dim() == 1 else co
            if ro.dim() != 2 or co.shape != ro.shape or ro.shape[1] != 2 * g - 1 or ro.shape[0] not in (1, H):
                raise ShapeError("bias: relative-2d tables must have length 2*sqrt(N)-1")  # attention.cpp:82-83
            packed = torch.stack([ro, co.to(ro.dtype)], dim=1).contiguous()  # [Hb, 2, 2g-1]
            return Relative2dBias(packed, packed), packed
        if isinstance(bias, Relative1dBias):
            off = bias.offsets
            if off.dim() == 1:
                off = off.unsqueeze(0)
            if off.dim() != 2 or off.shape[1] != 2 * N - 1 or off.shape[0] not in (1, H):
                raise ShapeError("bias: relative-1d offsets must have length 2N-1")  # attention.cpp:66-67
            off = off.contiguous()
            return Relative1dBias(off), off
        if bias.dim() == 2:
            bias = bias.unsqueeze(0)
        if bias.dim() != 3 or bias.shape[1] != N or bias.shape[2] != N or bias.shape[0] not in (1, H):
            raise ShapeError("bias: dense table must be N x N")  # attention.cpp:60-61
        if bias.stride(2) != 1 or bias.stride(0) != bias.stride(1) * N:
            bias = bias.contiguous()
        return bias, bias

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def launch_count(self) -> int:
        return int(self.lib.ba_launch_count(self.h))

    def profile_begin(self, max_calls: int) -> None:
        _check(self.lib.ba_profile_begin(self.h, max_calls))

    def profile_end(self):
        """-> (calls, pack_ms_total, attn_ms_total) from CUDA events recorded on the launching stream."""
        n, a, b = C.c_int(), C.c_double(), C.c_double()
        _check(self.lib.ba_profile_end(self.h, C.byref(n), C.byref(a), C.byref(b)))
        return n.value, a.value, b.value

    def shard_units(self, B, H, N, world, rank):
        """ba_shard_units: this rank's contiguous range of the B*H*ceil(N/256) (head, 256-row block) units."""
        p = _Params(B=B, H=H, N=N, d=1)
        b, e = C.c_int64(), C.c_int64()
        _check(self.lib.ba_shard_units(C.byref(p), world, rank, C.byref(b), C.byref(e)))
        return b.value, e.value

    def select_kernel(self, B, H, N, d, dtype=torch.bfloat16, bias=None) -> str:
        p = self._params(B, H, N, d, dtype, bias)
        k = self.lib.ba_select_kernel(C.byref(p))
        return {1: "simt", 2: "tcgen05"}.get(k, "none")

    # ------------------------------------------------------------------------------------------
    def pack_signs(self, X: torch.Tensor):
        """binary_quantize for every head: returns (words int64 [B,H,N,ceil(d/64)] holding the u64 bit patterns, mu fp32 [B,H])."""
        if X.dim() != 4:
            raise ShapeError("pack_signs: X must be [B,H,N,d]")
        X = X.contiguous()
        B, H, N, d = X.shape
        if X.numel() == 0:
            raise ShapeError("binary_quantize: empty matrix")  # quantize.cpp:17
        words = torch.empty((B, H, N, (d + 63) // 64), dtype=torch.int64, device=X.device)
        mu = torch.empty((B, H), dtype=torch.float32, device=X.device)
        p = self._params(B, H, N, d, X.dtype)
        _check(self.lib.ba_pack_signs(self.h, C.byref(p), _ptr(X), _ptr(words), _ptr(mu), self._stream()))
        return words, mu

    def quantize_values(self, V: torch.Tensor):
        """quantize_values for every head (quantize.cpp:57-74): returns (levels int8 [B,H,N,d], scales float64 [B,H,d])."""
        if V.dim() != 4:
            raise ShapeError("quantize_values: V must be [B,H,N,d]")
        V = V.contiguous()
        B, H, N, d = V.shape
        vq = torch.empty((B, H, N, d), dtype=torch.int8, device=V.device)
        sc = torch.empty((B, H, d), dtype=torch.float64, device=V.device)
        p = self._params(B, H, N, d, V.dtype)
        _check(self.lib.ba_quantize_values(self.h, C.byref(p), _ptr(V), _ptr(vq), _ptr(sc), self._stream()))
        return vq, sc

    def binary_logits(self, q_words: torch.Tensor, k_words: torch.Tensor, d: int, head: int = 0) -> torch.Tensor:
        """binary_gemm for one head: int32 [N,N] = d - 2*popc(q xor k)."""
        B, H, N, _ = q_words.shape
        S = torch.empty((N, N), dtype=torch.int32, device=q_words.device)
        p = self._params(B, H, N, d, torch.bfloat16)
        _check(self.lib.ba_binary_logits(self.h, C.byref(p), _ptr(q_words.contiguous()), _ptr(k_words.contiguous()),
                                         head, _ptr(S), self._stream()))
        return S

    def attention_probs(self, Q, K, bias=None, scale=None, head: int = 0, rows=None, binary: bool = True) -> torch.Tensor:
        """Attention-map rows of one head, float64 [len(rows), N] (the reference's `with_probs` output restricted to
        sampled query rows): binary=True follows binary_attention_unfused (attention.cpp:149-248), binary=False the
        full-precision reference_attention (attention.cpp:99-147).  `head` indexes the flattened [B*H] grid."""
        if Q.dim() != 4 or K.shape != Q.shape:
            raise ShapeError("attention: Q, K must be [B,H,N,d]")
        B, H, N, d = Q.shape
        Q, K = Q.contiguous(), K.contiguous()
        bias, bias_t = self._check_bias(bias, H, N)
        p = self._params(B, H, N, d, Q.dtype, bias, scale)
        rows_t = torch.arange(N, device=Q.device, dtype=torch.int32) if rows is None else \
            torch.as_tensor(rows, dtype=torch.int32).to(Q.device).contiguous()
        if rows_t.numel() < 1 or int(rows_t.min()) < 0 or int(rows_t.max()) >= N:
            raise ShapeError("attention_probs: rows must be a non-empty list of indices in [0, N)")
        P = torch.empty((rows_t.numel(), N), dtype=torch.float64, device=Q.device)
        _check(self.lib.ba_attention_probs(self.h, C.byref(p), 1 if binary else 0, _ptr(Q), _ptr(K), _ptr(bias_t), head,
                                           _ptr(rows_t), rows_t.numel(), _ptr(P), self._stream()))
        return P

    def attention_fidelity(self, p_ref: torch.Tensor, p_other: torch.Tensor, k: int) -> "FidelityReport":
        """attention_fidelity (fidelity.cpp:40-85) of two row-stochastic [rows, cols] device matrices."""
        if p_ref.dim() != 2 or p_ref.shape != p_other.shape:
            raise ShapeError("attention_fidelity: shape mismatch")  # fidelity.cpp:42-43
        a = p_ref.to(torch.float64).contiguous()
        b = p_other.to(torch.float64).contiguous()
        out = _Fidelity()
        _check(self.lib.ba_attention_fidelity(self.h, _ptr(a), _ptr(b), a.shape[0], a.shape[1], int(k), C.byref(out), self._stream()))
        return FidelityReport(out.cos_sim, out.relative_l1, out.rmse, out.precision_at_k, int(k))

    def forward(self, Q, K, V, bias=None, scale=None, kernel="auto", return_stats=False, quantize_pv=False, block_cols=None,
                units=None, out=None, out_dtype=torch.float32):
        """binary_attention(Q, K, V, bias, scale) -> O for [B,H,N,d] device tensors.  O is float32 like the reference's
        output; out_dtype=torch.bfloat16 (ba_params.out_bf16) has the kernel's epilogue write the same values rounded to
        bfloat16 (nearest-even) instead -- bit-identical to forward(...).to(torch.bfloat16), half the output bytes.
        quantize_pv=True selects the reference's default u8 x s8 integer P.V mode (attention.hpp:35; CUDA-core kernel);
        block_cols is that mode's key-block size (default min(64, N), like AttentionConfig::make).
        units=(begin, end): compute only those (head, 256-row block) units of the flattened grid (ba_shard_units); the other
        rows of `out` (zeros when not given) are left untouched."""
        if Q.dim() != 4:
            raise ShapeError("attention: Q must be [B,H,N,d]")
        if K.shape != Q.shape:
            raise ShapeError("attention: K must be N x d")  # attention.cpp:22
        if V.shape != Q.shape:
            raise ShapeError("attention: V must be N x d")  # attention.cpp:23
        if not (Q.dtype == K.dtype == V.dtype):
            raise ValidationError("Q, K, V must share one dtype")
        B, H, N, d = Q.shape
        Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
        bias, bias_t = self._check_bias(bias, H, N)
        p = self._params(B, H, N, d, Q.dtype, bias, scale, kernel, quantize_pv, block_cols)
        if units is not None:
            p.unit_begin, p.unit_end = int(units[0]), int(units[1])
            if p.unit_begin == p.unit_end:
                p.unit_begin = p.unit_end = -1  # (0, 0 means "everything" in the ABI; an empty range must stay empty)
        if out_dtype not in (torch.float32, torch.bfloat16):
            raise ValidationError("out_dtype must be torch.float32 or torch.bfloat16")
        p.out_bf16 = 1 if out_dtype == torch.bfloat16 else 0
        if out is not None:
            if out.shape != (B, H, N, d) or out.dtype != out_dtype or not out.is_contiguous():
                raise ShapeError(f"attention: out must be a contiguous {out_dtype} [B,H,N,d] tensor")
            O = out
        else:
            O = (torch.zeros if units is not None else torch.empty)((B, H, N, d), dtype=out_dtype, device=Q.device)
        if units is not None and p.unit_begin < 0:
            return O
        m = torch.empty((B, H, N), dtype=torch.float32, device=Q.device) if return_stats else None
        l = torch.empty((B, H, N), dtype=torch.float32, device=Q.device) if return_stats else None
        _check(self.lib.ba_binary_attention_fwd(self.h, C.byref(p), _ptr(Q), _ptr(K), _ptr(V), _ptr(bias_t), _ptr(O),
                                                _ptr(m), _ptr(l), None, self._stream()))
        return (O, m, l) if return_stats else O

    def forward_host(self, Q, K, V, bias=None, scale=None, kernel="auto", out=None, out_dtype=torch.float32, quantize_pv=False,
                     block_cols=None):
        """Same call with HOST tensors (ideally pinned): H2D + kernels + D2H inside ba_binary_attention_host."""
        if Q.is_cuda or K.is_cuda or V.is_cuda:
            raise ValidationError("forward_host takes CPU tensors")
        if K.shape != Q.shape or V.shape != Q.shape or Q.dim() != 4:
            raise ShapeError("attention: Q, K, V must be [B,H,N,d]")
        B, H, N, d = Q.shape
        Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
        bias, bias_t = self._check_bias(bias, H, N)
        if bias_t is not None and not isinstance(bias, (Relative1dBias, Relative2dBias)) and not bias_t.is_cuda:
            bias = bias_t = bias_t.contiguous()
        p = self._params(B, H, N, d, Q.dtype, bias, scale, kernel, quantize_pv, block_cols)
        p.bias_on_device = 1 if (bias_t is not None and bias_t.is_cuda) else 0  # a table that already lives on the GPU (a model parameter)
        if out_dtype not in (torch.float32, torch.bfloat16):
            raise ValidationError("out_dtype must be torch.float32 or torch.bfloat16")
        p.out_bf16 = 1 if out_dtype == torch.bfloat16 else 0
        if out is None:
            out = torch.empty((B, H, N, d), dtype=out_dtype, pin_memory=True)
        elif out.shape != (B, H, N, d) or out.dtype != out_dtype or not out.is_contiguous():
            raise ShapeError(f"attention: out must be a contiguous {out_dtype} [B,H,N,d] tensor")
        _check(self.lib.ba_binary_attention_host(self.h, C.byref(p), _ptr(Q), _ptr(K), _ptr(V), _ptr(bias_t), _ptr(out),
                                                 None, None))
        return out


_handles: dict[int, BinaryAttention] = {}


def _handle_for(device: torch.device) -> BinaryAttention:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _handles:
        _handles[idx] = BinaryAttention(torch.device("cuda", idx))
    return _handles[idx]


def binary_attention(Q, K, V, bias=None, scale=None, kernel="auto"):
    """BASELINE.json's operator: binary_attention(Q, K, V, bias, scale) -> O.

    Q, K, V: [B,H,N,d] CUDA tensors (bf16 for the tcgen05 kernel; fp16/fp32 run the CUDA-core kernel);
    bias: None, dense [N,N] / [1|H,N,N] (bf16 or fp32) or Relative1dBias(offsets [1|H, 2N-1]), added before the softmax; scale = 1/temperature
    (default 1/sqrt(d)).  The per-head factor mu_q*mu_k is computed inside, as in the reference."""
    if not Q.is_cuda:
        raise CudaError("binary_attention needs CUDA tensors: this package has no CPU fallback")
    return _handle_for(Q.device).forward(Q, K, V, bias, scale, kernel)


def binary_attention_fused(q, k, v, cfg: AttentionConfig, with_probs: bool = False) -> AttentionOutput:
    """Drop-in shaped like binattn::binary_attention_fused (attention.hpp:69-71): one head, [N,d] tensors."""
    n, d = cfg.seq_len, cfg.head_dim
    for name, t in (("Q", q), ("K", k), ("V", v)):  # attention.cpp:21-23
        if t.dim() != 2 or t.shape[0] != n or t.shape[1] != d:
            raise ShapeError(f"attention: {name} must be N x d")
    if not cfg.temperature > 0.0:  # attention.cpp:24-25
        raise ValidationError("attention: temperature must be positive")
    if cfg.block_rows < 1 or cfg.block_rows > n or cfg.block_cols < 1 or cfg.block_cols > n:  # attention.cpp:26-28
        raise ValidationError("attention: block sizes must be in [1, N]")
    if with_probs:
        raise UnsupportedError("with_probs is diagnostics-only in the reference and is not carried over")
    if isinstance(cfg.bias, Relative2dBias):
        pass  # shape rules are checked when the table is expanded (Relative2dBias.materialize)
    elif isinstance(cfg.bias, Relative1dBias):
        if cfg.bias.offsets.dim() != 1 or cfg.bias.offsets.shape[0] != 2 * n - 1:
            raise ShapeError("bias: relative-1d offsets must have length 2N-1")  # attention.cpp:66-67
    elif cfg.bias is not None and (cfg.bias.dim() != 2 or cfg.bias.shape[0] != n or cfg.bias.shape[1] != n):
        raise ShapeError("bias: dense table must be N x N")  # attention.cpp:60-61
    ba = _handle_for(q.device)
    O, m, l = ba.forward(q[None, None], k[None, None], v[None, None], cfg.bias, 1.0 / cfg.temperature,
                         return_stats=True, quantize_pv=cfg.quantize_pv, block_cols=cfg.block_cols)
    return AttentionOutput(O[0, 0], m[0, 0], l[0, 0])
