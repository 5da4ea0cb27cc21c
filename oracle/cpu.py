"""ctypes doorway to the two CPU checkers.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never from the product package.

  port()  -> oracle/libbinattn_oracle.so   (our plain-C restatement, binattn_oracle.c)
  ref()   -> oracle/_ref/libbinattn_ref.so (the unmodified reference, built by oracle/Makefile)

Both expose the same methods; ref() returns None when the prebuilt library is absent.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_f64 = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i8 = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")

ERRORS = {1: "ShapeError", 2: "ValidationError", 3: "MemoryError", 4: "Error"}


class CpuError(RuntimeError):
    def __init__(self, code):
        super().__init__(ERRORS.get(code, f"rc={code}"))
        self.code = code
        self.kind = ERRORS.get(code, "Error")


def _opt(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def words_needed(d: int) -> int:
    return (d + 63) // 64


class CpuLib:
    """Same surface for the C port (prefix 'bo_') and the compiled reference (prefix 'ref_')."""

    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.p = prefix
        self.is_reference = prefix == "ref_"
        L, p, sz = self.lib, prefix, C.c_size_t
        getattr(L, p + "pack_signs").argtypes = [_f64, sz, sz, _u64]
        getattr(L, p + "binary_quantize").argtypes = [_f64, sz, sz, _u64, C.POINTER(C.c_double)]
        getattr(L, p + "binary_quantize").restype = C.c_int
        getattr(L, p + "xnor_popcount_dot").argtypes = [_u64, _u64, sz]
        getattr(L, p + "xnor_popcount_dot").restype = C.c_int64
        getattr(L, p + "hamming_distance").argtypes = [_u64, _u64, sz]
        getattr(L, p + "hamming_distance").restype = C.c_uint64
        getattr(L, p + "binary_gemm").argtypes = [_u64, sz, _u64, sz, sz, _i32]
        getattr(L, p + "quantize_values").argtypes = [_f64, sz, sz, _i8, _f64]
        getattr(L, p + "materialize_bias_rel1d").argtypes = [_f64, sz, _f64]
        vp = C.c_void_p
        getattr(L, p + "reference_attention").argtypes = [_f64, _f64, _f64, sz, sz, C.c_double, vp, _f64, _f64, _f64, vp]
        getattr(L, p + "binary_attention_unfused").argtypes = [_f64, _f64, _f64, sz, sz, C.c_double, C.c_int, vp, _f64, _f64, _f64, vp]
        getattr(L, p + "binary_attention_fused").argtypes = [_f64, _f64, _f64, sz, sz, C.c_double, sz, sz, C.c_int, vp, _f64, _f64, _f64]
        getattr(L, p + "attention_fidelity").argtypes = [_f64, _f64, sz, sz, sz, _f64]
        if self.is_reference:
            L.ref_materialize_bias_rel2d.argtypes = [_f64, _f64, sz, sz, _f64]
            L.ref_rng_new.restype = vp
            L.ref_rng_new.argtypes = [C.c_uint64, C.c_uint64]
            L.ref_rng_free.argtypes = [vp]
            L.ref_rng_u64.argtypes = [vp]
            L.ref_rng_u64.restype = C.c_uint64
            L.ref_random_dense.argtypes = [vp, sz, C.c_double, _f64]
            L.ref_binary_attention_fused_heads.argtypes = [_f64, _f64, _f64, sz, sz, sz, C.c_double, sz, sz, C.c_int, vp, sz, _f64, C.c_int, C.c_int]
        else:
            L.bo_materialize_bias_rel2d.argtypes = [_f64, _f64, sz, _f64]
            L.bo_rng_sizeof.restype = sz
            L.bo_rng_init.argtypes = [vp, C.c_uint64, C.c_uint64]
            L.bo_rng_u64.argtypes = [vp]
            L.bo_rng_u64.restype = C.c_uint64
            L.bo_random_dense.argtypes = [vp, sz, C.c_double, _f64]
            L.bo_binary_attention_fused_heads.argtypes = [_f64, _f64, _f64, sz, sz, sz, C.c_double, sz, sz, C.c_int, vp, sz, _f64, C.c_int]

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    @staticmethod
    def _chk(rc):
        if rc:
            raise CpuError(rc)

    # --- rng (rng.hpp; tests/oracles.hpp random_dense) -------------------------------------------
    def make_rng(self, seed: int, stream: int = 0):
        if self.is_reference:
            return _RefRng(self.lib, seed, stream)
        return _PortRng(self.lib, seed, stream)

    # --- bitops / quantize -------------------------------------------------------------------------
    def pack_signs(self, m: np.ndarray) -> np.ndarray:
        m = np.ascontiguousarray(m, dtype=np.float64)
        rows, d = m.shape
        out = np.zeros((rows, words_needed(d)), dtype=np.uint64)
        rc = self._f("pack_signs")(m, rows, d, out)
        if self.is_reference:  # the port's version returns void
            self._chk(rc)
        return out

    def binary_quantize(self, m: np.ndarray):
        m = np.ascontiguousarray(m, dtype=np.float64)
        rows, d = m.shape
        out = np.zeros((rows, words_needed(d)), dtype=np.uint64)
        mu = C.c_double(0.0)
        self._chk(self._f("binary_quantize")(m, rows, d, out, C.byref(mu)))
        return out, mu.value

    def xnor_popcount_dot(self, a: np.ndarray, b: np.ndarray, d: int) -> int:
        return int(self._f("xnor_popcount_dot")(np.ascontiguousarray(a, dtype=np.uint64), np.ascontiguousarray(b, dtype=np.uint64), d))

    def hamming_distance(self, a: np.ndarray, b: np.ndarray, d: int) -> int:
        return int(self._f("hamming_distance")(np.ascontiguousarray(a, dtype=np.uint64), np.ascontiguousarray(b, dtype=np.uint64), d))

    def binary_gemm(self, s: np.ndarray, t: np.ndarray, d: int) -> np.ndarray:
        s = np.ascontiguousarray(s, dtype=np.uint64)
        t = np.ascontiguousarray(t, dtype=np.uint64)
        out = np.zeros((s.shape[0], t.shape[0]), dtype=np.int32)
        rc = self._f("binary_gemm")(s, s.shape[0], t, t.shape[0], d, out)
        if self.is_reference:
            self._chk(rc)
        return out

    def quantize_values(self, v: np.ndarray):
        v = np.ascontiguousarray(v, dtype=np.float64)
        data = np.zeros(v.shape, dtype=np.int8)
        scales = np.zeros(v.shape[1], dtype=np.float64)
        self._f("quantize_values")(v, v.shape[0], v.shape[1], data, scales)
        return data, scales

    # --- bias ----------------------------------------------------------------------------------------
    def bias_rel1d(self, offsets: np.ndarray, n: int) -> np.ndarray:
        offsets = np.ascontiguousarray(offsets, dtype=np.float64)
        if offsets.size != 2 * n - 1:
            raise CpuError(1)
        out = np.zeros((n, n), dtype=np.float64)
        self._f("materialize_bias_rel1d")(offsets, n, out)
        return out

    def bias_rel2d(self, row_off: np.ndarray, col_off: np.ndarray, n: int) -> np.ndarray:
        row_off = np.ascontiguousarray(row_off, dtype=np.float64)
        col_off = np.ascontiguousarray(col_off, dtype=np.float64)
        out = np.zeros((n, n), dtype=np.float64)
        if self.is_reference:
            self._chk(self.lib.ref_materialize_bias_rel2d(row_off, col_off, row_off.size, n, out))
        else:
            g = int(round(n ** 0.5))
            if g * g != n or row_off.size != 2 * g - 1 or col_off.size != 2 * g - 1:
                raise CpuError(1)
            self._chk(self.lib.bo_materialize_bias_rel2d(row_off, col_off, n, out))
        return out

    # --- attention -------------------------------------------------------------------------------------
    @staticmethod
    def _prep(q, k, v, bias):
        q = np.ascontiguousarray(q, dtype=np.float64)
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        n, d = q.shape
        if k.shape != (n, d) or v.shape != (n, d):
            raise CpuError(1)  # attention.cpp:21-23 ShapeError
        if bias is not None:
            bias = np.ascontiguousarray(bias, dtype=np.float64)
            if bias.shape != (n, n):
                raise CpuError(1)  # attention.cpp:60-61
        return q, k, v, bias, n, d

    def reference_attention(self, q, k, v, tau=None, bias=None, with_probs=False):
        q, k, v, bias, n, d = self._prep(q, k, v, bias)
        tau = float(np.sqrt(d)) if tau is None else tau
        y, m, l = np.zeros((n, d)), np.zeros(n), np.zeros(n)
        probs = np.zeros((n, n)) if with_probs else None
        self._chk(self._f("reference_attention")(q, k, v, n, d, tau, _opt(bias), y, m, l, _opt(probs)))
        return (y, m, l, probs) if with_probs else (y, m, l)

    def binary_attention_unfused(self, q, k, v, tau=None, bias=None, quantize_pv=False, with_probs=False):
        q, k, v, bias, n, d = self._prep(q, k, v, bias)
        tau = float(np.sqrt(d)) if tau is None else tau
        y, m, l = np.zeros((n, d)), np.zeros(n), np.zeros(n)
        probs = np.zeros((n, n)) if with_probs else None
        self._chk(self._f("binary_attention_unfused")(q, k, v, n, d, tau, int(quantize_pv), _opt(bias), y, m, l, _opt(probs)))
        return (y, m, l, probs) if with_probs else (y, m, l)

    def binary_attention_fused(self, q, k, v, tau=None, bias=None, quantize_pv=False, block_rows=None, block_cols=None):
        """attention.cpp:250; defaults follow AttentionConfig::make (attention.cpp:45-53)."""
        q, k, v, bias, n, d = self._prep(q, k, v, bias)
        tau = float(np.sqrt(d)) if tau is None else tau
        br = min(64, n) if block_rows is None else block_rows
        bc = min(64, n) if block_cols is None else block_cols
        y, m, l = np.zeros((n, d)), np.zeros(n), np.zeros(n)
        self._chk(self._f("binary_attention_fused")(q, k, v, n, d, tau, br, bc, int(quantize_pv), _opt(bias), y, m, l))
        return y, m, l

    def attention_fidelity(self, p_ref, p_other, k: int):
        """fidelity.cpp:40-85 -> (cos_sim, relative_l1, rmse, precision_at_k)."""
        p_ref = np.ascontiguousarray(p_ref, dtype=np.float64)
        p_other = np.ascontiguousarray(p_other, dtype=np.float64)
        if p_ref.ndim != 2 or p_ref.shape != p_other.shape:
            raise CpuError(1)  # fidelity.cpp:42-43 ShapeError
        out = np.zeros(4)
        self._chk(self._f("attention_fidelity")(p_ref, p_other, p_ref.shape[0], p_ref.shape[1], k, out))
        return tuple(float(x) for x in out)

    def binary_attention_fused_heads(self, q, k, v, tau=None, bias=None, quantize_pv=False, nthreads=1, intra_threads=1):
        """q,k,v: [heads, n, d] float64; bias: [bias_heads, n, n] or None.  Heads spread over host threads."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        heads, n, d = q.shape
        tau = float(np.sqrt(d)) if tau is None else tau
        bh = 0
        if bias is not None:
            bias = np.ascontiguousarray(bias, dtype=np.float64)
            bh = bias.shape[0]
        y = np.zeros_like(q)
        br = bc = min(64, n)
        if self.is_reference:
            rc = self.lib.ref_binary_attention_fused_heads(q, k, v, heads, n, d, tau, br, bc, int(quantize_pv), _opt(bias), bh, y, nthreads, intra_threads)
        else:
            rc = self.lib.bo_binary_attention_fused_heads(q, k, v, heads, n, d, tau, br, bc, int(quantize_pv), _opt(bias), bh, y, nthreads)
        self._chk(rc)
        return y


class _PortRng:
    def __init__(self, lib, seed, stream):
        self.lib = lib
        self.buf = C.create_string_buffer(lib.bo_rng_sizeof())
        lib.bo_rng_init(self.buf, seed, stream)

    def u64(self) -> int:
        return int(self.lib.bo_rng_u64(self.buf))

    def random_dense(self, rows, cols, scale=1.0) -> np.ndarray:
        out = np.zeros((rows, cols), dtype=np.float64)
        self.lib.bo_random_dense(self.buf, rows * cols, scale, out)
        return out


class _RefRng:
    def __init__(self, lib, seed, stream):
        self.lib = lib
        self.h = lib.ref_rng_new(seed, stream)

    def __del__(self):
        try:
            self.lib.ref_rng_free(self.h)
        except Exception:
            pass

    def u64(self) -> int:
        return int(self.lib.ref_rng_u64(self.h))

    def random_dense(self, rows, cols, scale=1.0) -> np.ndarray:
        out = np.zeros((rows, cols), dtype=np.float64)
        self.lib.ref_random_dense(self.h, rows * cols, scale, out)
        return out


_PORT = None
_REF = None


def build(quiet: bool = True) -> None:
    """Compile the C port and, when /root/reference is present, oracle/_ref."""
    subprocess.run(["make", "-C", HERE, "all"], check=True, capture_output=quiet)


def port() -> CpuLib:
    global _PORT
    if _PORT is None:
        path = os.path.join(HERE, "libbinattn_oracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", HERE, "liboracle"], check=True, capture_output=True)
        _PORT = CpuLib(path, "bo_")
    return _PORT


def ref() -> CpuLib | None:
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libbinattn_ref.so")
        if not os.path.exists(path):
            if os.path.isdir("/root/reference/proj/src"):
                subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)
            if not os.path.exists(path):
                return None
        _REF = CpuLib(path, "ref_")
    return _REF


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64/float32 values to bfloat16 (round-to-nearest-even), returned as float64.

    The CUDA path consumes bf16 tensors; the CPU checkers must see the SAME rounded values
    (a tiny negative that rounds to -0 flips the x >= 0 sign rule)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(x))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16-representable float values -> uint16 bit patterns (for torch.bfloat16 views)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16).reshape(np.shape(x))
