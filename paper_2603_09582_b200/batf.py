"""BATF v1 tensor files -- the reference's bit-exact interchange format (proj/include/binattn/tensor_file.hpp:11-23,
proj/src/tensor_file.cpp:23-34, 127-189), so the CUDA driver and the reference can exchange Q/K/V, packed sign planes
(dtype 4) and outputs as files (the reference CLI's `demo --save-tensors` writes Q/K/V, binattn_cli.cpp:557-564).

Layout, all little-endian: magic "BATF" | version u32 = 1 | dtype u8 (0 f32, 1 f64, 2 int8, 3 uint8, 4 packed-bit) |
ndim u8 = 2 | rows u64 | cols u64 | payload (row-major; int8 is followed by `cols` f64 channel scales; packed-bit is
rows x ceil(cols/64) u64 words with zero pad bits).  The reader is as strict as the reference's: bad magic, version,
dtype code, ndim, truncation, trailing bytes, non-finite values, -128 levels, non-positive scales and non-zero pad bits
are all FormatError.  Host-side file IO only: nothing here runs on the hot path.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np

MAGIC = b"BATF"
VERSION = 1
F32, F64, I8, U8, PACKED_BIT = 0, 1, 2, 3, 4
HEADER_BYTES = 26


class FormatError(ValueError):
    """binattn::FormatError (errors.hpp:28-31)."""


class IoError(OSError):
    """binattn::IoError (errors.hpp:40-43)."""


@dataclass
class Tensor:
    """One BATF tensor.  dtype F32/F64: data float64 [rows, cols] (F32 values are float32-representable);
    I8: data int8 + scales float64 [cols]; U8: data uint8; PACKED_BIT: data uint64 [rows, ceil(cols/64)], cols = bits."""
    dtype: int
    rows: int
    cols: int
    data: np.ndarray
    scales: Optional[np.ndarray] = None


def words_needed(cols: int) -> int:  # BitMatrix::words_needed, tensor.hpp:57-94
    return (cols + 63) // 64


def _check_pad_bits(words: np.ndarray, cols: int) -> None:
    wpr = words_needed(cols)
    if cols % 64 != 0 and wpr > 0 and words.size:
        mask = np.uint64((1 << (cols % 64)) - 1)
        if np.any(words.reshape(-1, wpr)[:, wpr - 1] & ~mask):
            raise FormatError("nonzero pad bits in packed-bit payload")


def write_tensor(path, data: np.ndarray, dtype: int, cols: Optional[int] = None, scales: Optional[np.ndarray] = None) -> None:
    """write_tensor overloads of tensor_file.cpp:85-125.  `cols` is the logical bit count for PACKED_BIT."""
    a = np.asarray(data)
    if a.ndim != 2:
        raise FormatError("expected a 2-d tensor")
    rows = a.shape[0]
    if dtype == F32:
        payload = np.ascontiguousarray(a, dtype="<f4").tobytes()
        ncols = a.shape[1]
    elif dtype == F64:
        payload = np.ascontiguousarray(a, dtype="<f8").tobytes()
        ncols = a.shape[1]
    elif dtype == I8:
        if scales is None or np.asarray(scales).shape != (a.shape[1],):
            raise FormatError("int8 tensors carry one f64 scale per column")
        payload = np.ascontiguousarray(a, dtype=np.int8).tobytes() + np.ascontiguousarray(scales, dtype="<f8").tobytes()
        ncols = a.shape[1]
    elif dtype == U8:
        payload = np.ascontiguousarray(a, dtype=np.uint8).tobytes()
        ncols = a.shape[1]
    elif dtype == PACKED_BIT:
        if cols is None:
            raise FormatError("packed-bit tensors need the logical column count")
        w = np.ascontiguousarray(a).view(np.uint64) if a.dtype == np.int64 else np.ascontiguousarray(a, dtype="<u8")
        if w.shape[1] != words_needed(cols):
            raise FormatError("packed-bit tensors have ceil(cols/64) words per row")
        _check_pad_bits(w, cols)
        payload = w.tobytes()
        ncols = cols
    else:
        raise FormatError("unknown dtype code")
    header = MAGIC + struct.pack("<IBBQQ", VERSION, dtype, 2, rows, ncols)
    try:
        with open(path, "wb") as f:
            f.write(header + payload)
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


def read_tensor(path) -> Tensor:
    """read_tensor of tensor_file.cpp:127-189, same acceptance rules."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError(f"cannot open for reading: {path}") from e
    if len(raw) < 4 or raw[:4] != MAGIC:
        raise FormatError("bad magic")
    if len(raw) < HEADER_BYTES:
        raise FormatError("truncated tensor file")
    version, dt, ndim, rows, cols = struct.unpack("<IBBQQ", raw[4:HEADER_BYTES])
    if version != VERSION:
        raise FormatError("unsupported version")
    if dt > 4:
        raise FormatError("unknown dtype code")
    if ndim != 2:
        raise FormatError("expected a 2-d tensor")
    if rows != 0 and cols > (2**64 - 1) // rows:
        raise FormatError("dimension overflow")
    if rows * cols > (1 << 34):
        raise FormatError("tensor too large")
    body = raw[HEADER_BYTES:]
    count = rows * cols

    def take(nbytes):
        nonlocal body
        if len(body) < nbytes:
            raise FormatError("truncated tensor file")
        head, body = body[:nbytes], body[nbytes:]
        return head

    if dt in (F32, F64):
        item = "<f4" if dt == F32 else "<f8"
        vals = np.frombuffer(take(count * (4 if dt == F32 else 8)), dtype=item).astype(np.float64).reshape(rows, cols)
        t = Tensor(dt, rows, cols, vals)
        if not np.all(np.isfinite(vals)):
            raise FormatError("non-finite payload entry")
    elif dt == I8:
        vals = np.frombuffer(take(count), dtype=np.int8).reshape(rows, cols).copy()
        sc = np.frombuffer(take(cols * 8), dtype="<f8").copy()
        if np.any(vals == -128):
            raise FormatError("invalid int8 payload: QuantizedValues: -128 is not a valid level")
        if not np.all(np.isfinite(sc)) or np.any(~(sc > 0.0)):
            raise FormatError("invalid int8 payload: QuantizedValues: channel scale must be positive finite")
        t = Tensor(dt, rows, cols, vals, sc)
    elif dt == U8:
        t = Tensor(dt, rows, cols, np.frombuffer(take(count), dtype=np.uint8).reshape(rows, cols).copy())
    else:
        wpr = words_needed(cols)
        words = np.frombuffer(take(rows * wpr * 8), dtype="<u8").reshape(rows, wpr).copy()
        _check_pad_bits(words, cols)
        t = Tensor(dt, rows, cols, words)
    if body:
        raise FormatError("trailing bytes after payload")
    return t
