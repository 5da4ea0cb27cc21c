"""BATF tensor files: the Python reader/writer against files written by the UNMODIFIED reference
(tests/golden/batf, made by oracle/gen_batf_golden.py), the reference's own format tests (proj/tests/test_tensor_io.cpp),
and -- where oracle/_ref is present -- the reference reader on files we write."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from oracle import cpu
from paper_2603_09582_b200 import batf

G = os.path.join(os.path.dirname(__file__), "golden", "batf")


@pytest.fixture(scope="module")
def vals():
    return np.load(os.path.join(G, "values.npz"))


def test_reads_reference_written_files_exactly(vals):
    t = batf.read_tensor(os.path.join(G, "eye_2x2_f32.batf"))
    assert (t.dtype, t.rows, t.cols) == (batf.F32, 2, 2) and np.array_equal(t.data, vals["eye"])
    assert os.path.getsize(os.path.join(G, "eye_2x2_f32.batf")) == 26 + 16  # test_tensor_io.cpp:57-69
    z = batf.read_tensor(os.path.join(G, "zero_1x1_f64.batf"))
    assert z.dtype == batf.F64 and z.data[0, 0] == 0.0 and not np.signbit(z.data[0, 0])  # :71-78
    assert np.array_equal(batf.read_tensor(os.path.join(G, "rand_7x65_f32.batf")).data, vals["m32"])
    assert np.array_equal(batf.read_tensor(os.path.join(G, "rand_3x5_f64.batf")).data, vals["m64"])
    b = batf.read_tensor(os.path.join(G, "signs_197x72_bits.batf"))
    assert (b.dtype, b.rows, b.cols) == (batf.PACKED_BIT, 197, 72) and np.array_equal(b.data, vals["words"])


@pytest.mark.parametrize("name,key,dtype,cols", [("eye_2x2_f32", "eye", batf.F32, None), ("zero_1x1_f64", None, batf.F64, None),
                                                 ("rand_7x65_f32", "m32", batf.F32, None), ("rand_3x5_f64", "m64", batf.F64, None),
                                                 ("signs_197x72_bits", "words", batf.PACKED_BIT, 72)])
def test_writer_is_byte_identical_to_the_reference(tmp_path, vals, name, key, dtype, cols):
    data = np.zeros((1, 1)) if key is None else vals[key]
    p = tmp_path / "out.batf"
    batf.write_tensor(p, data, dtype, cols=cols)
    assert p.read_bytes() == open(os.path.join(G, name + ".batf"), "rb").read()


def test_round_trip_all_kinds_and_odd_widths(tmp_path):  # test_tensor_io.cpp:162-190
    rng = np.random.default_rng(3)
    for cols in (1, 63, 64, 65, 130):
        p = tmp_path / f"t{cols}.batf"
        d = rng.standard_normal((4, cols))
        batf.write_tensor(p, d, batf.F64)
        assert np.array_equal(batf.read_tensor(p).data, d)
        batf.write_tensor(p, d, batf.F32)
        assert np.array_equal(batf.read_tensor(p).data, d.astype(np.float32).astype(np.float64))
        bits = rng.integers(0, 2, (4, cols)).astype(bool)
        words = np.zeros((4, batf.words_needed(cols)), np.uint64)
        for c in range(cols):
            words[:, c // 64] |= bits[:, c].astype(np.uint64) << np.uint64(c % 64)
        batf.write_tensor(p, words, batf.PACKED_BIT, cols=cols)
        back = batf.read_tensor(p)
        assert back.cols == cols and np.array_equal(back.data, words)
        q = rng.integers(-127, 128, (4, cols)).astype(np.int8)
        sc = rng.uniform(0.01, 2.0, cols)
        batf.write_tensor(p, q, batf.I8, scales=sc)
        back = batf.read_tensor(p)
        assert np.array_equal(back.data, q) and np.array_equal(back.scales, sc)
        u = rng.integers(0, 256, (4, cols)).astype(np.uint8)
        batf.write_tensor(p, u, batf.U8)
        assert np.array_equal(batf.read_tensor(p).data, u)


def test_strict_reader_rejections(tmp_path):  # test_tensor_io.cpp:106-160, 192-196
    good = open(os.path.join(G, "rand_3x5_f64.batf"), "rb").read()
    bits = open(os.path.join(G, "signs_197x72_bits.batf"), "rb").read()

    def bad(raw):
        p = tmp_path / "bad.batf"
        p.write_bytes(raw)
        with pytest.raises(batf.FormatError):
            batf.read_tensor(p)

    bad(b"XATF" + good[4:])                                   # bad magic
    bad(good[:-3])                                            # truncated payload
    bad(good + b"\x00")                                       # trailing bytes
    bad(good[:4] + struct.pack("<I", 2) + good[8:])           # unsupported version
    bad(good[:8] + bytes([9]) + good[9:])                     # unknown dtype code
    bad(good[:9] + bytes([3]) + good[10:])                    # ndim != 2
    tampered = bytearray(bits)
    tampered[26 + 15] |= 0x80                                 # top pad bit of row 0's second word (cols = 72)
    bad(bytes(tampered))                                      # hand-edited pad bit, :128-143
    nan = bytearray(good)
    nan[26:34] = struct.pack("<d", float("nan"))
    bad(bytes(nan))                                           # non-finite payload entry
    q = tmp_path / "q.batf"
    with pytest.raises(batf.FormatError):
        batf.write_tensor(q, np.zeros((2, 2), np.uint64), batf.PACKED_BIT, cols=300)  # wrong words per row
    batf.write_tensor(q, np.array([[-128]], np.int8), batf.I8, scales=np.array([1.0]))
    with pytest.raises(batf.FormatError):
        batf.read_tensor(q)                                   # -128 is not a valid level (tensor.cpp:53-56)
    with pytest.raises(batf.IoError):
        batf.read_tensor(tmp_path / "missing.batf")


def test_reference_reader_accepts_our_files(tmp_path, vals):
    R = cpu.ref()
    if R is None:
        pytest.skip("oracle/_ref not built here")
    L = R.lib
    L.ref_read_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p]
    dt, rows, cols = C.c_int(), C.c_size_t(), C.c_size_t()
    p = tmp_path / "bits.batf"
    batf.write_tensor(p, vals["words"], batf.PACKED_BIT, cols=72)
    words = np.zeros_like(vals["words"])
    assert L.ref_read_tensor(str(p).encode(), C.byref(dt), C.byref(rows), C.byref(cols), None, words.ctypes.data, None, None) == 0
    assert (dt.value, rows.value, cols.value) == (4, 197, 72) and np.array_equal(words, vals["words"])
    p = tmp_path / "dense.batf"
    batf.write_tensor(p, vals["m32"], batf.F32)
    dense = np.zeros((7, 65))
    assert L.ref_read_tensor(str(p).encode(), C.byref(dt), C.byref(rows), C.byref(cols), dense.ctypes.data, None, None, None) == 0
    assert dt.value == 0 and np.array_equal(dense, vals["m32"])
    tampered = bytearray(p.read_bytes())
    tampered[0] = ord("X")
    p.write_bytes(bytes(tampered))
    assert L.ref_read_tensor(str(p).encode(), C.byref(dt), C.byref(rows), C.byref(cols), None, None, None, None) == 2  # FormatError
