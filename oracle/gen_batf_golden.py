"""Write tests/golden/batf/*.batf with the UNMODIFIED reference writer (oracle/_ref: tensor_file.cpp:85-125).

Run here (the container that has /root/reference):   python -m oracle.gen_batf_golden
The files are small fixtures: the Python BATF reader/writer (paper_2603_09582_b200/batf.py) must read them exactly and
must produce byte-identical files from the same values.  Cases follow the reference's own file-format tests
(proj/tests/test_tensor_io.cpp:57-104) plus a packed sign plane of a real head shape."""
import ctypes as C
import os

import numpy as np

from oracle import cpu

OUT = os.path.join(os.path.dirname(cpu.HERE), "tests", "golden", "batf")


def ref_file_api():
    R = cpu.ref()
    assert R is not None, "oracle/_ref missing: run `make -C oracle ref` where /root/reference exists"
    L = R.lib
    L.ref_write_dense.argtypes = [C.c_char_p, np.ctypeslib.ndpointer(np.float64, flags="C"), C.c_size_t, C.c_size_t, C.c_int]
    L.ref_write_bits.argtypes = [C.c_char_p, np.ctypeslib.ndpointer(np.uint64, flags="C"), C.c_size_t, C.c_size_t]
    return R, L


def main():
    R, L = ref_file_api()
    os.makedirs(OUT, exist_ok=True)
    w = lambda name: os.path.join(OUT, name).encode()
    eye = np.array([[1.0, 0.0], [0.0, 1.0]])
    assert L.ref_write_dense(w("eye_2x2_f32.batf"), eye, 2, 2, 1) == 0            # test_tensor_io.cpp:57-69
    assert L.ref_write_dense(w("zero_1x1_f64.batf"), np.zeros((1, 1)), 1, 1, 0) == 0  # :71-78
    rng = R.make_rng(5)
    m32 = rng.random_dense(7, 65).astype(np.float32).astype(np.float64)           # :80-95 (seeded 7x65 real32)
    assert L.ref_write_dense(w("rand_7x65_f32.batf"), np.ascontiguousarray(m32), 7, 65, 1) == 0
    m64 = R.make_rng(6).random_dense(3, 5)                                        # :97-104
    assert L.ref_write_dense(w("rand_3x5_f64.batf"), np.ascontiguousarray(m64), 3, 5, 0) == 0
    q = cpu.bf16_round(R.make_rng(0, 0).random_dense(197, 72))                    # a packed sign plane, d = 72 (56 pad bits)
    words = R.pack_signs(q)
    assert L.ref_write_bits(w("signs_197x72_bits.batf"), np.ascontiguousarray(words), 197, 72) == 0
    np.savez_compressed(os.path.join(OUT, "values.npz"), eye=eye, m32=m32, m64=m64, q=q, words=words)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
