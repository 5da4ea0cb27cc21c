"""Generate tests/golden/binattn_golden.npz by running the UNMODIFIED reference (oracle/_ref).

Run here (the container that has /root/reference):   python -m oracle.gen_golden
The GPU box has no /root/reference; it uses the committed .npz.  Every case stores the seed recipe
(so inputs are regenerable through the pinned rng of rng.hpp), the inputs themselves, and the
reference's outputs.  Cases mirror the reference's own tests (file:line in each `src` field) plus one
head at the BASELINE.json shapes with bf16-rounded inputs (the dtype the CUDA path consumes).
"""
import json
import os

import numpy as np

from oracle import cpu

OUT = os.path.join(os.path.dirname(cpu.HERE), "tests", "golden", "binattn_golden.npz")


def main():
    R = cpu.ref()
    assert R is not None, "oracle/_ref missing: run `make -C oracle ref` where /root/reference exists"
    arrays, meta = {}, {}

    def put(case, **kw):
        for k, v in kw.items():
            arrays[f"{case}/{k}"] = np.asarray(v)

    # ---- bitops (proj/tests/test_bitops.cpp) ------------------------------------------------------
    rng = R.make_rng(11)
    m = rng.random_dense(3, 130)
    put("pack_seed11", m=m, words=R.pack_signs(m))
    meta["pack_seed11"] = {"src": "test_bitops.cpp:25-33", "seed": 11, "shape": [3, 130]}

    rng = R.make_rng(15)
    a, b = rng.random_dense(8, 96), rng.random_dense(8, 96)
    put("gemm_seed15", a=a, b=b, g=R.binary_gemm(R.pack_signs(a), R.pack_signs(b), 96))
    meta["gemm_seed15"] = {"src": "test_bitops.cpp:136-145", "seed": 15, "shape": [8, 8, 96]}

    rng = R.make_rng(17)
    a, b = rng.random_dense(97, 129), rng.random_dense(83, 129)
    put("gemm_seed17", a=a, b=b, g=R.binary_gemm(R.pack_signs(a), R.pack_signs(b), 129))
    meta["gemm_seed17"] = {"src": "test_bitops.cpp:155-165", "seed": 17, "shape": [97, 83, 129]}

    # ---- quantize (proj/tests/test_quantize.cpp) ---------------------------------------------------
    rng = R.make_rng(21)
    m = rng.random_dense(16, 64)
    w, mu = R.binary_quantize(m)
    put("quant_seed21", m=m, words=w, mu=mu)
    meta["quant_seed21"] = {"src": "test_quantize.cpp:26-33", "seed": 21, "shape": [16, 64]}

    # ---- attention (proj/tests/test_attention.cpp) -------------------------------------------------
    def attn_case(name, src, seed, n, d, bias_scale=None, br=None, bc=None, draws_before=0):
        rng = R.make_rng(seed)
        for _ in range(draws_before):
            rng.u64()
        q, k, v = rng.random_dense(n, d), rng.random_dense(n, d), rng.random_dense(n, d)
        bias = rng.random_dense(n, n, bias_scale) if bias_scale else None
        yu, mu_, lu = R.binary_attention_unfused(q, k, v, bias=bias, quantize_pv=False)
        yf, mf, lf = R.binary_attention_fused(q, k, v, bias=bias, quantize_pv=False, block_rows=br, block_cols=bc)
        yq = R.binary_attention_fused(q, k, v, bias=bias, quantize_pv=True, block_rows=br, block_cols=bc)[0]
        qw, muq = R.binary_quantize(q)
        kw, muk = R.binary_quantize(k)
        put(name, q=q, k=k, v=v, y_unfused=yu, m_unfused=mu_, l_unfused=lu, y_fused=yf, m_fused=mf, l_fused=lf,
            y_fused_int8=yq, q_words=qw, k_words=kw, mu=np.array([muq, muk]), logits=R.binary_gemm(qw, kw, d))
        if bias is not None:
            put(name, bias=bias)
        meta[name] = {"src": src, "seed": seed, "n": n, "d": d, "bias_scale": bias_scale, "block_rows": br,
                      "block_cols": bc}

    attn_case("attn_seed35", "test_attention.cpp:176-208", 35, 12, 16)
    attn_case("attn_seed38", "test_attention.cpp:254-272", 38, 48, 16, bias_scale=0.4, br=3, bc=5)
    attn_case("attn_seed40", "test_attention.cpp:300-314", 40, 64, 32, br=16, bc=16)
    attn_case("attn_seed43", "test_attention.cpp:349-365", 43, 50, 12, br=7, bc=9)

    # seed 37: three shapes drawn from ONE rng stream (test_attention.cpp:234-252)
    rng = R.make_rng(37)
    for idx, (n, d) in enumerate([(7, 16), (64, 16), (33, 5)]):
        q, k, v = rng.random_dense(n, d), rng.random_dense(n, d), rng.random_dense(n, d)
        yu, mu_, lu = R.binary_attention_unfused(q, k, v, quantize_pv=False)
        yf, mf, lf = R.binary_attention_fused(q, k, v, quantize_pv=False, block_rows=n, block_cols=n)
        put(f"attn_seed37_{idx}", q=q, k=k, v=v, y_unfused=yu, m_unfused=mu_, l_unfused=lu, y_fused=yf, m_fused=mf,
            l_fused=lf)
        meta[f"attn_seed37_{idx}"] = {"src": "test_attention.cpp:234-252", "seed": 37, "n": n, "d": d,
                                      "block_rows": n, "block_cols": n, "stream_index": idx}

    # ---- one head at the BASELINE.json shapes, bf16-rounded inputs, dense bias sigma=0.5 ---------------
    # (inputs: seed 0 is the reference CLI default, binattn_cli.cpp:31-35; stream = head index)
    for name, n, d, stream in [("c1_head0", 197, 64, 0), ("c1_head5", 197, 64, 5), ("c3_head0", 256, 72, 0),
                               ("mix_n300_d72", 300, 72, 1), ("mix_n130_d128", 130, 128, 2)]:
        rng = R.make_rng(0, stream)
        q, k, v = (cpu.bf16_round(rng.random_dense(n, d)) for _ in range(3))
        bias = cpu.bf16_round(rng.random_dense(n, n, 0.5))
        qw, muq = R.binary_quantize(q)
        kw, muk = R.binary_quantize(k)
        y, m_, l_ = R.binary_attention_fused(q, k, v, bias=bias, quantize_pv=False)
        y_nb = R.binary_attention_fused(q, k, v, quantize_pv=False)[0]
        y_int8 = R.binary_attention_fused(q, k, v, bias=bias, quantize_pv=True)[0]
        # inputs are regenerable from (seed, stream); only outputs are stored to keep the file small
        put(name, q_words=qw, k_words=kw, mu=np.array([muq, muk]), y=y, m=m_, l=l_, y_nobias=y_nb,
            y_int8=y_int8.astype(np.float32), logits_rows=R.binary_gemm(qw[:4], kw, d))
        meta[name] = {"src": "BASELINE.json configs", "seed": 0, "stream": stream, "n": n, "d": d,
                      "bias_scale": 0.5, "dtype": "bf16", "order": "q,k,v,bias from one rng stream, bf16_round each"}

    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(arrays)} arrays, {os.path.getsize(OUT)/1024:.0f} KiB")


if __name__ == "__main__":
    main()
