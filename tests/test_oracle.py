"""Pins the CPU oracle (oracle/binattn_oracle.c) before anything trusts it:

 (1) the known-answer vectors of the reference's own test-suite (file:line cited per test),
 (2) golden fixtures produced by the unmodified reference (tests/golden, oracle/gen_golden.py),
 (3) a live diff against the compiled reference (oracle/_ref) wherever it is present.
"""
import itertools

import numpy as np
import pytest

from oracle import cpu


def rel_l2(a, b):  # tests/oracles.hpp:95-103
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / den if den > 0 else np.linalg.norm(a - b)


# ---------------------------------------------------------------- bitops KATs (test_bitops.cpp)
def test_pack_signs_zero_maps_to_plus_one(port):  # test_bitops.cpp:10-17
    w = port.pack_signs(np.array([[1.5, -2.0, 0.0]]))
    assert w.shape == (1, 1) and int(w[0, 0]) == 0b101
    assert int(port.pack_signs(np.array([[-0.0]]))[0, 0]) == 1  # -0.0 >= 0.0 (bitops.cpp:45)


def test_all_negative_rows_pack_to_zero_words(port):  # test_bitops.cpp:19-23
    assert not port.pack_signs(-np.ones((4, 64))).any()


def test_self_and_complement_dot_d64(port):  # test_bitops.cpp:35-43
    a, b = port.pack_signs(np.ones((1, 64))), port.pack_signs(-np.ones((1, 64)))
    assert port.xnor_popcount_dot(a[0], a[0], 64) == 64
    assert port.xnor_popcount_dot(a[0], b[0], 64) == -64
    assert port.hamming_distance(a[0], a[0], 64) == 0


def test_four_bit_identity(port):  # test_bitops.cpp:45-53
    a = port.pack_signs(np.array([[1.0, -1, 1, 1]]))
    b = port.pack_signs(np.array([[1.0, 1, -1, 1]]))
    assert port.xnor_popcount_dot(a[0], b[0], 4) == 0
    assert port.hamming_distance(a[0], b[0], 4) == 2


def test_complement_pair_d100(port):  # test_bitops.cpp:55-61
    a, b = port.pack_signs(np.full((1, 100), 2.0)), port.pack_signs(np.full((1, 100), -2.0))
    assert port.hamming_distance(a[0], b[0], 100) == 100
    assert port.xnor_popcount_dot(a[0], b[0], 100) == -100
    assert a.shape == (1, 2) and int(a[0, 1]) == (1 << 36) - 1  # pad bits are zero (tensor.hpp:56)


def test_dot_hamming_identity_exhaustive(port):  # test_bitops.cpp:80-110
    for d in range(1, 6):
        for wa, wb in itertools.product(range(1 << d), repeat=2):
            a, b = np.array([wa], dtype=np.uint64), np.array([wb], dtype=np.uint64)
            dot, ham = port.xnor_popcount_dot(a, b, d), port.hamming_distance(a, b, d)
            assert dot == d - 2 * ham and -d <= dot <= d and dot % 2 == d % 2


def test_identity_random_widths(port):  # test_bitops.cpp:112-125 (seed 14)
    rng = port.make_rng(14)
    for _ in range(50):
        d = 1 + rng.u64() % 1024
        qa, qb = rng.random_dense(1, d), rng.random_dense(1, d)
        a, b = port.pack_signs(qa), port.pack_signs(qb)
        dot = port.xnor_popcount_dot(a[0], b[0], d)
        assert dot == d - 2 * port.hamming_distance(a[0], b[0], d)
        assert dot == int(np.sum(np.where(qa >= 0, 1, -1) * np.where(qb >= 0, 1, -1)))


@pytest.mark.parametrize("case", ["gemm_seed15", "gemm_seed17"])
def test_binary_gemm_golden(port, golden, case):  # test_bitops.cpp:136-145, 155-165
    c = golden.case(case)
    d = c["a"].shape[1]
    g = port.binary_gemm(port.pack_signs(c["a"]), port.pack_signs(c["b"]), d)
    assert np.array_equal(g, c["g"])
    pm1 = np.where(c["a"] >= 0, 1, -1) @ np.where(c["b"] >= 0, 1, -1).T  # oracles.hpp:27-38 pm1_gemm
    assert np.array_equal(g, pm1)


def test_pack_golden_and_rng_stream(port, golden):  # test_bitops.cpp:25-33 (seed 11)
    c = golden.case("pack_seed11")
    m = port.make_rng(11).random_dense(3, 130)
    assert np.array_equal(m, c["m"])  # the rng port reproduces rng.hpp bit for bit
    assert np.array_equal(port.pack_signs(m), c["words"])


# ---------------------------------------------------------------- quantize KATs (test_quantize.cpp)
def test_binary_quantize_kats(port, golden):
    w, mu = port.binary_quantize(np.array([[2.0, -2], [2, -2]]))  # test_quantize.cpp:9-14
    assert mu == 2.0
    w, mu = port.binary_quantize(np.array([[0.0]]))  # :16-20
    assert mu == 0.0 and int(w[0, 0]) == 1
    with pytest.raises(cpu.CpuError) as e:  # :22-24
        port.binary_quantize(np.zeros((0, 4)))
    assert e.value.kind == "ShapeError"
    c = golden.case("quant_seed21")  # :26-33
    w, mu = port.binary_quantize(c["m"])
    assert mu == float(c["mu"]) and np.array_equal(w, c["words"])
    assert abs(mu - np.abs(c["m"]).mean()) <= 1e-12


def test_quantize_values_kats(port):  # test_quantize.cpp:99-138
    v = np.array([[1.0, 0.0, -4.0], [-0.5, 0.0, 2.0]])
    data, scales = port.quantize_values(v)
    assert scales[1] == 1.0 and scales[0] == 1.0 / 127.0 and scales[2] == 4.0 / 127.0
    assert data.min() >= -127 and data[0, 0] == 127 and data[0, 2] == -127 and data[1, 0] == -64


# ---------------------------------------------------------------- bias (test_attention.cpp:11-57)
def test_bias_materialisation(port):
    n, c = 5, 3.25
    assert (port.bias_rel1d(np.full(2 * n - 1, c), n) == c).all()
    off = np.array([10.0, 20, 30, 40, 50])
    b = port.bias_rel1d(off, 3)
    for i in range(3):
        for j in range(3):
            assert b[i, j] == off[i - j + 2]
    ro, co = np.array([1.0, -2.0, 4.0]), np.array([8.0, 16.0, 32.0])
    b = port.bias_rel2d(ro, co, 4)
    for i in range(4):
        for j in range(4):
            assert b[i, j] == ro[i // 2 - j // 2 + 1] + co[i % 2 - j % 2 + 1]
    with pytest.raises(cpu.CpuError):
        port.bias_rel2d(np.array([1.0, 2, 3]), np.array([1.0, 2, 3]), 5)


# ---------------------------------------------------------------- attention KATs (test_attention.cpp)
def test_reference_attention_frozen_fixture(port):  # test_attention.cpp:92-109
    q = np.array([[1.0, 0], [0, 1], [1, 1]])
    k = np.array([[1.0, 1], [-1, 0], [0, 2]])
    v = np.array([[1.0, 2], [3, 4], [5, 6]])
    y, m, l, p = port.reference_attention(q, k, v, with_probs=True)
    want_p = [0.575975345215362, 0.14002924504337802, 0.28399540974126003, 0.28399540974126003,
              0.14002924504337802, 0.5759753452153619, 0.4717263166328708, 0.05654736673425857, 0.4717263166328708]
    want_y = [2.416040129051796, 3.416040129051796, 3.5839598709482035, 4.5839598709482035, 3.0000000000000004,
              4.000000000000001]
    np.testing.assert_allclose(p.ravel(), want_p, rtol=1e-14)
    np.testing.assert_allclose(y.ravel(), want_y, rtol=1e-14)


def test_binary_fixture_d1_n2(port):  # test_attention.cpp:163-174
    q, k, v = np.array([[2.0], [-1.0]]), np.array([[1.0], [-3.0]]), np.array([[4.0], [-2.0]])
    for fn in (port.binary_attention_unfused, port.binary_attention_fused):
        y, m, l = fn(q, k, v, tau=1.0)
        assert m[0] == pytest.approx(3.0)
        assert y[0, 0] == pytest.approx(3.985164261060192, rel=1e-14)
        assert y[1, 0] == pytest.approx(-1.9851642610601914, rel=1e-14)


def test_self_similarity_dominates_diagonal(port):  # test_attention.cpp:143-161 (seed 34)
    n, d = 4, 8
    rng = port.make_rng(34)
    q = np.array([2.0 if rng.u64() & 1 else -2.0 for _ in range(n * d)]).reshape(n, d)
    y, m, l, p = port.binary_attention_unfused(q, q, rng.random_dense(n, d), with_probs=True)
    np.testing.assert_allclose(m, 4.0 * d / np.sqrt(d), rtol=1e-12)
    assert (np.diag(p)[:, None] >= p).all()


def test_shape_and_validation_errors(port):  # test_attention.cpp:126-141
    rng = port.make_rng(33)
    q, bad, v = rng.random_dense(4, 3), rng.random_dense(4, 2), rng.random_dense(4, 3)
    with pytest.raises(cpu.CpuError) as e:
        port.binary_attention_fused(q, v, bad)
    assert e.value.kind == "ShapeError"
    with pytest.raises(cpu.CpuError) as e:
        port.binary_attention_fused(q, q, v, block_rows=9)
    assert e.value.kind == "ValidationError"
    with pytest.raises(cpu.CpuError) as e:
        port.binary_attention_fused(q, q, v, tau=0.0)
    assert e.value.kind == "ValidationError"


@pytest.mark.parametrize("case", ["attn_seed35", "attn_seed38", "attn_seed40", "attn_seed43", "attn_seed37_0",
                                  "attn_seed37_1", "attn_seed37_2"])
def test_attention_golden(port, golden, case):
    c, meta = golden.case(case), golden.meta[case]
    bias = c.get("bias")
    yu, mu_, lu = port.binary_attention_unfused(c["q"], c["k"], c["v"], bias=bias)
    yf, mf, lf = port.binary_attention_fused(c["q"], c["k"], c["v"], bias=bias, block_rows=meta["block_rows"],
                                             block_cols=meta["block_cols"])
    for got, want in [(yu, "y_unfused"), (mu_, "m_unfused"), (lu, "l_unfused"), (yf, "y_fused"), (mf, "m_fused"),
                      (lf, "l_fused")]:
        assert np.array_equal(got, c[want]), want  # bit-identical to the reference's fp64 output
    if "y_fused_int8" in c:
        yq = port.binary_attention_fused(c["q"], c["k"], c["v"], bias=bias, quantize_pv=True,
                                         block_rows=meta["block_rows"], block_cols=meta["block_cols"])[0]
        assert np.array_equal(yq, c["y_fused_int8"])
        qw, muq = port.binary_quantize(c["q"])
        kw, muk = port.binary_quantize(c["k"])
        assert np.array_equal(qw, c["q_words"]) and np.array_equal(kw, c["k_words"])
        assert np.array_equal(np.array([muq, muk]), c["mu"])
        assert np.array_equal(port.binary_gemm(qw, kw, c["q"].shape[1]), c["logits"])


def test_single_block_fused_equals_unfused_bitwise(port, golden):  # test_attention.cpp:234-252
    for idx in range(3):
        c = golden.case(f"attn_seed37_{idx}")
        n = c["q"].shape[0]
        a = port.binary_attention_unfused(c["q"], c["k"], c["v"])
        b = port.binary_attention_fused(c["q"], c["k"], c["v"], block_rows=n, block_cols=n)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_online_softmax_exact_across_blocks(port, golden):  # test_attention.cpp:254-272
    c = golden.case("attn_seed38")
    n = 48
    for br in (1, 3, 16, n):
        for bc in (1, 5, 16, n):
            yf = port.binary_attention_fused(c["q"], c["k"], c["v"], bias=c["bias"], block_rows=br, block_cols=bc)[0]
            assert rel_l2(yf, c["y_unfused"]) <= 1e-12


def test_fused_int8_vs_unfused_fp(port, golden):  # test_attention.cpp:300-314
    c = golden.case("attn_seed40")
    assert rel_l2(c["y_fused_int8"], c["y_unfused"]) <= 1e-2


def test_shift_and_scale_invariance(port):  # test_attention.cpp:316-347
    rng = port.make_rng(41)
    n, d = 12, 8
    q, k, v = rng.random_dense(n, d), rng.random_dense(n, d), rng.random_dense(n, d)
    y0 = port.binary_attention_unfused(q, k, v)[0]
    y1 = port.binary_attention_unfused(q, k, v, bias=port.bias_rel1d(np.full(2 * n - 1, -1.75), n))[0]
    assert rel_l2(y1, y0) <= 1e-12
    rng = port.make_rng(42)
    q, k = rng.random_dense(10, 32), rng.random_dense(10, 32)
    b0, s0 = port.binary_quantize(q)
    b1, s1 = port.binary_quantize(7.0 * q)
    assert np.array_equal(b0, b1) and s1 == pytest.approx(7.0 * s0, rel=1e-12)


@pytest.mark.parametrize("case", ["c1_head0", "c1_head5", "c3_head0", "mix_n300_d72", "mix_n130_d128"])
def test_baseline_shape_golden(port, golden, case):
    """One head at the BASELINE.json shapes, bf16-rounded inputs regenerated from the seed recipe."""
    c, meta = golden.case(case), golden.meta[case]
    n, d = meta["n"], meta["d"]
    rng = port.make_rng(meta["seed"], meta["stream"])
    q, k, v = (cpu.bf16_round(rng.random_dense(n, d)) for _ in range(3))
    bias = cpu.bf16_round(rng.random_dense(n, n, meta["bias_scale"]))
    qw, muq = port.binary_quantize(q)
    kw, muk = port.binary_quantize(k)
    assert np.array_equal(qw, c["q_words"]) and np.array_equal(kw, c["k_words"])
    assert np.array_equal(np.array([muq, muk]), c["mu"])
    assert np.array_equal(port.binary_gemm(qw[:4], kw, d), c["logits_rows"])
    y, m, l = port.binary_attention_fused(q, k, v, bias=bias)
    assert np.array_equal(y, c["y"]) and np.array_equal(m, c["m"]) and np.array_equal(l, c["l"])
    assert np.array_equal(port.binary_attention_fused(q, k, v)[0], c["y_nobias"])
    yq = port.binary_attention_fused(q, k, v, bias=bias, quantize_pv=True)[0]
    assert np.abs(yq - c["y_int8"]).max() <= 1e-6  # stored as float32


# ---------------------------------------------------------------- live diff against oracle/_ref
def test_port_matches_compiled_reference(port, ref):
    for seed, (n, d), bscale in [(101, (33, 5), None), (102, (70, 72), 0.5), (103, (129, 64), 0.5), (104, (64, 130), None)]:
        pr, rr = port.make_rng(seed), ref.make_rng(seed)
        q, k, v = pr.random_dense(n, d), pr.random_dense(n, d), pr.random_dense(n, d)
        assert np.array_equal(q, rr.random_dense(n, d)) and np.array_equal(k, rr.random_dense(n, d))
        assert np.array_equal(v, rr.random_dense(n, d))
        bias = pr.random_dense(n, n, bscale) if bscale else None
        assert np.array_equal(port.pack_signs(q), ref.pack_signs(q))
        assert port.binary_quantize(k)[1] == ref.binary_quantize(k)[1]
        qw, kw = port.pack_signs(q), port.pack_signs(k)
        assert np.array_equal(port.binary_gemm(qw, kw, d), ref.binary_gemm(qw, kw, d))
        for qpv in (False, True):
            a = port.binary_attention_fused(q, k, v, bias=bias, quantize_pv=qpv, block_rows=min(n, 17), block_cols=min(n, 29))
            b = ref.binary_attention_fused(q, k, v, bias=bias, quantize_pv=qpv, block_rows=min(n, 17), block_cols=min(n, 29))
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
            a = port.binary_attention_unfused(q, k, v, bias=bias, quantize_pv=qpv)
            b = ref.binary_attention_unfused(q, k, v, bias=bias, quantize_pv=qpv)
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
        a, b = port.reference_attention(q, k, v, bias=bias), ref.reference_attention(q, k, v, bias=bias)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_heads_driver_matches_single_calls(port):
    rng = port.make_rng(7)
    q, k, v = (rng.random_dense(3 * 20, 8).reshape(3, 20, 8) for _ in range(3))
    bias = rng.random_dense(2 * 20, 20, 0.5).reshape(2, 20, 20)
    y = port.binary_attention_fused_heads(q, k, v, bias=bias, nthreads=2)
    for h in range(3):
        assert np.array_equal(y[h], port.binary_attention_fused(q[h], k[h], v[h], bias=bias[h % 2])[0])


# ---------------------------------------------------------------- attention-map fidelity KATs (test_fidelity.cpp)
def _row_stochastic(rng, n, cols):
    p = rng.random((n, cols))
    return p / p.sum(axis=1, keepdims=True)


def _brute_precision(a, b, k):  # test_fidelity.cpp:28-57 (selection with lower-index tie-breaks)
    n, cols = a.shape
    keff = min(k, cols)

    def topk(row):
        used, picked = set(), []
        for _ in range(keff):
            best = None
            for j in range(cols):
                if j in used:
                    continue
                if best is None or row[j] > row[best]:
                    best = j
            used.add(best)
            picked.append(best)
        return picked
    return sum(len(set(topk(a[i])) & set(topk(b[i]))) / keff for i in range(n)) / n


def test_fidelity_self_comparison(port):  # test_fidelity.cpp:70-78
    p = _row_stochastic(np.random.default_rng(61), 6, 6)
    cos, rl1, rmse, prec = port.attention_fidelity(p, p, 3)
    assert abs(cos - 1.0) <= 4e-16 and (rl1, rmse, prec) == (0.0, 0.0, 1.0)  # (sqrt(x)*sqrt(x) may round off x by an ulp)


def test_fidelity_tie_break_toward_lower_index(port):  # test_fidelity.cpp:80-87
    n = 4
    uni = np.full((n, n), 1.0 / n)
    hot0, hot2 = np.zeros((n, n)), np.zeros((n, n))
    hot0[:, 0] = 1.0
    hot2[:, 2] = 1.0
    assert port.attention_fidelity(hot0, uni, 1)[3] == 1.0
    assert port.attention_fidelity(hot2, uni, 1)[3] == 0.0


def test_fidelity_matches_brute_force(port):  # test_fidelity.cpp:89-109
    rng = np.random.default_rng(62)
    a, b = _row_stochastic(rng, 8, 8), _row_stochastic(rng, 8, 8)
    cos, rl1, rmse, prec = port.attention_fidelity(a, b, 3)
    assert prec == _brute_precision(a, b, 3)
    assert cos == pytest.approx((a * b).sum() / np.sqrt((a * a).sum() * (b * b).sum()), rel=1e-12)
    assert rl1 == pytest.approx(np.abs(a - b).sum() / np.abs(a).sum(), rel=1e-12)
    assert rmse == pytest.approx(np.sqrt(((a - b) ** 2).mean()), rel=1e-12)


def test_fidelity_k_clamps_and_asymmetry(port):  # test_fidelity.cpp:111-135
    rng = np.random.default_rng(63)
    a, b = _row_stochastic(rng, 4, 4), _row_stochastic(rng, 4, 4)
    assert port.attention_fidelity(a, b, 100)[3] == 1.0
    a, b = _row_stochastic(rng, 5, 7), _row_stochastic(rng, 5, 7)
    ab, ba_ = port.attention_fidelity(a, b, 2), port.attention_fidelity(b, a, 2)
    assert ab[2] == ba_[2]
    assert ab[1] == pytest.approx(np.abs(a - b).sum() / np.abs(a).sum(), rel=1e-12)
    assert ba_[1] == pytest.approx(np.abs(a - b).sum() / np.abs(b).sum(), rel=1e-12)


def test_fidelity_validation(port):  # test_fidelity.cpp:163-170
    a = _row_stochastic(np.random.default_rng(66), 4, 4)
    with pytest.raises(cpu.CpuError):
        port.attention_fidelity(a, _row_stochastic(np.random.default_rng(1), 5, 5), 2)  # ShapeError
    with pytest.raises(cpu.CpuError):
        port.attention_fidelity(a, np.full((4, 4), 0.5), 2)  # rows sum to 2: ValidationError
    with pytest.raises(cpu.CpuError):
        port.attention_fidelity(a, a, 0)  # k = 0


def test_fidelity_port_equals_reference(port, ref):
    """Live diff against the compiled reference, on the attention maps the metric is meant for: the full-precision map
    against the binary one (fidelity.cpp:40-85 over attention.cpp:99-147 / 149-248 with_probs)."""
    rng = np.random.default_rng(5)
    for n, d, k in [(33, 16, 5), (64, 32, 8), (12, 8, 20)]:
        q, kk, v = (cpu.bf16_round(rng.standard_normal((n, d))) for _ in range(3))
        bias = cpu.bf16_round(0.5 * rng.standard_normal((n, n)))
        p_ref = ref.reference_attention(q, kk, v, bias=bias, with_probs=True)[3]
        p_bin = ref.binary_attention_unfused(q, kk, v, bias=bias, with_probs=True)[3]
        assert np.array_equal(p_bin, port.binary_attention_unfused(q, kk, v, bias=bias, with_probs=True)[3])
        r_ref, r_port = ref.attention_fidelity(p_ref, p_bin, k), port.attention_fidelity(p_ref, p_bin, k)
        assert r_ref[3] == r_port[3]
        assert np.allclose(r_ref[:3], r_port[:3], rtol=1e-13, atol=0)
