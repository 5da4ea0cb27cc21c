"""Parity tests proper: the CUDA path (through the C ABI) against the CPU oracle on identical inputs.

Bars (BASELINE.json north star): packed sign bits and integer logits BIT-EXACT; O within max-abs 2e-3 of the
reference's fp64 path (quantize_pv=false); mu within 2e-6 relative.
Every test runs for each kernel variant the build offers ("simt" always; "tcgen05" when it takes the shape).
"""
import numpy as np
import pytest

from oracle import cpu
from tests.helpers import make_head_inputs, to_torch, words_to_numpy

pytestmark = pytest.mark.gpu

TOL_O = 2e-3      # max-abs on O vs the fp64 oracle (north star)
TOL_MU = 2e-6     # relative, fp32 tree sum vs sequential fp64 sum


@pytest.fixture(scope="module")
def ba():
    import torch
    import paper_2603_09582_b200 as pkg
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    return pkg.BinaryAttention(torch.device("cuda:0"))


def kernels_for(ba, B, H, N, d, dtype, bias=None):
    import torch
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16}[dtype]
    ks = ["simt"]
    if ba.select_kernel(B, H, N, d, tdt, bias) == "tcgen05":
        ks.append("tcgen05")
    return ks


# ------------------------------------------------------------------------------------------ K1 pack + mu
@pytest.mark.parametrize("dtype", ["bf16", "f32", "f16"])
@pytest.mark.parametrize("n,d", [(197, 64), (256, 72), (130, 128), (33, 5), (3, 130), (50, 12), (1, 1), (700, 200),
                                 (513, 96)])
def test_pack_signs_bit_exact(ba, port, n, d, dtype):
    heads = [make_head_inputs(port, 5, s, n, d, dtype=dtype) for s in range(3)]
    X = to_torch(np.stack([h[0] for h in heads])[None], dtype)
    words, mu = ba.pack_signs(X)
    assert words.shape == (1, 3, n, (d + 63) // 64)
    for h in range(3):
        ow, omu = port.binary_quantize(heads[h][0])
        assert np.array_equal(words_to_numpy(words[0, h]), ow)  # byte-identical to BitMatrix::words()
        assert abs(float(mu[0, h]) - omu) <= TOL_MU * omu


def test_pack_signs_kats(ba, port):
    import torch
    # test_bitops.cpp:10-17 (zero -> +1), :19-23 (all negative -> zero words); -0.0 >= 0 (bitops.cpp:45)
    x = torch.tensor([[[[1.5, -2.0, 0.0]]]], device="cuda", dtype=torch.float32)
    w, mu = ba.pack_signs(x)
    assert int(w[0, 0, 0, 0]) == 0b101 and float(mu[0, 0]) == pytest.approx(3.5 / 3)
    w, _ = ba.pack_signs(-torch.ones(1, 1, 4, 64, device="cuda", dtype=torch.bfloat16))
    assert not w.any()
    w, mu = ba.pack_signs(torch.tensor([[[[-0.0, 0.0]]]], device="cuda", dtype=torch.bfloat16))
    assert int(w[0, 0, 0, 0]) == 0b11 and float(mu[0, 0]) == 0.0  # test_quantize.cpp:16-20
    up = torch.full((1, 1, 1, 100), 2.0, device="cuda", dtype=torch.bfloat16)  # test_bitops.cpp:55-61
    wu, _ = ba.pack_signs(up)
    wd, _ = ba.pack_signs(-up)
    assert int(wu[0, 0, 0, 0]) == -1 and int(wu[0, 0, 0, 1]) == (1 << 36) - 1 and not wd.any()
    S = ba.binary_logits(wu, wd, 100)
    assert int(S[0, 0]) == -100
    x = torch.tensor([[[[2.0, -2.0], [2.0, -2.0]]]], device="cuda", dtype=torch.float32)  # test_quantize.cpp:9-14
    assert float(ba.pack_signs(x)[1][0, 0]) == 2.0


def test_scale_invariance_of_bits(ba, port):  # test_attention.cpp:330-347
    q = make_head_inputs(port, 42, 0, 10, 32, dtype="f32")[0]
    w0, m0 = ba.pack_signs(to_torch(q[None, None], "f32"))
    w1, m1 = ba.pack_signs(to_torch(7.0 * q[None, None], "f32"))
    assert (w0 == w1).all() and float(m1) == pytest.approx(7.0 * float(m0), rel=1e-6)


def test_pack_signs_nan_maps_to_zero_bit(ba):
    """bit = 1 iff x >= 0.0 (bitops.cpp:45): NaN of either sign packs as 0 in every kernel variant (the reference itself
    rejects non-finite inputs, tensor.cpp:15; the ABI has no such check, so the rule must not depend on dtype or d)."""
    import torch
    for d in (64, 72, 200):
        x = torch.randn(1, 2, 70, d, device="cuda")
        x[0, 0, 3, 5] = float("nan")
        x[0, 1, 69, d - 1] = -float("nan")
        x[0, 1, 0, 0] = float("inf")
        for dt in (torch.bfloat16, torch.float32, torch.float16):
            xd = x.to(dt)
            words, _ = ba.pack_signs(xd)
            w = words_to_numpy(words).reshape(2, 70, -1)
            want = (xd.float() >= 0).cpu().numpy()
            got = np.zeros_like(want)
            for c in range(d):
                got[0, :, :, c] = ((w[:, :, c // 64] >> np.uint64(c % 64)) & np.uint64(1)).astype(bool)
            assert np.array_equal(got, want), (d, dt)


def test_masked_first_keys_do_not_poison_the_row(ba, port):
    """Mask-style bias (-inf on the leading keys of some rows): every kernel gives the finite reference answer (the CUDA-core
    kernel's per-key running max used to evaluate exp2(-inf - -inf) there)."""
    import torch
    n, d = 96, 32
    q, k, v, _ = make_head_inputs(port, 45, 0, n, d)
    b = np.zeros((n, n))
    b[5, :40] = -np.inf
    b[77, :60] = -np.inf   # (under one 64-key block: a fully masked first block is NaN in the reference itself, attention.cpp:308-312)
    y = port.binary_attention_fused(q, k, v, bias=b)[0]
    assert np.isfinite(y).all()
    for dt in ("bf16", "f32"):
        Q, K, V = (to_torch(x[None, None], dt) for x in (q, k, v))
        bt = torch.from_numpy(b).to("cuda", torch.float32)[None]
        for kern in kernels_for(ba, 1, 1, n, d, dt, bt):
            O = ba.forward(Q, K, V, bt, kernel=kern)
            assert torch.isfinite(O).all(), kern
            assert np.abs(O[0, 0].cpu().numpy() - y).max() <= TOL_O, kern


def test_pack_is_bit_reproducible(ba, port):
    X = to_torch(make_head_inputs(port, 9, 0, 2000, 128)[0][None, None], "bf16")
    w0, m0 = ba.pack_signs(X)
    for _ in range(3):
        w1, m1 = ba.pack_signs(X)
        assert (w0 == w1).all() and (m0 == m1).all()


# ------------------------------------------------------------------------------------------ K3 integer logits
@pytest.mark.parametrize("n,d", [(197, 64), (256, 72), (97, 129), (130, 128), (40, 200)])
def test_binary_logits_bit_exact(ba, port, n, d):
    q, k, _, _ = make_head_inputs(port, 17, 1, n, d)
    qw, _ = ba.pack_signs(to_torch(q[None, None], "bf16"))
    kw, _ = ba.pack_signs(to_torch(k[None, None], "bf16"))
    S = ba.binary_logits(qw, kw, d).cpu().numpy()
    want = port.binary_gemm(port.pack_signs(q), port.pack_signs(k), d)
    assert np.array_equal(S, want)
    assert ((S % 2) == d % 2).all() and np.abs(S).max() <= d  # test_bitops.cpp:80-110


# ------------------------------------------------------------------------------------------ K2 fused attention
def run_and_compare(ba, port, heads, n, d, dtype, bias_mode, scale=None, tol=None):
    """heads: list of (q,k,v,bias) float64; bias_mode in {None,'per_head','shared'}."""
    import torch
    H = len(heads)
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], dtype) for i in range(3))
    bias_t = None
    bdt = "bf16" if dtype == "bf16" else "f32"  # bias values were rounded to `dtype`; f16 values are exact in f32
    if bias_mode == "per_head":
        bias_t = to_torch(np.stack([h[3] for h in heads]), bdt)
    elif bias_mode == "shared":
        bias_t = to_torch(heads[0][3][None], bdt)
    results = {}
    for kern in kernels_for(ba, 1, H, n, d, dtype, bias_t):
        O, m, l = ba.forward(Q, K, V, bias_t, scale, kernel=kern, return_stats=True)
        torch.cuda.synchronize()
        O, m, l = O.cpu().numpy().astype(np.float64), m.cpu().numpy().astype(np.float64), l.cpu().numpy().astype(np.float64)
        assert np.isfinite(O).all()
        for h in range(H):
            q, k, v, b = heads[h]
            b = None if bias_mode is None else (heads[0][3] if bias_mode == "shared" else b)
            tau = None if scale is None else 1.0 / scale
            y, om, ol = port.binary_attention_fused(q, k, v, tau=tau, bias=b)
            err = np.abs(O[0, h] - y).max()
            assert err <= (tol or {}).get(kern, TOL_O), f"{kern}: head {h} max-abs {err:.3e}"
            # log-sum-exp is tile-invariant: m + ln(l)  (AttentionOutput::row_max/row_sum, attention.hpp:45-46)
            # (the tcgen05 kernel's row_sum is the sum of the bf16-rounded weights it actually multiplied with V,
            #  accumulated by the tensor core: each weight is within 2^-9 relative of exp(S-m), so ln(l) is within
            #  2e-3 of the fp64 value; a diagnostic, not part of O)
            np.testing.assert_allclose(m[0, h] + np.log(l[0, h]), om + np.log(ol), rtol=0, atol=2.5e-3)
        results[kern] = O
    return results


@pytest.mark.parametrize("bias_mode", [None, "per_head", "shared"])
@pytest.mark.parametrize("n,d", [(197, 64), (256, 72), (130, 128), (64, 64), (129, 64), (300, 72), (48, 16), (33, 8)])
def test_attention_matches_oracle_bf16(ba, port, n, d, bias_mode):
    heads = [make_head_inputs(port, 3, s, n, d, bias_scale=0.5) for s in range(3)]
    run_and_compare(ba, port, heads, n, d, "bf16", bias_mode)


@pytest.mark.parametrize("dtype", ["f32", "f16"])
@pytest.mark.parametrize("n,d", [(50, 12), (33, 5), (7, 16), (100, 100), (64, 129)])
def test_attention_matches_oracle_other_dtypes(ba, port, n, d, dtype):
    heads = [make_head_inputs(port, 4, s, n, d, bias_scale=0.4, dtype=dtype) for s in range(2)]
    run_and_compare(ba, port, heads, n, d, dtype, "per_head")


def test_attention_custom_scale_and_d1_fixture(ba, port):
    import torch
    # test_attention.cpp:163-174: d=1, N=2, tau=1 -> Y = [3.985164261060192, -1.9851642610601914]
    q = torch.tensor([[[[2.0], [-1.0]]]], device="cuda")
    k = torch.tensor([[[[1.0], [-3.0]]]], device="cuda")
    v = torch.tensor([[[[4.0], [-2.0]]]], device="cuda")
    O, m, l = ba.forward(q, k, v, None, 1.0, return_stats=True)
    assert O.flatten().tolist() == pytest.approx([3.985164261060192, -1.9851642610601914], abs=1e-5)
    assert float(m[0, 0, 0]) == pytest.approx(3.0, abs=1e-5)
    heads = [make_head_inputs(port, 6, 0, 90, 64, bias_scale=0.5)]
    run_and_compare(ba, port, heads, 90, 64, "bf16", "per_head", scale=0.05)


@pytest.mark.parametrize("case", ["c1_head0", "c1_head5", "c3_head0", "mix_n300_d72", "mix_n130_d128"])
def test_attention_matches_reference_golden(ba, port, golden, case):
    """Against outputs of the UNMODIFIED reference (tests/golden, oracle/gen_golden.py)."""
    import torch
    c, meta = golden.case(case), golden.meta[case]
    n, d = meta["n"], meta["d"]
    q, k, v, bias = make_head_inputs(port, meta["seed"], meta["stream"], n, d, bias_scale=meta["bias_scale"])
    Q, K, V = (to_torch(x[None, None], "bf16") for x in (q, k, v))
    B = to_torch(bias[None], "bf16")
    qw, muq = ba.pack_signs(Q)
    kw, muk = ba.pack_signs(K)
    assert np.array_equal(words_to_numpy(qw[0, 0]), c["q_words"]) and np.array_equal(words_to_numpy(kw[0, 0]), c["k_words"])
    assert abs(float(muq) - c["mu"][0]) <= TOL_MU * c["mu"][0] and abs(float(muk) - c["mu"][1]) <= TOL_MU * c["mu"][1]
    assert np.array_equal(ba.binary_logits(qw, kw, d).cpu().numpy()[:4], c["logits_rows"])
    for kern in kernels_for(ba, 1, 1, n, d, "bf16", B):
        O = ba.forward(Q, K, V, B, kernel=kern)[0, 0].cpu().numpy().astype(np.float64)
        O_nb = ba.forward(Q, K, V, None, kernel=kern)[0, 0].cpu().numpy().astype(np.float64)
        assert np.abs(O - c["y"]).max() <= TOL_O and np.abs(O_nb - c["y_nobias"]).max() <= TOL_O
        # secondary, not gated at 2e-3: distance to the reference's default int8 P.V mode (SURVEY.md finding 2)
        assert np.abs(O - c["y_int8"]).max() <= 2e-2


def test_constant_bias_shift_invariance(ba, port):  # test_attention.cpp:316-328
    import torch
    n, d = 120, 64
    q, k, v, _ = make_head_inputs(port, 41, 0, n, d)
    Q, K, V = (to_torch(x[None, None], "bf16") for x in (q, k, v))
    shift = torch.full((1, n, n), -1.75, device="cuda", dtype=torch.float32)
    for kern in kernels_for(ba, 1, 1, n, d, "bf16"):
        y0 = ba.forward(Q, K, V, None, kernel=kern)
        y1 = ba.forward(Q, K, V, shift, kernel=kern)
        assert (y0 - y1).abs().max().item() <= 1e-5


def test_bias_row_stride(ba, port):
    """bias_ld > N (padded rows) gives the same result as the dense N x N table."""
    import torch
    n, d = 197, 64
    q, k, v, bias = make_head_inputs(port, 8, 0, n, d, bias_scale=0.5)
    Q, K, V = (to_torch(x[None, None], "bf16") for x in (q, k, v))
    dense = to_torch(bias[None], "bf16")
    padded = torch.zeros(1, n, 200, device="cuda", dtype=torch.bfloat16)
    padded[:, :, :n] = dense
    for kern in kernels_for(ba, 1, 1, n, d, "bf16", dense):
        y0 = ba.forward(Q, K, V, dense, kernel=kern)
        y1 = ba.forward(Q, K, V, padded[:, :, :n], kernel=kern)
        assert torch.equal(y0, y1)


def test_run_to_run_and_shard_identity(ba, port):
    """Determinism + SURVEY.md 8e: running a sub-range of heads gives byte-identical rows to the full run."""
    import torch
    from paper_2603_09582_b200 import shard_range
    B, H, n, d = 2, 4, 197, 64
    heads = [make_head_inputs(port, 12, s, n, d, bias_scale=0.5) for s in range(B * H)]
    Q, K, V = (to_torch(np.stack([h[i] for h in heads]).reshape(B, H, n, d), "bf16") for i in range(3))
    for kern in kernels_for(ba, B, H, n, d, "bf16"):
        full = ba.forward(Q, K, V, None, kernel=kern)
        assert torch.equal(full, ba.forward(Q, K, V, None, kernel=kern))
        for world in (2, 3):
            parts = []
            for rank in range(world):
                b, e = shard_range(B * H, world, rank)
                sl = lambda t: t.reshape(1, B * H, n, d)[:, b:e].contiguous()
                parts.append(ba.forward(sl(Q), sl(K), sl(V), None, kernel=kern))
            assert torch.equal(torch.cat(parts, dim=1).reshape(B, H, n, d), full)


def test_host_buffer_entry_point(ba, port):
    import torch
    n, d = 197, 64
    heads = [make_head_inputs(port, 13, s, n, d, bias_scale=0.5) for s in range(4)]
    Qh, Kh, Vh = (to_torch(np.stack([h[i] for h in heads])[None], "bf16", "cpu").pin_memory() for i in range(3))
    bh = to_torch(np.stack([h[3] for h in heads]), "bf16", "cpu").pin_memory()
    out = ba.forward_host(Qh, Kh, Vh, bh)
    dev = ba.forward(Qh.cuda(), Kh.cuda(), Vh.cuda(), bh.cuda())
    assert torch.equal(out, dev.cpu())


def test_host_buffer_pipeline_chunks(ba):
    """The host entry point cuts the head grid into chunks that flow through copy-in / compute / copy-out streams.
    360 heads of 25 KB make three chunks whose boundaries (166, 332) are not multiples of H, so the per-head bias
    lookup of a ranged call (head0 offset) is exercised too; results must equal the one-shot device call bit for bit."""
    import torch
    B, H, n, d = 30, 12, 197, 64
    g = torch.Generator().manual_seed(3)
    Qh, Kh, Vh = (torch.randn(B, H, n, d, generator=g).to(torch.bfloat16).pin_memory() for _ in range(3))
    bh = (0.5 * torch.randn(H, n, n, generator=g)).to(torch.bfloat16).pin_memory()
    for bias in (bh, None):
        out = ba.forward_host(Qh, Kh, Vh, bias)
        dev = ba.forward(Qh.cuda(), Kh.cuda(), Vh.cuda(), None if bias is None else bias.cuda())
        assert torch.equal(out, dev.cpu())


@pytest.mark.parametrize("n,d,with_bias", [(1500, 64, True), (2048, 128, False), (1111, 72, True)])
def test_long_sequence_rows_match_oracle(ba, port, n, d, with_bias):
    """BASELINE.json configs[3]/[4] regime (many key tiles per unit, the rolling S refill and the lazy rescale at
    work): two heads against the oracle, every row."""
    heads = [make_head_inputs(port, 21, s, n, d, bias_scale=0.5 if with_bias else None) for s in range(2)]
    run_and_compare(ba, port, heads, n, d, "bf16", "per_head" if with_bias else None)


@pytest.mark.parametrize("n,d", [(65, 64), (72, 64), (73, 64), (200, 64), (201, 64), (133, 128), (136, 72)])
@pytest.mark.parametrize("bias_kind", [None, "bf16", "f32"])
def test_tail_folding_edges(ba, port, n, d, bias_kind):
    """1..8 keys past the last full 64-key tile are folded into that tile (CUDA-core logits + a fifth P.V k-step);
    9 or more get a tile of their own.  Both sides of the switch, the shortest folded sequence (65), both bias
    paths (bf16 table staged by TMA / fp32 table read directly), d = 128 (register denominators) and d = 72."""
    import torch
    heads = [make_head_inputs(port, 23, s, n, d, bias_scale=0.5 if bias_kind else None) for s in range(2)]
    if bias_kind != "f32":
        run_and_compare(ba, port, heads, n, d, "bf16", "per_head" if bias_kind else None)
        return
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    bias = to_torch(np.stack([h[3] for h in heads]), "f32")  # bf16-representable values in an fp32 table
    O = ba.forward(Q, K, V, bias, kernel="tcgen05").cpu().numpy().astype(np.float64)
    for h in range(2):
        q, k, v, b = heads[h]
        assert np.abs(O[0, h] - port.binary_attention_fused(q, k, v, bias=b)[0]).max() <= TOL_O


@pytest.mark.parametrize("n,d", [(197, 64), (256, 72), (130, 128), (64, 64), (300, 72), (1000, 64), (40, 200)])
@pytest.mark.parametrize("per_head", [False, True])
def test_relative_1d_bias_generated_in_kernel(ba, port, n, d, per_head):
    """Relative1dBias (attention.hpp:18-21): the kernels build b_ij = offsets[i-j+N-1] from the 2N-1 offsets; the oracle
    gets the dense table the reference's materialize_bias makes of the same offsets (attention.cpp:65-76).  Also equal,
    bit for bit, to our own dense-bias path fed that table (same kernel arithmetic, different bias source)."""
    import torch
    import paper_2603_09582_b200 as pkg
    H = 2
    heads = [make_head_inputs(port, 31, s, n, d) for s in range(H)]
    rng = np.random.default_rng(7)
    offs = cpu.bf16_round(0.5 * rng.standard_normal((H if per_head else 1, 2 * n - 1)))
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    for odt in ("f32", "bf16"):
        rel = pkg.Relative1dBias(to_torch(offs, odt))
        tables = np.stack([port.bias_rel1d(offs[h if per_head else 0], n) for h in range(H)])
        for kern in kernels_for(ba, 1, H, n, d, "bf16"):
            O = ba.forward(Q, K, V, rel, kernel=kern)
            for h in range(H):
                q, k, v, _ = heads[h]
                y = port.binary_attention_fused(q, k, v, bias=tables[h])[0]
                assert np.abs(O[0, h].cpu().numpy().astype(np.float64) - y).max() <= TOL_O, (kern, odt, h)
            if kern == "tcgen05":
                dense = ba.forward(Q, K, V, to_torch(tables, "f32"), kernel=kern)
                assert torch.equal(O, dense)
    with pytest.raises(pkg.ShapeError):  # attention.cpp:66-67
        ba.forward(Q, K, V, pkg.Relative1dBias(torch.zeros(2 * n, device="cuda")))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("n,d", [(197, 64), (256, 72), (64, 32), (50, 12), (130, 128)])
def test_quantize_values_bit_exact(ba, port, n, d, dtype):
    """K1v vs quantize_values (quantize.cpp:57-74): s8 levels identical, fp64 scales identical; never -128, a zero column
    gets scale 1 (test_quantize.cpp:99-138)."""
    import torch
    heads = [make_head_inputs(port, 44, s, n, d, dtype=dtype)[2] for s in range(2)]
    heads[1] = heads[1].copy()
    heads[1][:, 3] = 0.0  # all-zero column
    vq, sc = ba.quantize_values(to_torch(np.stack(heads)[None], dtype))
    for h in range(2):
        oq, os_ = port.quantize_values(heads[h])
        assert np.array_equal(vq[0, h].cpu().numpy(), oq)
        assert np.array_equal(sc[0, h].cpu().numpy(), os_)
    assert int(vq.min()) >= -127 and float(sc[0, 1, 3]) == 1.0


@pytest.mark.parametrize("bias_mode", [None, "per_head"])
@pytest.mark.parametrize("n,d,bc", [(197, 64, None), (256, 72, None), (64, 32, 16), (130, 128, 64), (48, 16, 5), (300, 72, 33)])
def test_int8_pv_mode_matches_reference_default(ba, port, n, d, bc, bias_mode):
    """quantize_pv = true, the reference's DEFAULT mode (attention.hpp:35, attention.cpp:332-343, 361-363): same key-block
    size on both sides.  fp32 exp against fp64 exp can flip round(255 P^) at a .5 boundary (one level = 1/255 of a weight),
    hence a tolerance; the reference's own bound for this mode against its fp64 path is rel-L2 1e-2
    (test_attention.cpp:300-314), which must hold here too."""
    heads = [make_head_inputs(port, 45, s, n, d, bias_scale=0.5 if bias_mode else None) for s in range(2)]
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    bias_t = to_torch(np.stack([h[3] for h in heads]), "bf16") if bias_mode else None
    O, m, l = ba.forward(Q, K, V, bias_t, quantize_pv=True, block_cols=bc, return_stats=True)
    O = O.cpu().numpy().astype(np.float64)
    for h in range(2):
        q, k, v, b = heads[h]
        y8, om, ol = port.binary_attention_fused(q, k, v, bias=b, quantize_pv=True, block_cols=bc)
        assert np.abs(O[0, h] - y8).max() <= 1e-3, np.abs(O[0, h] - y8).max()
        np.testing.assert_allclose(m[0, h].cpu().numpy(), om, rtol=0, atol=1e-4)
        np.testing.assert_allclose(l[0, h].cpu().numpy(), ol, rtol=2e-5)
        y64 = port.binary_attention_fused(q, k, v, bias=b)[0]
        assert np.linalg.norm(O[0, h] - y64) / np.linalg.norm(y64) <= 1e-2


def test_int8_pv_mode_errors(ba):
    import torch
    import paper_2603_09582_b200 as pkg
    q = torch.zeros(1, 1, 100, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(pkg.ValidationError):  # attention.cpp:26-28
        ba.forward(q, q, q, quantize_pv=True, block_cols=101)
    with pytest.raises(pkg.UnsupportedError):
        ba.forward(q, q, q, quantize_pv=True, block_cols=80)
    with pytest.raises(pkg.UnsupportedError):
        ba.forward(q, q, q, quantize_pv=True, kernel="tcgen05")


@pytest.mark.parametrize("n,d,g", [(256, 64, 16), (1024, 72, 32), (4096, 64, 64), (576, 64, 24)])
def test_relative_2d_bias(ba, port, n, d, g):
    """Relative2dBias (attention.hpp:22-26, attention.cpp:78-96) through BA_BIAS_REL2D: generated inside the second-generation
    kernel (N = 1024, 4096: g % 32 == 0) or expanded on the device into the handle's table (N = 256, 576), checked against
    the oracle fed the reference's own materialize_bias table; a non-square N is a ShapeError like the reference's."""
    import torch
    import paper_2603_09582_b200 as pkg
    q, k, v, _ = make_head_inputs(port, 43, 0, n, d)
    rng = np.random.default_rng(9)
    ro, co = (cpu.bf16_round(0.5 * rng.standard_normal(2 * g - 1)) for _ in range(2))
    table = port.bias_rel2d(ro, co, n)
    Q, K, V = (to_torch(x[None, None], "bf16") for x in (q, k, v))
    rel = pkg.Relative2dBias(to_torch(ro, "f32"), to_torch(co, "f32"))
    assert np.array_equal(rel.materialize(n)[0].cpu().numpy().astype(np.float64), table)
    O = ba.forward(Q, K, V, rel)
    if n <= 1024:
        y = port.binary_attention_fused(q, k, v, bias=table)[0]
        assert np.abs(O[0, 0].cpu().numpy().astype(np.float64) - y).max() <= TOL_O
    else:  # a whole head of N = 4096 takes the oracle too long: the dense path (itself oracle-checked) fed the same table
        Od = ba.forward(Q, K, V, torch.from_numpy(table).to("cuda", torch.float32)[None])
        assert (O - Od).abs().max().item() <= TOL_O
    with pytest.raises(pkg.ShapeError):
        ba.forward(Q[:, :, :200], K[:, :, :200], V[:, :, :200], rel)


def test_relative_2d_bias_in_kernel_bit_identical(ba, port, monkeypatch):
    """In-kernel generation vs the same kernel's dense path fed materialize_bias' table: bit-identical when every sum
    row + col is bf16-representable (offsets on a 1/8 grid), per-head tables, bf16 and fp32 offsets."""
    import torch
    import paper_2603_09582_b200 as pkg
    monkeypatch.setenv("BA_TC2_MIN_N_BIAS", "512")  # the dense call must run on the second-generation kernel too (dev knob)
    B, H, n, d, g = 2, 3, 1024, 64, 32
    gen = torch.Generator(device="cuda").manual_seed(44)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(3))
    for dt in (torch.float32, torch.bfloat16):
        ro = (torch.randint(-8, 9, (H, 2 * g - 1), device="cuda", generator=gen).float() / 8).to(dt)
        co = (torch.randint(-8, 9, (H, 2 * g - 1), device="cuda", generator=gen).float() / 8).to(dt)
        rel = pkg.Relative2dBias(ro, co)
        table = rel.materialize(n).to(torch.bfloat16)   # exact: sums are multiples of 1/8 in [-2, 2]
        assert torch.equal(table.float(), rel.materialize(n).float())
        assert torch.equal(ba.forward(Q, K, V, rel), ba.forward(Q, K, V, table))


def test_torch_library_op(ba, port):
    """torch.ops.binattn.binary_attention / _rel1d: same bytes as the handle API, and traceable through the fake kernel."""
    import torch
    import paper_2603_09582_b200 as pkg
    import paper_2603_09582_b200.torch_op  # noqa: F401  (registers the ops)
    n, d = 197, 64
    heads = [make_head_inputs(port, 42, s, n, d, bias_scale=0.5) for s in range(2)]
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    bias = to_torch(np.stack([h[3] for h in heads]), "bf16")
    assert torch.equal(torch.ops.binattn.binary_attention(Q, K, V, bias, None), ba.forward(Q, K, V, bias))
    assert torch.equal(torch.ops.binattn.binary_attention(Q, K, V, None, 0.2), ba.forward(Q, K, V, None, 0.2))
    off = 0.5 * torch.randn(2, 2 * n - 1, device="cuda")
    assert torch.equal(torch.ops.binattn.binary_attention_rel1d(Q, K, V, off, None),
                       ba.forward(Q, K, V, pkg.Relative1dBias(off)))
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode():
        fq = torch.empty(1, 2, n, d, dtype=torch.bfloat16, device="cuda")
        out = torch.ops.binattn.binary_attention(fq, fq, fq, None, None)
        assert out.shape == (1, 2, n, d) and out.dtype == torch.float32
        out = torch.ops.binattn.binary_attention_ex(fq, fq, fq, None, None, True, True)
        assert out.shape == (1, 2, n, d) and out.dtype == torch.bfloat16
    # the extended op: the reference's default integer P.V arithmetic and / or bfloat16 output
    assert torch.equal(torch.ops.binattn.binary_attention_ex(Q, K, V, bias, None, True, False), ba.forward(Q, K, V, bias, quantize_pv=True))
    assert torch.equal(torch.ops.binattn.binary_attention_ex(Q, K, V, bias, None, False, True),
                       ba.forward(Q, K, V, bias).to(torch.bfloat16))


def test_packed_planes_as_batf_files(ba, port, tmp_path):
    """the sign planes K1 writes go to a BATF packed-bit file (dtype 4) byte-identical to the one the
    oracle's pack produces, and the reference's strict reader (zero pad bits!) accepts it when oracle/_ref is on the box."""
    import ctypes as C
    from paper_2603_09582_b200 import batf
    n, d = 197, 72
    q = make_head_inputs(port, 41, 0, n, d)[0]
    words, _ = ba.pack_signs(to_torch(q[None, None], "bf16"))
    ours, want = tmp_path / "gpu.batf", tmp_path / "cpu.batf"
    batf.write_tensor(ours, words_to_numpy(words[0, 0]), batf.PACKED_BIT, cols=d)
    batf.write_tensor(want, port.pack_signs(q), batf.PACKED_BIT, cols=d)
    assert ours.read_bytes() == want.read_bytes()
    R = cpu.ref()
    if R is not None:
        R.lib.ref_read_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        dt, rows, cols = C.c_int(), C.c_size_t(), C.c_size_t()
        back = np.zeros((n, 2), np.uint64)
        assert R.lib.ref_read_tensor(str(ours).encode(), C.byref(dt), C.byref(rows), C.byref(cols), None, back.ctypes.data,
                                     None, None) == 0
        assert (dt.value, rows.value, cols.value) == (4, n, d) and np.array_equal(back, port.pack_signs(q))


def test_large_logit_scale_rescale_path(ba, port):
    """Inputs scaled by 16 make mu_q*mu_k/tau ~ 20 per unit of dot: row maxima move by far more than the lazy-rescale
    threshold from tile to tile, so the O/l rescale branch runs for real; the result must still match the oracle.
    In this regime a row's weight sits on two or three tied keys, so the 2^-9 rounding of each bf16 weight no longer
    averages out: the tensor-core path is held to its guaranteed bound 2^-8 * max|V| (each bf16 weight is within 2^-9
    relative of exp(S - m), so |dO| <= 2^-9 * max_j |v_j - O| <= 2^-8 * max|V|; stated in include/binattn_cuda.h with a
    measured error-vs-peakedness table in INTEGRATION.md) instead of the typical-input bar."""
    n, d = 300, 64
    heads = []
    for s in range(2):
        q, k, v, b = make_head_inputs(port, 22, s, n, d, bias_scale=0.5)
        heads.append((q * 16.0, k * 16.0, v, b))  # power of two: still exactly representable in bf16
    bound = 2.0 ** -8 * max(float(np.abs(h[2]).max()) for h in heads)
    run_and_compare(ba, port, heads, n, d, "bf16", "per_head", tol={"tcgen05": bound})


def test_error_codes_on_device(ba):
    import torch
    import paper_2603_09582_b200 as pkg
    q = torch.zeros(1, 1, 4, 8, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(pkg.ShapeError):
        ba.forward(q, q[:, :, :, :4], q)
    with pytest.raises(pkg.ValidationError):  # attention.cpp:24-25
        ba.forward(q, q, q, None, 0.0)
    with pytest.raises(pkg.ShapeError):  # attention.cpp:60-61
        ba.forward(q, q, q, torch.zeros(1, 3, 3, device="cuda"))
    with pytest.raises(pkg.ShapeError):  # quantize.cpp:17
        ba.pack_signs(torch.zeros(1, 1, 0, 8, device="cuda"))


def test_full_size_c2_properties(ba, port):
    """BASELINE.json configs[1] (DeiT-B, B=256 H=12 N=197 d=64) at full size: sampled heads against the oracle,
    plus size-independent properties (key-permutation invariance, rows of P sum to one via V = 1)."""
    import torch
    B, H, n, d = 256, 12, 197, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, n, n, device="cuda", generator=g)).to(torch.bfloat16)
    for kern in kernels_for(ba, B, H, n, d, "bf16", bias):
        O = ba.forward(Q, K, V, bias, kernel=kern)
        assert torch.isfinite(O).all()
        for (b, h) in [(0, 0), (17, 5), (255, 11)]:
            f = lambda t: t[b, h].float().cpu().numpy().astype(np.float64)
            y = port.binary_attention_fused(f(Q), f(K), f(V), bias=bias[h].float().cpu().numpy().astype(np.float64))[0]
            assert np.abs(O[b, h].cpu().numpy() - y).max() <= TOL_O
        ones = ba.forward(Q[:8], K[:8], torch.ones_like(V[:8]), bias, kernel=kern)
        assert (ones - 1.0).abs().max().item() <= 1e-3  # softmax rows sum to one
        perm = torch.randperm(n, device="cuda", generator=g)
        Op = ba.forward(Q[:8], K[:8, :, perm], V[:8, :, perm], bias[:, :, perm], kernel=kern)
        # attention is a set function of (k_j, v_j, b_ij); two bf16-P runs with different tile groupings may each sit
        # ~7e-4 from the exact result (SURVEY.md 8c error budget), so the pairwise bound is the parity bound itself
        assert (Op - O[:8]).abs().max().item() <= TOL_O


@pytest.mark.parametrize("n,d", [(197, 64), (256, 72), (130, 128), (64, 32), (300, 96), (200, 64), (72, 128)])
def test_tensor_core_logits_bit_exact(ba, port, n, d):
    """The e4m3 +-1 tcgen05 contraction inside the fused kernel reproduces the integer logits exactly
    (debug dump of the TMEM accumulators; BASELINE.json: 'integer QK^T logits must be bit-exact')."""
    import ctypes as C
    import torch
    if ba.select_kernel(1, 2, n, d, torch.bfloat16) != "tcgen05":
        pytest.skip("tcgen05 kernel does not take this shape")
    heads = [make_head_inputs(port, 21, s, n, d) for s in range(2)]
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    S = torch.full((n, n), -12345, dtype=torch.int32, device="cuda")
    ba.lib.ba_debug_tcgen05_logits.argtypes = [C.c_void_p, C.c_int]
    ba.lib.ba_debug_tcgen05_logits(C.c_void_p(S.data_ptr()), 1)
    try:
        ba.forward(Q, K, V, None, kernel="tcgen05")
        torch.cuda.synchronize()
    finally:
        ba.lib.ba_debug_tcgen05_logits(None, -1)
    want = port.binary_gemm(port.pack_signs(heads[1][0]), port.pack_signs(heads[1][1]), d)
    assert np.array_equal(S.cpu().numpy(), want)


def test_full_size_c4_properties(ba, port):
    """BASELINE.json configs[3] (DiT-XL/2 at 512 px: B=32 H=16 N=1024 d=72, dense per-head bias) at full size: sampled
    heads against the oracle, rows of P sum to one, linearity in V."""
    import torch
    B, H, n, d = 32, 16, 1024, 72
    g = torch.Generator(device="cuda").manual_seed(4)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, n, n, device="cuda", generator=g)).to(torch.bfloat16)
    O = ba.forward(Q, K, V, bias)
    assert torch.isfinite(O).all()
    for (b, h) in [(0, 0), (13, 7), (31, 15)]:
        f = lambda t: t[b, h].float().cpu().numpy().astype(np.float64)
        y = port.binary_attention_fused(f(Q), f(K), f(V), bias=bias[h].float().cpu().numpy().astype(np.float64))[0]
        assert np.abs(O[b, h].cpu().numpy() - y).max() <= TOL_O
    ones = ba.forward(Q[:4], K[:4], torch.ones_like(V[:4]), bias)
    assert (ones - 1.0).abs().max().item() <= 1e-3
    V2 = torch.randn(4, H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    Vs = (V[:4].float() + V2.float()).to(torch.bfloat16)   # rounded sum: compare against the same rounded operand
    lin = ba.forward(Q[:4], K[:4], Vs, bias) - (O[:4] + ba.forward(Q[:4], K[:4], V2, bias))
    dv = (Vs.float() - V[:4].float() - V2.float()).abs().max().item()
    assert lin.abs().max().item() <= dv + 2 * 1e-3         # O is linear in V up to V's own rounding and the bf16 weights


@pytest.mark.parametrize("with_rel1d", [False, True])
def test_full_size_c5_properties(ba, port, with_rel1d):
    """BASELINE.json configs[4] at its largest point (B=1 H=16 N=16384 d=128): a whole-head oracle run would take minutes,
    so sampled ROWS are checked against a row-wise numpy restatement of attention.cpp:289-364 fed the oracle's own sign
    planes and scales (quantize.cpp:16-23), next to the size-independent properties."""
    import torch
    import paper_2603_09582_b200 as pkg
    B, H, n, d = 1, 16, 16384, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    offs = (0.5 * torch.randn(H, 2 * n - 1, device="cuda", generator=g)).to(torch.bfloat16).float() if with_rel1d else None
    bias = pkg.Relative1dBias(offs) if with_rel1d else None
    O = ba.forward(Q, K, V, bias)
    assert torch.isfinite(O).all()
    rng = np.random.default_rng(9)
    for h in (0, 9, 15):
        q, k, v = (t[0, h].float().cpu().numpy().astype(np.float64) for t in (Q, K, V))
        (_, mu_q), (_, mu_k) = port.binary_quantize(q), port.binary_quantize(k)
        sk = np.where(k >= 0.0, 1.0, -1.0)
        for r in [0, n - 1] + [int(x) for x in rng.integers(0, n, size=3)]:
            dot = sk @ np.where(q[r] >= 0.0, 1.0, -1.0)                       # integer-valued, exact in fp64
            s = mu_q * mu_k * dot / np.sqrt(d)                                # attention.cpp:34-36
            if with_rel1d:
                s = s + offs[h].cpu().numpy().astype(np.float64)[r - np.arange(n) + n - 1]   # attention.cpp:65-76
            p = np.exp(s - s.max())
            y = (p / p.sum()) @ v
            assert np.abs(O[0, h, r].cpu().numpy() - y).max() <= TOL_O
    ones = ba.forward(Q[:, :2], K[:, :2], torch.ones_like(V[:, :2]),
                      pkg.Relative1dBias(offs[:2]) if with_rel1d else None)
    assert (ones - 1.0).abs().max().item() <= 1e-3
    if not with_rel1d:
        perm = torch.randperm(n, device="cuda", generator=g)
        Op = ba.forward(Q[:, :2], K[:, :2][:, :, perm], V[:, :2][:, :, perm])
        assert (Op - O[:, :2]).abs().max().item() <= TOL_O


@pytest.mark.parametrize("n,d", [(197, 64), (577, 64), (2049, 64), (130, 128)])
def test_contiguous_bias_table_with_unaligned_rows(ba, n, d):
    """A contiguous [H,N,N] bf16 table with N % 8 != 0 (rows that are not 16-byte multiples: what a caller of the reference
    naturally holds for N = 197) is re-laid with padded rows once per call and takes the same TMA path as a padded table: the
    two give the same bits, in the bf16 mode and in the integer mode; BA_NO_BIAS_PAD=1 keeps the direct-load path alive."""
    import os
    import torch
    g = torch.Generator(device="cuda").manual_seed(13)
    Q, K, V = (torch.randn(2, 3, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    padded = (0.5 * torch.randn(3, n, (n + 7) // 8 * 8, device="cuda", generator=g)).to(torch.bfloat16)[:, :, :n]
    contig = padded.contiguous()
    assert contig.stride(1) == n and padded.stride(1) != n
    a = ba.forward(Q, K, V, padded)
    assert torch.equal(ba.forward(Q, K, V, contig), a)
    assert torch.equal(ba.forward(Q, K, V, contig[:1]), ba.forward(Q, K, V, padded[:1]))  # one shared table
    assert torch.equal(ba.forward(Q, K, V, contig, quantize_pv=True), ba.forward(Q, K, V, padded, quantize_pv=True))
    os.environ["BA_NO_BIAS_PAD"] = "1"
    try:
        slow = ba.forward(Q, K, V, contig)
    finally:
        del os.environ["BA_NO_BIAS_PAD"]
    assert float((slow - a).abs().max()) <= 2e-3  # the direct-load path (first-generation kernel for every N): same math, other tiling
