"""GPU parity of the caller-side diagnostics: attention-map rows for sampled query rows
(the reference's `with_probs` outputs) and attention_fidelity (fidelity.cpp:40-85), through the C ABI, against the CPU
oracle.  fp64 kernels that follow the reference's arithmetic: the bar is ~1e-12, and exact for the top-k overlap."""
import numpy as np
import pytest

from oracle import cpu
from tests.helpers import make_head_inputs, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ba():
    import torch
    import paper_2603_09582_b200 as pkg
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    return pkg.BinaryAttention(torch.device("cuda:0"))

TOL_P = 1e-12   # max-abs on fp64 probabilities (sums are block-tree ordered, the reference's are sequential)


def _abi_tau(d):
    """ba_params carries 1/tau as float32 (include/binattn_cuda.h): the oracle gets exactly that temperature."""
    return 1.0 / float(np.float32(1.0 / np.sqrt(d)))


def _stochastic(rng, n, cols):
    p = rng.random((n, cols))
    return p / p.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("n,d,bias_kind", [(197, 64, "dense"), (64, 32, None), (300, 72, "dense"), (130, 128, "rel1d"), (40, 200, None)])
def test_attention_map_rows_match_oracle(ba, port, n, d, bias_kind):
    import torch
    import paper_2603_09582_b200 as pkg
    H = 2
    heads = [make_head_inputs(port, 41, s, n, d, bias_scale=0.5 if bias_kind == "dense" else None) for s in range(H)]
    Q, K = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(2))
    rng = np.random.default_rng(3)
    bias, tables = None, [None] * H
    if bias_kind == "dense":
        tables = [h[3] for h in heads]
        bias = to_torch(np.stack(tables), "bf16")
    elif bias_kind == "rel1d":
        offs = cpu.bf16_round(0.5 * rng.standard_normal((H, 2 * n - 1)))
        tables = [port.bias_rel1d(offs[h], n) for h in range(H)]
        bias = pkg.Relative1dBias(to_torch(offs, "f32"))
    rows = sorted(set([0, n - 1] + [int(r) for r in rng.integers(0, n, size=12)]))
    tau = _abi_tau(d)
    for h in range(H):
        q, k, v, _ = heads[h]
        want_bin = port.binary_attention_unfused(q, k, v, tau=tau, bias=tables[h], with_probs=True)[3][rows]
        want_full = port.reference_attention(q, k, v, tau=tau, bias=tables[h], with_probs=True)[3][rows]
        got_bin = ba.attention_probs(Q, K, bias, head=h, rows=rows, binary=True).cpu().numpy()
        got_full = ba.attention_probs(Q, K, bias, head=h, rows=rows, binary=False).cpu().numpy()
        assert got_bin.shape == (len(rows), n)
        assert np.abs(got_bin - want_bin).max() <= TOL_P
        assert np.abs(got_full - want_full).max() <= TOL_P
        assert np.abs(got_bin.sum(axis=1) - 1.0).max() <= 1e-12
        # the metric the reference's harness reports: full-precision map vs binary map (same rows on both sides)
        for kk in (1, 5, 1000 if n <= 128 else 64):
            want = port.attention_fidelity(want_full, want_bin, kk)
            got = ba.attention_fidelity(torch.from_numpy(want_full).cuda(), torch.from_numpy(want_bin).cuda(), kk)
            assert got.precision_at_k == want[3]
            assert np.allclose([got.cos_sim, got.relative_l1, got.rmse], want[:3], rtol=1e-12, atol=0)


def test_all_rows_default_and_row_order(ba, port):
    n, d = 70, 64
    q, k, v, _ = make_head_inputs(port, 42, 0, n, d)
    Q, K = (to_torch(x[None, None], "bf16") for x in (q, k))
    want = port.binary_attention_unfused(q, k, v, tau=_abi_tau(d), with_probs=True)[3]
    assert np.abs(ba.attention_probs(Q, K).cpu().numpy() - want).max() <= TOL_P
    got = ba.attention_probs(Q, K, rows=[5, 3, 5]).cpu().numpy()   # any order, repeats allowed
    assert np.abs(got - want[[5, 3, 5]]).max() <= TOL_P


def test_fidelity_known_answers(ba):
    """The reference's own KATs (test_fidelity.cpp:70-135) through the CUDA path."""
    import torch
    rng = np.random.default_rng(61)
    p = torch.from_numpy(_stochastic(rng, 6, 6)).cuda()
    r = ba.attention_fidelity(p, p, 3)                                             # :70-78
    assert abs(r.cos_sim - 1.0) <= 4e-16 and (r.relative_l1, r.rmse, r.precision_at_k) == (0.0, 0.0, 1.0)
    n = 4
    uni = torch.full((n, n), 1.0 / n, dtype=torch.float64).cuda()
    hot0, hot2 = torch.zeros((n, n), dtype=torch.float64), torch.zeros((n, n), dtype=torch.float64)
    hot0[:, 0] = 1.0
    hot2[:, 2] = 1.0
    assert ba.attention_fidelity(hot0.cuda(), uni, 1).precision_at_k == 1.0        # :80-87 ties go to the lower column
    assert ba.attention_fidelity(hot2.cuda(), uni, 1).precision_at_k == 0.0
    a, b = (torch.from_numpy(_stochastic(rng, 4, 4)).cuda() for _ in range(2))
    r = ba.attention_fidelity(a, b, 100)                                           # :111-118 k clamps to N
    assert r.precision_at_k == 1.0 and r.k == 100
    a, b = (torch.from_numpy(_stochastic(rng, 5, 7)).cuda() for _ in range(2))
    assert ba.attention_fidelity(a, b, 2).rmse == ba.attention_fidelity(b, a, 2).rmse  # :120-135


@pytest.mark.parametrize("rows,cols,k", [(8, 8, 3), (33, 197, 10), (5, 4096, 32), (3, 1000, 128)])
def test_fidelity_random_matches_oracle(ba, port, rows, cols, k):
    import torch
    rng = np.random.default_rng(rows * 1000 + cols)
    a, b = _stochastic(rng, rows, cols), _stochastic(rng, rows, cols)
    b[0, :] = a[0, :]                      # a tied row
    if cols >= 8:
        a[1, :8] = a[1, 0]                 # ties inside a row (renormalised below)
        a[1] /= a[1].sum()
    want = port.attention_fidelity(a, b, k)
    got = ba.attention_fidelity(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), k)
    assert got.precision_at_k == want[3]
    assert np.allclose([got.cos_sim, got.relative_l1, got.rmse], want[:3], rtol=1e-12, atol=0)
    again = ba.attention_fidelity(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), k)
    assert again == got                    # deterministic


def test_fidelity_and_probs_errors(ba):
    import torch
    import paper_2603_09582_b200 as pkg
    a = torch.from_numpy(_stochastic(np.random.default_rng(66), 4, 4)).cuda()
    with pytest.raises(pkg.ShapeError):        # test_fidelity.cpp:163-167
        ba.attention_fidelity(a, torch.from_numpy(_stochastic(np.random.default_rng(1), 5, 5)).cuda(), 2)
    with pytest.raises(pkg.ValidationError):   # :168-169 rows sum to 2
        ba.attention_fidelity(a, torch.full((4, 4), 0.5, dtype=torch.float64).cuda(), 2)
    with pytest.raises(pkg.ValidationError):   # fidelity.cpp:44
        ba.attention_fidelity(a, a, 0)
    with pytest.raises(pkg.UnsupportedError):
        big = torch.full((2, 1000), 1e-3, dtype=torch.float64).cuda()
        ba.attention_fidelity(big, big, 500)
    Q = torch.randn(1, 1, 16, 64, device="cuda").to(torch.bfloat16)
    with pytest.raises(pkg.ShapeError):
        ba.attention_probs(Q, Q, rows=[16])
    with pytest.raises(pkg.ShapeError):
        ba.attention_probs(Q, Q, head=1)
