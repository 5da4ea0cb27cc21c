"""Parity tests of the second-generation tcgen05 kernel (csrc/attn_tc2.cuh; N >= 512, bf16, d % 8 == 0, d <= 128) through
the C ABI, against the CPU oracle on identical inputs, plus the large dense-bias shapes the N-sweep times (sampled rows)
and a run-to-run identity stress (a protocol race in a warp-specialised kernel shows up as an output that differs between
two runs of the same call long before it shows up as a wrong answer).

Bars as in test_gpu_parity.py: integer logits bit-exact, O within 2e-3 max-abs of the reference's fp64 path.
"""
import ctypes as C
import os

import numpy as np
import pytest

from tests.helpers import make_head_inputs, to_torch
from tests.test_gpu_parity import TOL_O, ba, run_and_compare  # noqa: F401  (ba is a fixture)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def tc2_takes_small_bias_shapes():
    """The dispatcher hands dense-bias shapes below 2048 keys to the first-generation kernel (it is level or ahead there);
    these tests are about the second generation, so it takes them from 512 keys on (dev knob read at every launch)."""
    os.environ["BA_TC2_MIN_N_BIAS"] = "512"
    yield
    os.environ.pop("BA_TC2_MIN_N_BIAS", None)


@pytest.fixture()
def gen1_only():
    """Route the tcgen05 path to the first-generation kernel for one test (dev switch read at every launch)."""
    os.environ["BA_TC2"] = "0"
    yield
    os.environ.pop("BA_TC2", None)


@pytest.mark.parametrize("bias_mode", [None, "per_head", "shared"])
@pytest.mark.parametrize("n,d", [(512, 64), (640, 32), (777, 72), (1023, 64), (1024, 128), (513, 96), (896, 8)])
def test_tc2_matches_oracle(ba, port, n, d, bias_mode):
    """Whole heads against binary_attention_fused (attention.cpp:250-382): whole and ragged key tiles, an odd number of
    128-row blocks (tile B of the last unit empty or partial), every padded head dim, with the row_max / row_sum outputs
    (general path) -- run_and_compare asks for them."""
    heads = [make_head_inputs(port, 31, s, n, d, bias_scale=0.5) for s in range(2)]
    run_and_compare(ba, port, heads, n, d, "bf16", bias_mode)


@pytest.mark.parametrize("n,d", [(512, 64), (1000, 72), (768, 128)])
def test_tc2_fast_path_without_stats(ba, port, n, d):
    """Without a bias and without the row_max / row_sum outputs the kernel takes its no-row-max path (reference = the a priori
    bound d*mu_q*mu_k/tau); O must match the oracle just the same, and the general path bit for bit in what it multiplies."""
    import torch
    heads = [make_head_inputs(port, 32, s, n, d) for s in range(3)]
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    O = ba.forward(Q, K, V, None, kernel="tcgen05")
    O2, _, _ = ba.forward(Q, K, V, None, kernel="tcgen05", return_stats=True)
    torch.cuda.synchronize()
    for h, (q, k, v, _) in enumerate(heads):
        y = port.binary_attention_fused(q, k, v)[0]
        assert np.abs(O[0, h].cpu().numpy() - y).max() <= TOL_O
        assert np.abs(O2[0, h].cpu().numpy() - y).max() <= TOL_O


@pytest.mark.parametrize("n,d", [(512, 64), (640, 72), (1024, 128), (768, 32)])
def test_tc2_logits_bit_exact(ba, port, n, d):
    """TMEM accumulators of the S MMA, dumped by the kernel's debug instantiation: == binary_gemm (bitops.cpp:96-131)."""
    import torch
    heads = [make_head_inputs(port, 33, s, n, d) for s in range(2)]
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


def test_tc2_rescale_path(ba, port):
    """Inputs scaled by 16: the a priori bound is far above 2^32, so the general path runs, and row maxima move by more than
    the lazy threshold between tiles -- the O / l rescale (both column halves of a row agreeing on the new reference
    through shared memory) runs for real.  A row's weight then sits on two or three tied keys and the 2^-9 rounding of the
    bf16 weights no longer averages out: the bar is the guaranteed bound of the bf16-P path, 2^-8 * max|V| (each weight is
    within 2^-9 relative of exp(S - m), so |dO| <= 2^-9 * max_j |v_j - O| <= 2^-8 * max|V|; include/binattn_cuda.h)."""
    n, d = 768, 64
    heads = []
    for s in range(2):
        q, k, v, b = make_head_inputs(port, 34, s, n, d, bias_scale=0.5)
        heads.append((q * 16.0, k * 16.0, v, b))
    bound = 2.0 ** -8 * max(float(np.abs(h[2]).max()) for h in heads)
    run_and_compare(ba, port, heads, n, d, "bf16", "per_head", tol={"tcgen05": bound})
    run_and_compare(ba, port, heads, n, d, "bf16", None, tol={"tcgen05": bound})


def test_gen1_still_matches_on_tc2_shapes(ba, port, gen1_only):
    heads = [make_head_inputs(port, 35, s, 640, 72, bias_scale=0.5) for s in range(2)]
    run_and_compare(ba, port, heads, 640, 72, "bf16", "per_head")


def _sampled_rows_check(port, O, Q, K, V, bias, heads, rows):
    """Row-wise numpy restatement of attention.cpp:289-364 fed the oracle's own scales (quantize.cpp:16-23): exact integer
    dots in fp64, dense bias row, softmax, P.V.  (Sampled rows stand in for whole heads: one head of N = 8192 takes the
    oracle minutes.)"""
    n, d = Q.shape[-2], Q.shape[-1]
    for h in heads:
        q, k, v = (t[0, h].float().cpu().numpy().astype(np.float64) for t in (Q, K, V))
        (_, mu_q), (_, mu_k) = port.binary_quantize(q), port.binary_quantize(k)
        sk = np.where(k >= 0.0, 1.0, -1.0)
        for r in rows:
            dot = sk @ np.where(q[r] >= 0.0, 1.0, -1.0)
            s = mu_q * mu_k * dot / np.sqrt(d)
            if bias is not None:
                s = s + bias[h, r].float().cpu().numpy().astype(np.float64)
            p = np.exp(s - s.max())
            y = (p / p.sum()) @ v
            assert np.abs(O[0, h, r].cpu().numpy() - y).max() <= TOL_O, f"head {h} row {r}"


@pytest.mark.parametrize("n", [4096, 8192])
@pytest.mark.parametrize("d", [64, 128])
def test_sweep_shapes_with_dense_bias(ba, port, n, d):
    """The kernels the N-sweep times with a dense per-head bf16 bias (BASELINE.json configs[4], H = 16): sampled rows of
    sampled heads against the row-wise restatement, and rows of P sum to one."""
    import torch
    H = 16
    g = torch.Generator(device="cuda").manual_seed(6)
    Q, K, V = (torch.randn(1, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, n, n, device="cuda", generator=g)).to(torch.bfloat16)
    O = ba.forward(Q, K, V, bias)
    assert torch.isfinite(O).all()
    rng = np.random.default_rng(10)
    _sampled_rows_check(port, O, Q, K, V, bias, (0, 7, 15), [0, 127, 128, n - 1] + [int(x) for x in rng.integers(0, n, size=3)])
    ones = ba.forward(Q[:, :2], K[:, :2], torch.ones_like(V[:, :2]), bias[:2])
    assert (ones - 1.0).abs().max().item() <= 1e-3


def test_full_size_c5_d64(ba, port):
    """BASELINE.json configs[4] at N = 16384, d = 64, no bias (the no-row-max path at full length)."""
    import torch
    H, n, d = 16, 16384, 64
    g = torch.Generator(device="cuda").manual_seed(7)
    Q, K, V = (torch.randn(1, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    O = ba.forward(Q, K, V)
    assert torch.isfinite(O).all()
    rng = np.random.default_rng(11)
    _sampled_rows_check(port, O, Q, K, V, None, (0, 5, 15), [0, n - 1] + [int(x) for x in rng.integers(0, n, size=3)])
    perm = torch.randperm(n, device="cuda", generator=g)
    Op = ba.forward(Q[:, :2], K[:, :2][:, :, perm], V[:, :2][:, :, perm])
    assert (Op - O[:, :2]).abs().max().item() <= TOL_O


def test_full_size_c3(ba, port):
    """BASELINE.json configs[2] (DiT-XL/2 at 256 px: B=64 H=16 N=256 d=72, dense per-head bias) at full size: sampled heads
    against the oracle, rows of P sum to one."""
    import torch
    B, H, n, d = 64, 16, 256, 72
    g = torch.Generator(device="cuda").manual_seed(8)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, n, n, device="cuda", generator=g)).to(torch.bfloat16)
    O = ba.forward(Q, K, V, bias)
    assert torch.isfinite(O).all()
    for (b, h) in [(0, 0), (17, 3), (40, 9), (63, 15)]:
        f = lambda t: t[b, h].float().cpu().numpy().astype(np.float64)
        y = port.binary_attention_fused(f(Q), f(K), f(V), bias=bias[h].float().cpu().numpy().astype(np.float64))[0]
        assert np.abs(O[b, h].cpu().numpy() - y).max() <= TOL_O
    ones = ba.forward(Q, K, torch.ones_like(V), bias)
    assert (ones - 1.0).abs().max().item() <= 1e-3


@pytest.mark.parametrize("B,H,n,d,with_bias,stats", [(4, 16, 1024, 72, True, False), (1, 2, 512, 128, True, False), (2, 4, 1024, 64, True, True),
                                                     (1, 8, 2048, 64, False, False), (3, 16, 768, 96, True, True), (1, 3, 577, 72, True, False)])
def test_run_to_run_identity_stress(ba, B, H, n, d, with_bias, stats):
    """60 runs of the same call must give the same bytes (multi-unit CTAs, bias ring, both softmax paths)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(9)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, n, (n + 7) // 8 * 8, device="cuda", generator=g)).to(torch.bfloat16)[:, :, :n] if with_bias else None
    first = None
    for _ in range(60):
        out = ba.forward(Q, K, V, bias, return_stats=stats)
        o = out[0] if stats else out
        torch.cuda.synchronize()
        if first is None:
            first = o.clone()
        else:
            assert torch.equal(o, first)


@pytest.mark.parametrize("B,H,n,d,dtype,with_bias", [(2, 3, 1024, 64, "bf16", True), (1, 5, 640, 72, "bf16", False), (2, 3, 300, 64, "bf16", True),
                                                     (3, 2, 197, 64, "bf16", True), (1, 3, 300, 40, "f32", True), (1, 2, 1536, 128, "bf16", True)])
def test_unit_shards_reproduce_the_full_run(ba, B, H, n, d, dtype, with_bias):
    """(head, 256-row block) shards (ba_shard_units -> ba_params.unit_begin / unit_end) written into one
    output buffer by 3, 5 and 7 'ranks' give the full run byte for byte -- ranges that split heads, both tcgen05 kernels
    (N = 300: three 128-row blocks in two shard units) and the CUDA-core kernel."""
    import torch
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]
    g = torch.Generator(device="cuda").manual_seed(12)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(tdt) for _ in range(3))
    bias = None
    if with_bias:
        bias = (0.5 * torch.randn(H, n, (n + 7) // 8 * 8, device="cuda", generator=g)).to(torch.bfloat16 if dtype == "bf16" else torch.float32)[:, :, :n]
    full = ba.forward(Q, K, V, bias)
    total = B * H * ((n + 255) // 256)
    for world in (3, 5, 7):
        out = torch.full_like(full, float("nan"))
        covered = 0
        for r in range(world):
            b, e = ba.shard_units(B, H, n, world, r)
            covered += e - b
            ba.forward(Q, K, V, bias, units=(b, e), out=out)
        torch.cuda.synchronize()
        assert covered == total
        assert torch.equal(out, full), f"world {world}"
