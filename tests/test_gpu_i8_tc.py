"""quantize_pv = true on the tensor cores: the I8 mode of the
second-generation kernel -- u8 weights x s8 value levels through tcgen05.mma.kind::i8 into an s32 accumulator per 64-key
block, the reference's per-block running max and rescale (attention.cpp:306-343), epilogue O / l / 255 * delta (361-363) --
against the CPU oracle of the reference's default mode, against the CUDA-core kernel of the same mode, and through the
sharded / bf16-output / fallback paths.  Bars: the reference's own for this mode (max-abs 1e-3 against the oracle with the
same block size -- fp32 exp against fp64 exp can flip round(255 P) at a .5 boundary, one level = 1/255 of a weight -- and a
rel-L2 against the fp64 path no larger than the mode's own, cf. test_attention.cpp:300-314)."""
import numpy as np
import pytest

from tests.helpers import make_head_inputs, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ba():
    import torch
    import paper_2603_09582_b200 as pkg
    return pkg.BinaryAttention(torch.device("cuda:0"))


@pytest.mark.parametrize("bias_mode", [None, "per_head"])
@pytest.mark.parametrize("n,d", [(197, 64), (577, 64), (128, 16), (256, 32), (384, 48), (1024, 64), (130, 64), (639, 32),
                                 (256, 72), (1024, 72), (384, 128), (130, 104), (256, 40), (577, 96)])  # d > 64: one pass per 64 columns of V
def test_tensor_core_int8_pv_matches_reference_default(ba, port, n, d, bias_mode):
    heads = [make_head_inputs(port, 71, s, n, d, bias_scale=0.5 if bias_mode else None) for s in range(2)]
    Q, K, V = (to_torch(np.stack([h[i] for h in heads])[None], "bf16") for i in range(3))
    bias_t = to_torch(np.stack([h[3] for h in heads]), "bf16") if bias_mode else None
    if bias_t is not None and n % 8:  # rows of a dense bf16 table must be 16-byte multiples for the TMA path: pad the row stride
        import torch
        padded = torch.zeros(2, n, (n + 7) // 8 * 8, device="cuda", dtype=torch.bfloat16)
        padded[:, :, :n] = bias_t
        bias_t = padded[:, :, :n]
    O, m, l = ba.forward(Q, K, V, bias_t, quantize_pv=True, kernel="tcgen05", return_stats=True)
    Oc = ba.forward(Q, K, V, bias_t, quantize_pv=True, kernel="simt")
    assert float((O - Oc).abs().max()) <= 5e-4  # the CUDA-core kernel of the same mode (expf there, ex2 here: rare level flips)
    O = O.cpu().numpy().astype(np.float64)
    for h in range(2):
        q, k, v, b = heads[h]
        y8, om, ol = port.binary_attention_fused(q, k, v, bias=b, quantize_pv=True, block_cols=64)
        assert np.abs(O[0, h] - y8).max() <= 1e-3, np.abs(O[0, h] - y8).max()
        np.testing.assert_allclose(m[0, h].cpu().numpy(), om, rtol=0, atol=1e-4)
        np.testing.assert_allclose(l[0, h].cpu().numpy(), ol, rtol=2e-5)
        # against the fp64 path: the mode's own quantisation error (the reference bounds it by rel-L2 1e-2 on ITS test shapes,
        # test_attention.cpp:300-314; it grows slowly with N) -- ours must not add to what the oracle of the mode shows
        y64 = port.binary_attention_fused(q, k, v, bias=b)[0]
        rel_ours = np.linalg.norm(O[0, h] - y64) / np.linalg.norm(y64)
        rel_mode = np.linalg.norm(y8 - y64) / np.linalg.norm(y64)
        assert rel_ours <= rel_mode + 5e-4 and rel_ours <= 2e-2, (rel_ours, rel_mode)


def test_tensor_core_int8_pv_dispatch(ba, monkeypatch):
    """auto takes the tensor-core kernel where it fits (same bits as kernel="tcgen05"), the CUDA-core one elsewhere or when
    BA_TC2_I8=0; asking for the tensor cores on a shape they do not take is an error, not a silent fallback."""
    import torch
    import paper_2603_09582_b200 as pkg
    g = torch.Generator(device="cuda").manual_seed(3)
    Q, K, V = (torch.randn(2, 3, 320, 64, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    auto = ba.forward(Q, K, V, quantize_pv=True)
    assert torch.equal(auto, ba.forward(Q, K, V, quantize_pv=True, kernel="tcgen05"))
    cc = ba.forward(Q, K, V, quantize_pv=True, kernel="simt")
    assert not torch.equal(auto, cc) and float((auto - cc).abs().max()) <= 5e-4
    monkeypatch.setenv("BA_TC2_I8", "0")
    assert torch.equal(ba.forward(Q, K, V, quantize_pv=True), cc)
    monkeypatch.delenv("BA_TC2_I8")
    assert torch.equal(ba.forward(Q, K, V, quantize_pv=True, block_cols=32), ba.forward(Q, K, V, quantize_pv=True, block_cols=32, kernel="simt"))
    for shape, dt in (((1, 1, 96, 64), torch.bfloat16), ((1, 1, 256, 20), torch.bfloat16), ((1, 1, 256, 160), torch.bfloat16),
                      ((1, 1, 256, 64), torch.float32)):
        x = torch.randn(*shape, device="cuda").to(dt)
        ba.forward(x, x, x, quantize_pv=True)  # auto: the CUDA-core kernel
        with pytest.raises(pkg.UnsupportedError):
            ba.forward(x, x, x, quantize_pv=True, kernel="tcgen05")
    with pytest.raises(pkg.UnsupportedError):
        ba.forward(Q, K, V, quantize_pv=True, block_cols=32, kernel="tcgen05")


def test_tensor_core_int8_pv_shards_and_bf16_output(ba):
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    _shards_and_bf16(ba, 64)
    _shards_and_bf16(ba, 72)


def _shards_and_bf16(ba, d):
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    Q, K, V = (torch.randn(1, 3, 700, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(3, 700, 704, device="cuda", generator=g)).to(torch.bfloat16)[:, :, :700]
    whole = ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05")
    out = torch.zeros_like(whole)
    total = 3 * 3
    for lo, hi in ((0, 2), (2, 7), (7, total)):
        ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05", units=(lo, hi), out=out)
    torch.cuda.synchronize()
    assert torch.equal(out, whole)
    assert torch.equal(ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05", out_dtype=torch.bfloat16), whole.to(torch.bfloat16))
    runs = [ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05") for _ in range(20)]
    torch.cuda.synchronize()
    assert all(torch.equal(r, whole) for r in runs)  # run-to-run identical


def test_tensor_core_int8_pv_full_size_c2_sample(ba, port):
    """BASELINE configs[1] at full size (B=256, H=12, N=197, d=64, per-head bias): sampled heads against the oracle."""
    import torch
    B, H, n, d = 256, 12, 197, 64
    g = torch.Generator(device="cuda").manual_seed(11)
    Q, K, V = (torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, n, 200, device="cuda", generator=g)).to(torch.bfloat16)[:, :, :n]
    O = ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05")
    for (b, h) in ((0, 0), (117, 5), (255, 11)):
        q, k, v = (x[b, h].float().cpu().numpy().astype(np.float64) for x in (Q, K, V))
        y8 = port.binary_attention_fused(q, k, v, bias=bias[h].float().cpu().numpy().astype(np.float64), quantize_pv=True, block_cols=64)[0]
        assert np.abs(O[b, h].cpu().numpy().astype(np.float64) - y8).max() <= 1e-3


def test_tensor_core_int8_pv_long_sequence_sample(ba, port):
    """N = 4096 (64 key blocks, the long-sequence regime of BASELINE configs[4]): one head against the oracle of the mode."""
    import torch
    n, d = 4096, 64
    q, k, v, _ = make_head_inputs(port, 73, 0, n, d)
    Q, K, V = (to_torch(x[None, None], "bf16") for x in (q, k, v))
    O = ba.forward(Q, K, V, quantize_pv=True, kernel="tcgen05")[0, 0].cpu().numpy().astype(np.float64)
    y8 = port.binary_attention_fused(q, k, v, quantize_pv=True, block_cols=64)[0]
    assert np.abs(O - y8).max() <= 1e-3, np.abs(O - y8).max()


def test_tensor_core_int8_pv_through_the_host_entry_point(ba):
    """ba_binary_attention_host with quantize_pv = 1: the head grid flows through the chunked H2D / kernel / D2H pipeline, every
    chunk with its own workspace slice (packed planes, s8 levels, scales, expanded planes) -- same bits as the device call.
    A contiguous host bias table with 394-byte rows is re-laid with 16-byte rows on the device (once per call), so it stays on
    the tensor cores like the row-padded device-resident one."""
    import torch
    import paper_2603_09582_b200 as pkg
    g = torch.Generator(device="cuda").manual_seed(9)
    Q, K, V = (torch.randn(40, 12, 197, 64, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(12, 197, 200, device="cuda", generator=g)).to(torch.bfloat16)[:, :, :197]
    hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
    assert torch.equal(ba.forward_host(hQ, hK, hV, quantize_pv=True, kernel="tcgen05"), ba.forward(Q, K, V, quantize_pv=True, kernel="tcgen05").cpu())
    ref = ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05").cpu()
    assert torch.equal(ba.forward_host(hQ, hK, hV, bias, quantize_pv=True, kernel="tcgen05"), ref)  # bias resident on the device
    assert torch.equal(ba.forward_host(hQ, hK, hV, bias.contiguous().cpu(), quantize_pv=True, kernel="tcgen05"), ref)
    assert torch.equal(ba.forward(Q, K, V, bias.contiguous(), quantize_pv=True, kernel="tcgen05").cpu(), ref)
