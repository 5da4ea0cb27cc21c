"""ba_params.out_bf16: O written as bfloat16 by every kernel's epilogue must be bit-identical to the
float32 output rounded to bfloat16 afterwards (round-to-nearest-even both ways) -- through the first- and second-generation
tcgen05 kernels (staged TMA-store and direct-store epilogues), the CUDA-core kernels, unit-sharded calls and the host-buffer
entry point."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ba():
    import paper_2603_09582_b200 as pkg
    return pkg.BinaryAttention(torch.device("cuda:0"))


def _inputs(B, H, N, d, dtype=torch.bfloat16, with_bias=True, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    Q, K, V = (torch.randn(B, H, N, d, device="cuda", generator=g).to(dtype) for _ in range(3))
    bias = None
    if with_bias:
        ld = (N + 7) // 8 * 8
        bias = (0.5 * torch.randn(H, N, ld, device="cuda", generator=g)).to(torch.bfloat16)[:, :, :N]
    return Q, K, V, bias


# (B, H, N, d, bias, kernel, env): which epilogue each one reaches is noted beside it
CASES = [
    (2, 3, 197, 64, True, "auto", {}),                      # first generation, staged epilogue (C2 shape)
    (1, 2, 129, 128, False, "auto", {}),                    # first generation, wide head: the two staging boxes are reused
    (1, 2, 2048, 128, True, "auto", {"BA_TC2": "0"}),       # first generation, long units
    (1, 2, 300, 72, True, "auto", {"BA_O_STAGE": "0"}),     # first generation, direct stores
    (2, 4, 1024, 72, True, "auto", {"BA_TC2_MIN_N_BIAS": "512"}),  # second generation, staged epilogue (C4 shape)
    (1, 3, 577, 64, False, "auto", {}),                     # second generation, ragged N, staged
    (1, 2, 4096, 128, True, "auto", {}),                    # second generation, direct stores (tiles >= 64)
    (1, 2, 4096, 64, False, "auto", {}),
    (1, 2, 640, 96, False, "auto", {"BA_O_STAGE": "0"}),    # second generation, direct stores forced
    (1, 2, 150, 40, True, "simt", {}),                      # CUDA-core kernel
]


@pytest.mark.parametrize("B,H,N,d,wb,kernel,env", CASES)
def test_bf16_output_is_the_rounded_fp32_output(ba, monkeypatch, B, H, N, d, wb, kernel, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    Q, K, V, bias = _inputs(B, H, N, d, with_bias=wb)
    O32 = ba.forward(Q, K, V, bias, kernel=kernel)
    O16 = ba.forward(Q, K, V, bias, kernel=kernel, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert O16.dtype == torch.bfloat16 and O16.shape == O32.shape
    assert not torch.isnan(O32).any()
    assert torch.equal(O16, O32.to(torch.bfloat16))


def test_bf16_output_fp32_inputs_and_integer_pv(ba):
    Q, K, V, bias = _inputs(1, 2, 130, 48, dtype=torch.float32)
    assert torch.equal(ba.forward(Q, K, V, bias, out_dtype=torch.bfloat16), ba.forward(Q, K, V, bias).to(torch.bfloat16))
    Q, K, V, bias = _inputs(2, 2, 197, 64)
    a = ba.forward(Q, K, V, bias, quantize_pv=True, out_dtype=torch.bfloat16)
    b = ba.forward(Q, K, V, bias, quantize_pv=True)
    assert torch.equal(a, b.to(torch.bfloat16))


def test_bf16_output_unit_shards_and_stats(ba):
    Q, K, V, bias = _inputs(1, 3, 1024, 64, with_bias=False)
    O16, m, l = ba.forward(Q, K, V, bias, out_dtype=torch.bfloat16, return_stats=True)
    O32, m32, l32 = ba.forward(Q, K, V, bias, return_stats=True)
    assert torch.equal(m, m32) and torch.equal(l, l32)  # the statistics stay float32 and do not depend on the output type
    assert torch.equal(O16, O32.to(torch.bfloat16))
    whole = ba.forward(Q, K, V, bias, out_dtype=torch.bfloat16)
    out = torch.zeros_like(whole)
    total = 3 * 4
    for lo, hi in ((0, 5), (5, 6), (6, total)):
        ba.forward(Q, K, V, bias, units=(lo, hi), out=out, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert torch.equal(out, whole)


def test_bf16_output_host_entry_point(ba):
    Q, K, V, bias = _inputs(3, 4, 197, 64)
    ref = ba.forward(Q, K, V, bias).to(torch.bfloat16).cpu()
    hO = ba.forward_host(Q.cpu().pin_memory(), K.cpu().pin_memory(), V.cpu().pin_memory(), bias.contiguous().cpu(),
                         out_dtype=torch.bfloat16)
    assert hO.dtype == torch.bfloat16 and torch.equal(hO, ref)


def test_out_dtype_validation(ba):
    import paper_2603_09582_b200 as pkg
    Q, K, V, _ = _inputs(1, 1, 64, 32, with_bias=False)
    with pytest.raises(pkg.ValidationError):
        ba.forward(Q, K, V, out_dtype=torch.float16)
    with pytest.raises(pkg.ShapeError):
        ba.forward(Q, K, V, out=torch.empty(1, 1, 64, 32, device="cuda"), out_dtype=torch.bfloat16)


def test_host_entry_point_with_the_bias_resident_on_the_device(ba):
    """ba_params.bias_on_device: Q, K, V, O are host buffers, the bias table already lives on the GPU -- same bits as the call
    that copies the table from host memory."""
    Q, K, V, bias = _inputs(3, 4, 197, 64)
    hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
    a = ba.forward_host(hQ, hK, hV, bias.contiguous().cpu())
    b = ba.forward_host(hQ, hK, hV, bias)            # strided device view (row stride 200)
    c = ba.forward_host(hQ, hK, hV, bias.contiguous())
    assert torch.equal(a, b) and torch.equal(a, c)
    assert torch.equal(a, ba.forward(Q, K, V, bias).cpu())
