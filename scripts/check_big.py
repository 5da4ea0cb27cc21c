"""Dev tool: index-overflow check -- a batch with more than 2^31 elements per tensor; sampled heads must equal the same heads
computed alone (bitwise), in the bf16 mode (no bias, per-head bias) and the integer mode."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
for (B, H, N, d) in [(600, 16, 4096, 128), (16000, 12, 197, 64)]:
    n_el = B * H * N * d
    print(f"B{B} H{H} N{N} d{d}: {n_el / 2**31:.2f} x 2^31 elements per tensor", flush=True)
    Q = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    K = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    V = torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16)
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    for name, kw in (("bf16 no bias", dict()), ("bf16 bias", dict(bias=bias)), ("integer mode", dict(bias=bias, quantize_pv=True))):
        O = ba.forward(Q, K, V, **kw)
        torch.cuda.synchronize()
        ok = True
        for b in (0, B // 2, B - 1):
            o1 = ba.forward(Q[b:b + 1], K[b:b + 1], V[b:b + 1], **kw)
            ok = ok and torch.equal(o1[0], O[b])
        print(f"   {name}: sampled batch elements equal the stand-alone call: {ok}   nan: {bool(torch.isnan(O[-1]).any())}", flush=True)
        del O
    del Q, K, V, bias
    torch.cuda.empty_cache()
