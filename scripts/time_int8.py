"""Dev tool: time the quantize_pv=true (integer P.V, CUDA-core) path next to the tensor-core product path."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
for (B, H, N, d) in [(256, 12, 197, 64), (64, 16, 256, 72), (32, 16, 1024, 72), (1, 16, 4096, 64)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    for name, kw in (("fp P.V (tcgen05)", {}), ("int8 P.V (CUDA cores)", {"quantize_pv": True})):
        for _ in range(2):
            ba.forward(Q, K, V, bias, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ba.forward(Q, K, V, bias, **kw)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"B{B} H{H} N{N} d{d} {name:22s} {ms:8.3f} ms  {4.0*B*H*N*N*d/ms/1e9:7.1f} eff. TOPS", flush=True)
