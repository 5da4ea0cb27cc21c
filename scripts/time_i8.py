"""Dev tool: K1 + K1v + K2 time of the integer P.V mode on the tensor cores, L2 flushed, a few shapes."""
import sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B, H, N, d) in [(256, 12, 197, 64), (32, 16, 1024, 72), (1, 16, 4096, 64), (1, 16, 16384, 64)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    for _ in range(3):
        ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05")
    ts = []
    for _ in range(9):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05"); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"B{B} H{H} N{N} d{d} bias, quantize_pv: {statistics.median(ts):.4f} ms  min {min(ts):.4f}", flush=True)
