"""Dev tool: K1 + K2 time with float32 and with bfloat16 output (ba_params.out_bf16), L2 flushed before every run."""
import sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B, H, N, d) in [(256, 12, 197, 64), (64, 12, 577, 64), (32, 16, 1024, 72), (1, 16, 4096, 64)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    res = {}
    for it in range(34):
        dt = (torch.float32, torch.bfloat16)[it & 1]
        if it < 4:
            ba.forward(Q, K, V, bias, out_dtype=dt); continue
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ba.forward(Q, K, V, bias, out_dtype=dt); e1.record(); torch.cuda.synchronize()
        res.setdefault(dt, []).append(e0.elapsed_time(e1))
    print(f"B{B} H{H} N{N} d{d} dense bias: fp32 O {statistics.median(res[torch.float32]):.4f} ms   bf16 O {statistics.median(res[torch.bfloat16]):.4f} ms", flush=True)
