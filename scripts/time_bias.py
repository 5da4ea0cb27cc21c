"""Dev tool: K1 + K2 time of the long-sequence shapes with a dense bias (and without), median of several L2-cold runs."""
import os, sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
shapes = [(1, 16, 16384, 128), (1, 16, 16384, 64), (1, 16, 8192, 128), (1, 16, 4096, 64)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B, H, N, d) in shapes:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    for wb in (True, False):
        bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16) if wb else None
        for _ in range(3):
            ba.forward(Q, K, V, bias)
        ts = []
        for _ in range(9):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ba.forward(Q, K, V, bias); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        print(f"N{N} d{d} bias={wb}: {t:.3f} ms  ({4.0 * B * H * N * N * d / (t * 1e-3) / 1e12:.0f} eff. TOPS)  min {min(ts):.3f}", flush=True)
        del bias
