"""Dev tool: ragged-N shapes through the second-generation kernel (bf16 mode from 512 keys up, integer mode from 128)."""
import sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn):
    for _ in range(3): fn()
    ts = []
    for _ in range(11):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
for (B, H, N, d) in [(256, 12, 197, 64), (64, 12, 577, 64), (16, 16, 1025, 64), (8, 16, 2049, 128)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    print(f"B{B} H{H} N{N} d{d}: bf16 no bias {t(lambda: ba.forward(Q, K, V)):.4f}  bf16 bias {t(lambda: ba.forward(Q, K, V, bias)):.4f}  "
          f"integer no bias {t(lambda: ba.forward(Q, K, V, quantize_pv=True)):.4f}  integer bias {t(lambda: ba.forward(Q, K, V, bias, quantize_pv=True)):.4f} ms", flush=True)
