"""Dev tool: C2 / C3-like shapes with the dense bias as a CONTIGUOUS [H,N,N] table (rows not 16-byte multiples when N % 8 != 0)
against the same table with rows padded to 16 bytes, bf16 mode and integer mode."""
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
for (B, H, N, d) in [(256, 12, 197, 64), (64, 12, 577, 64), (8, 16, 2049, 64)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    padded = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    contig = padded.contiguous()
    same = torch.equal(ba.forward(Q, K, V, padded), ba.forward(Q, K, V, contig))
    print(f"B{B} H{H} N{N} d{d}: bf16 mode padded {t(lambda: ba.forward(Q, K, V, padded)):.4f} ms  contiguous {t(lambda: ba.forward(Q, K, V, contig)):.4f} ms (same bits: {same});"
          f"  integer mode padded {t(lambda: ba.forward(Q, K, V, padded, quantize_pv=True)):.4f} ms  contiguous {t(lambda: ba.forward(Q, K, V, contig, quantize_pv=True)):.4f} ms", flush=True)
