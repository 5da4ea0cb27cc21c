"""Dev tool: steps/s of forward() with no per-kernel profiling events (for launch-overlap experiments)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
B, H, N, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 12, 197, 64))]
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
for _ in range(5):
    ba.forward(Q, K, V, bias)
torch.cuda.synchronize()
best = 1e9
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        ba.forward(Q, K, V, bias)
    e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 50)
print(f"B{B} H{H} N{N} d{d}: {best*1e3:.1f} us per step (best of 5 x 50)")
