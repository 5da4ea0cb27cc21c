"""Dev tool: one tcgen05 forward with a relative-1d bias (for sanitizer runs)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
B, H, N, d = 1, 2, int(sys.argv[1]) if len(sys.argv) > 1 else 197, 64
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
O = ba.forward(Q, K, V, pkg.Relative1dBias(torch.randn(H, 2 * N - 1, device="cuda")), kernel="tcgen05")
torch.cuda.synchronize()
print("ok", float(O.abs().max()))
