"""Dev tool: run a few forward calls of one shape (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
B, H, N, d = [int(x) for x in sys.argv[1:5]]
use_bias = sys.argv[5] == "1"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
qpv = len(sys.argv) > 7 and sys.argv[7] == "qpv"  # the reference's default integer P.V mode (tensor-core kernel)
ba = pkg.BinaryAttention(torch.device("cuda:0"))
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if use_bias else None
for _ in range(reps):
    O = ba.forward(Q, K, V, bias, kernel="tcgen05", quantize_pv=qpv)
torch.cuda.synchronize()
