import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(1)
B, H, N, d = 4, 16, 1024, 72
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16)
for i in range(2):
    o = ba.forward(Q, K, V, bias); torch.cuda.synchronize()
print("done", float(o.abs().max()))
