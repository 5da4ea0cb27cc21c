"""Measured |O - fp64 reference| of the bf16-P tensor-core path against row peakedness (logit scale): inputs Q, K scaled by s,
so mu_q*mu_k/tau grows by s^2 and each row's weight concentrates on fewer keys.  Prints a markdown table for INTEGRATION.md."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(3)
H, N, d = 4, 1024, 64
Q0, K0, V = (torch.randn(1, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
print("| input scale s | mu_q mu_k / tau | effective keys per row (1 / sum p^2, median) | max abs error | bound 2^-8 max|V| |")
print("|---|---|---|---|---|")
for s in (1, 2, 4, 8, 16, 32):
    Q, K = Q0 * s, K0 * s
    q, k, v = Q.double(), K.double(), V.double()
    mu = q.abs().mean(dim=(-2, -1), keepdim=True) * k.abs().mean(dim=(-2, -1), keepdim=True)
    sq, sk = torch.where(q >= 0, 1.0, -1.0).double(), torch.where(k >= 0, 1.0, -1.0).double()
    P = torch.softmax(mu * (sq @ sk.transpose(-1, -2)) / d ** 0.5, dim=-1)
    ref = P @ v
    O = ba.forward(Q, K, V)
    err = (O.double() - ref).abs().max().item()
    neff = (1.0 / (P * P).sum(-1)).median().item()
    print(f"| {s} | {float(mu.mean()) / d ** 0.5:.3g} | {neff:.1f} | {err:.2e} | {2.0 ** -8 * V.abs().max().item():.2e} |")
