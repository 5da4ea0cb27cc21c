"""Dev tool: one call of every non-tensor-core kernel (pack, logits, CUDA-core attention, int8 mode) for sanitizer runs."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
B, H, N, d = 1, 2, 150, 72
Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16)
w, mu = ba.pack_signs(Q)
ba.pack_signs(Q.float())
ba.binary_logits(w, w, d, head=1)
ba.forward(Q, K, V, bias, kernel="simt")
ba.forward(Q.float(), K.float(), V.float(), bias.float(), kernel="simt")
ba.forward(Q, K, V, bias, quantize_pv=True)
ba.forward(Q, K, V, pkg.Relative1dBias(torch.randn(H, 2 * N - 1, device="cuda")), kernel="simt")
ba.quantize_values(V)
Pb = ba.attention_probs(Q, K, bias, head=1, rows=[0, 7, 149])
Pf = ba.attention_probs(Q, K, bias, head=1, rows=[0, 7, 149], binary=False)
ba.attention_fidelity(Pf, Pb, 5)
torch.cuda.synchronize()
print("ok")
