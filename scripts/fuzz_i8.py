"""Dev tool: random shapes through the integer P.V mode -- tensor-core kernel against the CUDA-core kernel (<= 5e-4), and the
bf16 mode's second-generation kernel against the first-generation one (<= 2e-3) on the same shapes."""
import os, random, sys
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
torch.manual_seed(0)
worst = 0.0
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    B, H = random.choice([(1, 1), (1, 3), (2, 2), (3, 5)])
    N = random.choice([128, 129, 191, 192, 193, 255, 256, 257, 320, 511, 512, 513, 640, 777, 1024, 1100, 1500])
    d = 8 * random.randint(1, 16)
    wb = random.random() < 0.5
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
    a = ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05")
    b = ba.forward(Q, K, V, bias, quantize_pv=True, kernel="simt")
    e = (a - b).abs().max().item()
    os.environ["BA_TC2_MIN_N"] = "128"; os.environ["BA_TC2_MIN_N_BIAS"] = "128"
    c = ba.forward(Q, K, V, bias, kernel="tcgen05")
    os.environ["BA_TC2"] = "0"
    g1 = ba.forward(Q, K, V, bias, kernel="tcgen05")
    del os.environ["BA_TC2"], os.environ["BA_TC2_MIN_N"], os.environ["BA_TC2_MIN_N_BIAS"]
    e2 = (c - g1).abs().max().item()
    bad = e > 5e-4 or e2 > 2e-3 or bool(torch.isnan(a).any()) or bool(torch.isnan(c).any())
    worst = max(worst, e)
    print(f"B{B} H{H} N{N} d{d} bias={wb}: i8 tc-vs-cc {e:.2e}   bf16 gen2-vs-gen1 {e2:.2e} {'  <-- BAD' if bad else ''}", flush=True)
print("worst i8 difference", worst)
