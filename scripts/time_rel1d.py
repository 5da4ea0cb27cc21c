"""Dev tool: time K2 with no bias / dense bias / relative-1d bias."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]] or [(1, 16, 4096, 64), (1, 16, 4096, 128), (32, 16, 1024, 72), (256, 12, 197, 64)]
for (B, H, N, d) in shapes:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    dense = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    rel = pkg.Relative1dBias(0.5 * torch.randn(H, 2 * N - 1, device="cuda"))
    for name, b in (("none", None), ("dense", dense), ("rel1d", rel)):
        for _ in range(3):
            ba.forward(Q, K, V, b, kernel="tcgen05")
        ba.profile_begin(10)
        for _ in range(10):
            ba.forward(Q, K, V, b, kernel="tcgen05")
        torch.cuda.synchronize()
        n, k1, k2 = ba.profile_end()
        print(f"B{B} H{H} N{N} d{d} bias={name:6s} K1={k1/n*1e3:7.1f} us  K2={k2/n*1e3:8.1f} us", flush=True)
