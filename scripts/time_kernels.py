"""Ad-hoc GPU timing of the two K2 variants over the BASELINE shapes (dev tool, not the bench)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

ba = pkg.BinaryAttention(torch.device("cuda:0"))
shapes = [(1, 3, 197, 64), (256, 12, 197, 64), (64, 16, 256, 72), (32, 16, 1024, 72), (1, 16, 4096, 64), (1, 16, 4096, 128)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
for (B, H, N, d) in shapes:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    for kern in ("tcgen05", "simt"):
        for b in (None, bias):
            if kern == "simt" and N > 1024:
                continue
            t0 = time.time()
            O = ba.forward(Q, K, V, b, kernel=kern); torch.cuda.synchronize()
            first = time.time() - t0
            ba.profile_begin(10)
            for _ in range(10):
                O = ba.forward(Q, K, V, b, kernel=kern)
            torch.cuda.synchronize()
            n, k1, k2 = ba.profile_end()
            eff = 4.0 * B * H * N * N * d / (k2 / n / 1e3) / 1e12
            print(f"B{B} H{H} N{N} d{d} {kern:8s} bias={'y' if b is not None else 'n'} first={first*1e3:9.2f} ms  K1={k1/n*1e3:8.1f} us  K2={k2/n*1e3:9.1f} us  K2 eff={eff:8.1f} TOPS", flush=True)
