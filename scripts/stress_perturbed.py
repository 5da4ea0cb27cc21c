"""Dev tool: run-to-run identity of the second-generation kernel while a second stream keeps HBM and L2 busy with large copies
(perturbs the timing of every TMA load and barrier hand-over)."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(2)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
side = torch.cuda.Stream()
junk_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
junk_b = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for (B, H, N, d, wb) in [(2, 16, 2048, 128, True), (1, 16, 4096, 128, True), (2, 16, 2048, 96, True), (1, 16, 4096, 64, True), (1, 16, 4096, 128, False),
                         (4, 16, 1024, 72, False), (2, 16, 2048, 64, False), (16, 12, 577, 64, False)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
    ref, bad = None, 0
    for i in range(reps):
        if i % 3 != 0:
            with torch.cuda.stream(side):
                for _ in range(1 + i % 4):
                    junk_b.copy_(junk_a, non_blocking=True)
        o = ba.forward(Q, K, V, bias)
        torch.cuda.synchronize()
        if ref is None:
            ref = o.clone()
        elif not torch.equal(o, ref):
            bad += 1
    print(f"B{B} H{H} N{N} d{d} bias={wb}: {bad}/{reps - 1} runs differ from the first (with concurrent copies on a second stream)", flush=True)
