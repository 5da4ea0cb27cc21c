"""Dev tool: run-to-run identity of the tcgen05 path (a race shows up as a differing output)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for (B, H, N, d, wb, stats) in [(1, 2, 512, 128, True, True), (1, 2, 512, 128, True, False), (1, 2, 512, 128, False, True), (2, 4, 1024, 64, True, True),
                                (1, 8, 2048, 64, False, False), (1, 3, 320, 72, True, True), (4, 16, 1024, 72, True, False), (1, 16, 4096, 128, True, False), (4, 16, 1024, 72, False, False),
                                (8, 12, 512, 64, True, False), (2, 16, 2048, 128, True, False), (3, 16, 768, 96, True, True), (32, 16, 1024, 72, True, False)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, N, device="cuda")).to(torch.bfloat16) if wb else None
    ref = None
    bad = 0
    worst = 0.0
    for i in range(reps):
        out = ba.forward(Q, K, V, bias, return_stats=stats)
        o = out[0] if stats else out
        torch.cuda.synchronize()
        if ref is None:
            ref = o.clone()
        else:
            diff = (o - ref).abs().max().item()
            if diff != 0.0:
                bad += 1
                worst = max(worst, diff)
    print(f"B{B} H{H} N{N} d{d} bias={wb} stats={stats}: {bad}/{reps - 1} runs differ from the first (max diff {worst:.3e})", flush=True)
