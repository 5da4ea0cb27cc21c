"""Dev tool: run-to-run identity of the integer P.V mode on the tensor cores (every SM busy, one and two passes, ragged N)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(3)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 150
for (B, H, N, d, wb) in [(256, 12, 197, 64, True), (2, 16, 2048, 64, True), (2, 16, 2048, 128, True), (32, 16, 1024, 72, True), (1, 16, 4096, 64, False),
                         (16, 12, 577, 64, True), (4, 16, 1024, 96, False)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
    ref, bad = None, 0
    for i in range(reps):
        o = ba.forward(Q, K, V, bias, quantize_pv=True, kernel="tcgen05")
        torch.cuda.synchronize()
        if ref is None:
            ref = o.clone()
        elif not torch.equal(o, ref):
            bad += 1
    print(f"B{B} H{H} N{N} d{d} bias={wb}: {bad}/{reps - 1} runs differ from the first", flush=True)
