"""Dev tool: first- vs second-generation kernel on short sequences (BA_TC2_MIN_N / BA_TC2_MIN_N_BIAS), alternating, L2 flushed."""
import os, sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B, H, N, d) in [(64, 16, 256, 72), (256, 12, 197, 64), (64, 16, 256, 64), (32, 16, 384, 64), (32, 16, 320, 64), (64, 12, 448, 64), (16, 16, 512, 128)]:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    for wb in (False, True):
        bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N] if wb else None
        ts = {"gen1": [], "gen2": []}
        for it in range(26):
            which = ("gen1", "gen2")[it & 1]
            os.environ["BA_TC2_MIN_N"] = "100000" if which == "gen1" else "128"
            os.environ["BA_TC2_MIN_N_BIAS"] = os.environ["BA_TC2_MIN_N"]
            if it < 4:
                ba.forward(Q, K, V, bias); continue
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ba.forward(Q, K, V, bias); e1.record(); torch.cuda.synchronize()
            ts[which].append(e0.elapsed_time(e1))
        print(f"B{B} H{H} N{N} d{d} bias={wb}: gen1 {statistics.median(ts['gen1']):.4f} ms   gen2 {statistics.median(ts['gen2']):.4f} ms", flush=True)
