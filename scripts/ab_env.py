"""Dev tool: in-process A/B of an environment knob the library reads at every call (alternating settings run by run, L2
flushed before each): python scripts/ab_env.py BA_BIAS_L2 128 256"""
import os, sys, statistics
import torch
sys.path.insert(0, ".")
import paper_2603_09582_b200 as pkg

knob, va, vb = sys.argv[1:4]
small = len(sys.argv) > 4 and sys.argv[4] == "small"
ba = pkg.BinaryAttention(torch.device("cuda:0"))
torch.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
SHAPES = [(64, 12, 577, 64), (32, 16, 1024, 72), (8, 16, 2048, 64), (8, 16, 1536, 128)] if small else \
         [(1, 16, 16384, 128), (1, 16, 16384, 64), (1, 16, 8192, 64), (1, 16, 4096, 64)]
for (B, H, N, d) in SHAPES:
    Q, K, V = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    bias = (0.5 * torch.randn(H, N, (N + 7) // 8 * 8, device="cuda")).to(torch.bfloat16)[:, :, :N]
    ts = {va: [], vb: []}
    for it in range(24):
        v = (va, vb)[it & 1]
        os.environ[knob] = v
        if it < 4:
            ba.forward(Q, K, V, bias); continue
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ba.forward(Q, K, V, bias); e1.record(); torch.cuda.synchronize()
        ts[v].append(e0.elapsed_time(e1))
    print(f"B{B} N{N} d{d} bias: {knob}={va}: {statistics.median(ts[va]):.3f} ms   {knob}={vb}: {statistics.median(ts[vb]):.3f} ms", flush=True)
    del bias
